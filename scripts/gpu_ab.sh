# A/B builds of libtcg: VARIANTS="a b" CONFIGS="C3 C2" bash scripts/gpu_ab.sh
for v in ${VARIANTS:-p1 p2} ${VARIANTS:-p1 p2}; do
  TCG_LIBRARY=$PWD/paper_2604_09221_b200/libtcg_$v.so timeout 600 python scripts/measure_configs.py ${CONFIGS:-C3 C2} 2>&1 | sed "s/^/$v /" | cut -c1-170
done
for v in ${VARIANTS:-p1 p2}; do
  TCG_LIBRARY=$PWD/paper_2604_09221_b200/libtcg_$v.so timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v bench', d['value'], d['roofline']['kernels_ms'], d['parity'])"
done
v=${TEST_VARIANT:-}
if [ -n "$v" ]; then
  TCG_LIBRARY=$PWD/paper_2604_09221_b200/libtcg_$v.so timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1 | sed "s/^/$v /"
fi
