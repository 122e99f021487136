# A/B two builds of libtcg: VARIANTS="p1 p2" bash scripts/gpu_ab.sh
for v in ${VARIANTS:-p1 p2} ${VARIANTS:-p1 p2}; do
  TCG_LIBRARY=$PWD/paper_2604_09221_b200/libtcg_$v.so timeout 600 python scripts/measure_configs.py ${CONFIGS:-C3 C2} 2>&1 | sed "s/^/$v /" | cut -c1-170
done
for v in ${VARIANTS:-p1 p2}; do
  TCG_LIBRARY=$PWD/paper_2604_09221_b200/libtcg_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 | sed "s/^/$v /"
done
