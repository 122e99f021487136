export TCG_LIBRARY=$PWD/paper_2604_09221_b200/${LIB:-libtcg.so}
for c in 18 19 20 21; do
  TCG_CHUNK_LOG2=$c timeout 600 python scripts/measure_configs.py C3 C2 C5sweep 2>&1 | sed "s/^/$c /" | cut -c1-200
done
for c in 18 20; do TCG_CHUNK_LOG2=$c timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('bench chunk $c', d['value'], d['e2e']['value'], d['roofline']['kernels_ms'])"; done
