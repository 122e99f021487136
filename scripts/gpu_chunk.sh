export TCG_LIBRARY=$PWD/paper_2604_09221_b200/${LIB:-libtcg.so}
for c in ${CHUNKS:-20 21 22 23}; do
  TCG_CHUNK_LOG2=$c timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('bench chunk $c', '%.4g' % d['value'], r['kernels_ms'], r['dedup']['factor'], d['parity'])"
done
