# A/B of TCG_FLAT_BATCH builds (build/libtcg_b<N>.so): C4 and the flat C5 sampler
for pass in 1 2; do
  for b in ${BATCHES:-1 2 3 4}; do
    export TCG_LIBRARY=build/libtcg_b$b.so
    c4=$(timeout 600 python bench.py --workload c4 --steps 3 --warmup 1 2>/dev/null | python -c "import json,sys; print(round(json.loads(sys.stdin.read().strip().splitlines()[-1])['value']/1e9,3))")
    c5=$(timeout 300 python scripts/c5_split_ab.py 24 bowtie8 delaunay-8 2>&1 | grep -o "flat [0-9.]*e9" | tr '\n' ' ')
    echo "pass $pass batch $b: c4 $c4 e9 pairs/s; $c5"
  done
done
