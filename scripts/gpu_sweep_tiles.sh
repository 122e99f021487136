set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for b in 8 9 10 11; do
  TCG_TILE_BITS=$b timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_t$b.json 2> gpurun_out/bench_t$b.err
  python -c "import json; d=json.load(open('gpurun_out/bench_t$b.json')); print('bits $b value %.4g kernel_ms %.1f e2e %.4g' % (d['value'], d['roofline']['kernel_ms'], d['e2e']['value']), d['parity'])"
done
