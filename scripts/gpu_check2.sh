set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 600 python scripts/measure_configs.py C2 C3 C5sweep 2>&1 | tail -5
timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/bq.json 2> gpurun_out/bq.err
python -c "import json; d=json.load(open('gpurun_out/bq.json')); r=d['roofline']; print('value %.4g e2e %.4g frac %.4f' % (d['value'], d['e2e']['value'], r['frac']), r['kernels_ms'], d['parity'], d['clocks'])"
