# gpu tests (subset or all) + default bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu ${TESTK:+-k "$TESTK"} > gpurun_out/gpu_tests.log 2>&1; tail -4 gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err
grep -E "kernel ms|step ms" gpurun_out/ab.err | tail -2; python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('value', d['value'], d['parity'], d['roofline']['dedup'])"
