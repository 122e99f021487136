# super-tile build: identity test, full gpu tests, bench A/B vs the direct contraction
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python -m pytest tests/test_gpu_api.py -x -q -m gpu -k "super_tile or fallback" > gpurun_out/super_test.log 2>&1; tail -15 gpurun_out/super_test.log
timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/ab_super.json 2> gpurun_out/ab_super.err
grep -E "kernel ms|step ms" gpurun_out/ab_super.err | tail -3; python -c "import json; d=json.load(open('gpurun_out/ab_super.json')); print('super4', d['value'], d['parity'], d['roofline']['dedup'])"
TCG_SUPER_BITS=6 timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/ab_super6.json 2> gpurun_out/ab_super6.err
grep -E "kernel ms" gpurun_out/ab_super6.err | tail -2; python -c "import json; d=json.load(open('gpurun_out/ab_super6.json')); print('super6', d['value'], d['parity'])"
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; tail -5 gpurun_out/gpu_tests.log
