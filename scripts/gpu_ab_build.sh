# fast vs generic tile build: gpu tests, then the bench both ways
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; tail -15 gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/ab_fast.json 2> gpurun_out/ab_fast.err
grep -E "kernel ms|step ms" gpurun_out/ab_fast.err; python -c "import json; d=json.load(open('gpurun_out/ab_fast.json')); print('fast', d['value'], d['parity'])"
TCG_BUILD_GENERIC=1 timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/ab_gen.json 2> gpurun_out/ab_gen.err
grep -E "kernel ms" gpurun_out/ab_gen.err; python -c "import json; d=json.load(open('gpurun_out/ab_gen.json')); print('generic', d['value'], d['parity'])"
