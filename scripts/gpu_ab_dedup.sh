set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_dd.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_dd.log
for v in adaptive full adaptive full; do
  if [ $v = full ]; then export TCG_DEDUP_FULL=1; else unset TCG_DEDUP_FULL; fi
  timeout 600 python bench.py --no-extra --no-cpu-baseline > gpurun_out/bench_dd_$v.json 2> gpurun_out/bench_dd_$v.err; echo "bench $v rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/bench_dd_$v.json'));print('$v', d['value'], d['ms_per_step'], d['parity_ok'], d['roofline']['kernels_ms_per_step'])"
done
