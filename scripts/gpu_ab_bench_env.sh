# A/B the default bench with an env switch off/on (alternating), then the GPU tests with the
# default: ENVVAR=TCG_L15_STAGE bash scripts/gpu_ab_bench_env.sh
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
for v in 0 1 0 1; do
  export $ENVVAR=$v
  timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  echo "$ENVVAR=$v $(grep -E 'kernel ms by kind' gpurun_out/ab_$v.err | tail -1)"
  python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('value', d['value'], d['parity'])"
done
unset $ENVVAR
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
