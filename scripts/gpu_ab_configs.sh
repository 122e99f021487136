# A/B the default bench over env configurations (':'-separated assignments, alternating twice):
# CONFIGS="X=1 X=0:Y=2" bash scripts/gpu_ab_configs.sh   (TESTS=1: then the GPU tests, default env)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
for rep in 1 2; do for c in $CONFIGS; do
  tag=$(echo "$c" | tr ':=/.' '____' | tail -c 60)
  env $(echo "$c" | tr ':' ' ') timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
  echo "$c $(grep -E 'kernel ms by kind' gpurun_out/ab_$tag.err | tail -1)"
  python -c "import json; d=json.load(open('gpurun_out/ab_$tag.json')); print('value', d['value'], d['parity'])"
done; done
[ -n "$TESTS" ] && timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
true
