# A/B the default bench over values of one env switch (alternating), then the GPU tests
# with the default: ENVVAR=TCG_L2F_PAD VALUES="0 40000" bash scripts/gpu_ab_values.sh
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
for rep in 1 2; do for v in $VALUES; do
  export $ENVVAR=$v
  timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  echo "$ENVVAR=$v $(grep -E 'kernel ms by kind' gpurun_out/ab_$v.err | tail -1)"
  python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('value', d['value'], d['parity'])"
done; done
unset $ENVVAR
[ -n "$TESTS" ] && timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
true
