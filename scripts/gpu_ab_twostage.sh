# A/B: two-stage vs direct level 2 (TCG_L2_TWOSTAGE), after the related GPU tests
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "two_stage or level2 or parity or dedup or super_tile" 2>&1 | tail -3
for cfg in "TCG_L2_TWOSTAGE=0" "TCG_L2_TWOSTAGE=1"; do
  env $cfg timeout 600 python bench.py --no-cpu-baseline > gpurun_out/abt.json 2> gpurun_out/abt.err
  echo "$cfg"; grep -E "kernel ms by kind" gpurun_out/abt.err | tail -1; tail -1 gpurun_out/abt.err | cut -c1-300
  python -c "import json; d=json.load(open('gpurun_out/abt.json')); print('  value %.4g e2e %.4g' % (d['value'], d['e2e']['value']), d['parity'], d['roofline']['dedup'])"
done
