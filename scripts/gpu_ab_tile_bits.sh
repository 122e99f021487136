# A/B: tile sizes (TCG_TILE_BITS) and super-tile sizes on the C3 bench (same binary)
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out
for cfg in "TCG_TILE_BITS=11" "TCG_TILE_BITS=12" "TCG_TILE_BITS=12 TCG_SUPER_BITS=5"; do
  env $cfg timeout 600 python bench.py --no-cpu-baseline > gpurun_out/abb.json 2> gpurun_out/abb.err
  echo "$cfg"; grep -E "kernel ms by kind" gpurun_out/abb.err | tail -1; tail -1 gpurun_out/abb.err | cut -c1-200
  python -c "import json; d=json.load(open('gpurun_out/abb.json')); print('  value %.4g' % d['value'], d['parity'], d['roofline']['dedup']['distinct_tiles'], d['roofline']['dedup']['level2_records'])"
done
