# A/B: tile bits and super bits on the C3 bench (same binary)
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out
for cfg in "TCG_TILE_BITS=9 TCG_SUPER_BITS=5" "TCG_TILE_BITS=9 TCG_SUPER_BITS=6" "TCG_TILE_BITS=10 TCG_SUPER_BITS=4" "TCG_TILE_BITS=10 TCG_SUPER_BITS=5"; do
  env $cfg timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/abb.json 2> gpurun_out/abb.err
  echo "$cfg"; grep -E "kernel ms by kind" gpurun_out/abb.err | tail -1
  python -c "import json; d=json.load(open('gpurun_out/abb.json')); print('  value %.4g' % d['value'], d['parity'], d['roofline']['dedup']['distinct_tiles'], d['roofline']['dedup']['level2_records'], d['roofline']['dedup']['level2_distinct'])"
done
