set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for cfg in "8 lanes" "9 lanes" "10 lanes" "10 warp"; do
  set -- $cfg
  if [ "$2" = warp ]; then export TCG_BUILD_WARP=1; else unset TCG_BUILD_WARP; fi
  TCG_TILE_BITS=$1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bt.json 2> gpurun_out/bt.err
  python -c "import json; d=json.load(open('gpurun_out/bt.json')); r=d['roofline']; print('bits $1 $2 value %.4g e2e %.4g kms' % (d['value'], d['e2e']['value']), r['kernels_ms'], d['parity'])"
done
