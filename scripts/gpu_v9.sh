python -c "import __graft_entry__ as g; g.build()" > /dev/null
for b in 8 9; do TCG_TILE_BITS=$b timeout 300 python scripts/measure_configs.py C3 2>&1 | sed "s/^/bits=$b /" | cut -c1-170; done
timeout 600 python scripts/measure_configs.py C5 C4 2>&1 | cut -c1-200
TAG=v9 bash scripts/gpu_ncu.sh > gpurun_out/v9.log 2>&1; tail -1 gpurun_out/v9.log
