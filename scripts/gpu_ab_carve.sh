python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
for co in 50 38 64 75; do
  TCG_CARVEOUT=$co timeout 600 python scripts/measure_configs.py C3 C2 C5sweep 2>&1 | sed "s/^/carve=$co /" | cut -c1-150
done
