for rep in 1 2; do for v in 8 100000; do
  TCG_L2B_GRID=$v timeout 300 python scripts/measure_configs.py C2 C5sweep 2>&1 | sed "s/^/grid=$v /" | cut -c1-260
done; done
