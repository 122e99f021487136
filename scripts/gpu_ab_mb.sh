for v in "" _mb3 _mb4; do
  TCG_LIBRARY=$PWD/paper_2604_09221_b200/libtcg$v.so timeout 600 python scripts/measure_configs.py C5 2>&1 | sed "s/^/mb$v /" | cut -c1-220
done
