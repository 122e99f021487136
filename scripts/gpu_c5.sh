for v in b3 b2 b4; do for co in "" 8 25 50; do
  if [ -n "$co" ]; then export TCG_ENUM_CARVEOUT=$co; else unset TCG_ENUM_CARVEOUT; fi
  TCG_LIBRARY=$PWD/paper_2604_09221_b200/libtcg_$v.so timeout 300 python scripts/measure_configs.py C5 2>&1 | sed "s/^/$v co=$co /" | cut -c1-140
done; done
