for v in base ni; do
  TCG_LIBRARY=$PWD/paper_2604_09221_b200/libtcg_$v.so timeout 600 python scripts/measure_configs.py C3 C5sweep 2>&1 | sed "s/^/$v /" | cut -c1-170
done
