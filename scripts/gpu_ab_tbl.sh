for v in tb10 tb9 tb8; do
  for co in "" 50 25; do
    TCG_CARVEOUT=$co TCG_LIBRARY=$PWD/paper_2604_09221_b200/libtcg_$v.so timeout 600 python scripts/measure_configs.py C3 2>&1 | sed "s/^/$v carve=$co /" | cut -c1-200
  done
done
bash scripts/gpu_ab_mb.sh
