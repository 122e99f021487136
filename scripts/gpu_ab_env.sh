# A/B one build with and without an env switch: LIB=libtcg_x.so ENVVAR=TCG_NO_DEDUP bash scripts/gpu_ab_env.sh
export TCG_LIBRARY=$PWD/paper_2604_09221_b200/${LIB:-libtcg.so}
for v in on off on off; do
  if [ $v = on ]; then unset $ENVVAR; else export $ENVVAR=1; fi
  timeout 600 python scripts/measure_configs.py ${CONFIGS:-C3 C2} 2>&1 | sed "s/^/$v /" | cut -c1-230
done
unset $ENVVAR
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -x -q 2>&1 | tail -2
