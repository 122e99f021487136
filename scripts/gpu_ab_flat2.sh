# A/B of the full-diamond classifier: region graph at close (adj) vs per-region
# vertex + crossed sets (xsets), C5 and C4 alternating, then the parity tests
# that exercise the flat kernel with the adj library.
set -x
mkdir -p gpurun_out
for i in 1 2; do
  for v in xsets adj; do
    TCG_LIBRARY=build/libtcg_$v.so timeout 600 python bench.py --workload c5 --steps 3 --warmup 2 > gpurun_out/f2_c5_$v$i.json 2>&1
    TCG_LIBRARY=build/libtcg_$v.so timeout 600 python bench.py --workload c4 --steps 3 --warmup 1 > gpurun_out/f2_c4_$v$i.json 2>&1
    grep -h -o '"workload": "c[45][^"]*"\|"value": [0-9.e+]*\|"kernel_ms_per_step": [0-9.e+]*\|"parity_ok": [a-z]*' gpurun_out/f2_c5_$v$i.json gpurun_out/f2_c4_$v$i.json | tr '\n' ' '; echo " <- $v$i"
  done
done
TCG_LIBRARY=build/libtcg_adj.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_status.py tests/test_gpu_api.py -x -q -m gpu > gpurun_out/f2_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/f2_pytest.log
