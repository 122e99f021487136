# A/B of the flat (per-patchwork) classifier variants on C5 / C4, then the
# GPU tests with the in-tree library.
set -x
mkdir -p gpurun_out
for v in old new mb2; do
  TCG_LIBRARY=build/libtcg_$v.so timeout 600 python bench.py --workload c5 --steps 3 --warmup 2 > gpurun_out/ab_c5_$v.json 2>&1; echo "c5 $v rc=$?"
  TCG_LIBRARY=build/libtcg_$v.so timeout 600 python bench.py --workload c4 --steps 3 --warmup 1 > gpurun_out/ab_c4_$v.json 2>&1; echo "c4 $v rc=$?"
  grep -o '"workload": "[^"]*"\|"value": [0-9.e+]*\|"parity_ok": [a-z]*' gpurun_out/ab_c5_$v.json gpurun_out/ab_c4_$v.json | paste - - - - - - | cut -c1-400
done
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ab.log
