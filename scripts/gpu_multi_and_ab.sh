set -x
mkdir -p gpurun_out
# N>1 through torchrun on the single B200 (gloo collectives; ranks never wait on each other in a kernel)
for mode in "" "--weak"; do
  BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-extra $mode > gpurun_out/bench_n2$mode.json 2> gpurun_out/bench_n2$mode.err; echo "n2 $mode rc=$?"
  tail -c 1500 gpurun_out/bench_n2$mode.json
done
timeout 900 python -m pytest tests/test_gpu_api.py -q -m gpu -k "deterministic or multi_plan" > gpurun_out/pytest_det.log 2>&1; echo "det rc=$?"; tail -2 gpurun_out/pytest_det.log
for v in mb2 mb4; do
  TCG_LIBRARY=build/libtcg_$v.so timeout 600 python bench.py --workload c5 --steps 3 --warmup 2 > gpurun_out/ab_c5_$v.json 2>&1; echo "c5 $v rc=$?"
done
timeout 600 python bench.py --workload c5 --steps 3 --warmup 2 > gpurun_out/ab_c5_mb3.json 2>&1; echo "c5 mb3 rc=$?"
grep -h -o '"workload": "[^"]*"\|"value": [0-9.e+]*\|"kernel_ms_per_step": [0-9.e+]*' gpurun_out/ab_c5_mb*.json
