# N=2 bench path on one GPU (gloo collectives, both ranks on cuda:0), plus distributed.sweep_sharded
python -c "import __graft_entry__ as g; g.build()" > /dev/null
BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --slice-log2 30 > gpurun_out/multi.json 2> gpurun_out/multi.err
echo "rc=$?"; cat gpurun_out/multi.json; grep -v "^\s" gpurun_out/multi.err | tail -5
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 scripts/sharded_check.py 2>&1 | tail -4
