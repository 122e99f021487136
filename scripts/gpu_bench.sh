set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 300 python bench.py --steps 2 --warmup 3 --slice-log2 30 --no-cpu-baseline > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err
cat gpurun_out/bench_small.json; tail -5 gpurun_out/bench_small.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
