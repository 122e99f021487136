python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err
grep "step ms" gpurun_out/bench_d.err
BENCH_NO_CLOCKS=1 timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/bench_d2.json 2> gpurun_out/bench_d2.err
grep "step ms" gpurun_out/bench_d2.err
