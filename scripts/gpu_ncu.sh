# one ncu --set full capture of k_enumerate (bench command, 2^28 slices)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
CMD="python bench.py --steps 1 --warmup 3 --slice-log2 28 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_enumerate} -s 3 -c 1 -o gpurun_out/prof_${TAG:-x} -f $CMD > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
