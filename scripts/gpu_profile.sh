# ncu evidence for the bench's dominant kernel (k_enumerate): launch list + one full capture.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
CMD="python bench.py --steps 2 --warmup 3 --slice-log2 28 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
tail -3 gpurun_out/ncu_launch.log
ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 3 -c 1 -o gpurun_out/prof_enum -f $CMD > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
cat gpurun_out/prof_plain.json
