# per-kernel split of the C3 sweep: short bench + ncu launch list
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/split.json 2> gpurun_out/split.err
cat gpurun_out/split.json; grep -E "kernel ms|step ms" gpurun_out/split.err
CMD="python bench.py --steps 1 --warmup 3 --slice-log2 ${SLICE:-32} --offset 0x5A5A5A5A0 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG:-x}.csv $CMD > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/ncu_launch.log
