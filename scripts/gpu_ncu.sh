# ncu launch list + one --set full capture of the tile kernels, at an unbiased offset
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
CMD="python bench.py --steps 1 --warmup 3 --slice-log2 ${SLICE:-27} --offset 0x5A5A5A5A0 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_${TAG:-x}.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_tile} -s ${SKIP:-6} -c ${COUNT:-2} -o gpurun_out/prof_${TAG:-x} -f $CMD > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
python -c "import json; d=json.load(open('gpurun_out/prof_plain.json')); print(d['value'], d['roofline'])"
