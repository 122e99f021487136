# one ncu --set full capture of each build-side kernel of the C3 sweep (after a plain run exits 0)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
CMD="python bench.py --steps 1 --warmup 3 --slice-log2 ${SLICE:-30} --offset 0x5A5A5A5A0 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-k_tile_build|k_tile_dedup|k_l2_build|k_l2_dedup|k_tile_classify|k_l2_classify}" -s ${SKIP:-12} -c ${COUNT:-6} -o gpurun_out/prof_${TAG:-x} -f $CMD > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
