python -c "import __graft_entry__ as g; g.build()" > /dev/null
CMD="python scripts/prof_target.py bowtie8 rep 0x4000000000 0x4000000"
$CMD && ncu --set full --clock-control none --import-source on -k regex:k_tile_classify -s 2 -c 1 -o gpurun_out/prof_d8 -f $CMD > gpurun_out/ncu_d8.log 2>&1
CMD2="python scripts/prof_target.py bowtie8 sample 0x8000000000 0x1000000"
$CMD2 && ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 2 -c 1 -o gpurun_out/prof_c5 -f $CMD2 > gpurun_out/ncu_c5.log 2>&1
tail -1 gpurun_out/ncu_d8.log gpurun_out/ncu_c5.log
