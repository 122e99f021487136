# one ncu launch list + one --set full capture of the sweep kernels (TAG=v23)
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_v23.csv $CMD > gpurun_out/ncu_launch.log 2>&1
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k "regex:k_super_build|k_tile_from_super|k_tile_dedup|k_l15_build|k_l2_from_l15|k_l2_dedup|k_l2_classify" -s 8 -c 8 -o gpurun_out/prof_v23 -f $CMD > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
