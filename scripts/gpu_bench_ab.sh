set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for v in "" 1; do
  BENCH_NO_CLOCKS=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$v.json 2> gpurun_out/bench_c$v.err
  python -c "import json; d=json.load(open('gpurun_out/bench_c$v.json')); print('noclk=$v value %.4g ms/step %.1f kernel_ms %.1f e2e %.4g' % (d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['e2e']['value']), d['clocks'])"
done
CMD="python bench.py --steps 1 --warmup 3 --slice-log2 28 --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_tile -s 6 -c 2 -o gpurun_out/prof_v4 -f $CMD > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
