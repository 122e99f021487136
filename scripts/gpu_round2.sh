# Round-2 evidence run (one gpurun call): tests, smoke, bench (+ reference arm),
# the launch list of the bench command and an ncu --set full capture of one
# C3 step, converted to profiles-ready JSON.  TAG names the outputs.
set -x
TAG=${TAG:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -x -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"
  tail -5 gpurun_out/pytest_${TAG}.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_${TAG}.json; grep -E "step ms|kernel ms" gpurun_out/bench_${TAG}.err | cut -c1-600
if [ -z "$SKIP_REF" ]; then
  timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err; echo "ref rc=$?"
  cat gpurun_out/bench_ref_${TAG}.json
fi
if [ -z "$SKIP_NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo "ncu launches rc=$?"
  timeout 900 ncu --set full --metrics smsp__thread_inst_executed.sum,smsp__inst_executed.sum --clock-control none --import-source on --profile-from-start off -o gpurun_out/step_${TAG} -f python scripts/profile_step.py c3 > gpurun_out/ncu_step_${TAG}.log 2>&1; echo "ncu step rc=$?"
  tail -2 gpurun_out/ncu_step_${TAG}.log
  python scripts/ncu_kernels_json.py gpurun_out/step_${TAG}.ncu-rep gpurun_out/ncu_kernels_${TAG}.json "ncu --set full, one C3 step (scripts/profile_step.py c3), TAG=${TAG}" > /dev/null 2>&1; echo "parse rc=$?"
  timeout 600 ncu --set full --metrics smsp__thread_inst_executed.sum,smsp__inst_executed.sum --clock-control none --import-source on --profile-from-start off -o gpurun_out/step_c5_${TAG} -f python scripts/profile_step.py c5 > gpurun_out/ncu_step_c5_${TAG}.log 2>&1; echo "ncu c5 rc=$?"
  python scripts/ncu_kernels_json.py gpurun_out/step_c5_${TAG}.ncu-rep gpurun_out/ncu_kernels_c5_${TAG}.json "ncu --set full, one C5 launch (2^26 bowtie8 draws at 2^39, scripts/profile_step.py c5), TAG=${TAG}" > /dev/null 2>&1; echo "parse c5 rc=$?"
  # keep the merged-back output under gpurun's 64 MiB: summaries instead of reports
  python scripts/ncu_lines.py gpurun_out/step_${TAG}.ncu-rep k_l15_build 40 > gpurun_out/l15_lines_${TAG}.txt 2>&1
  python scripts/ncu_summary.py gpurun_out/step_c5_${TAG}.ncu-rep > gpurun_out/c5_full_${TAG}.txt 2>&1
  python scripts/ncu_lines.py gpurun_out/step_c5_${TAG}.ncu-rep k_sample_split 30 >> gpurun_out/c5_full_${TAG}.txt 2>&1
  if [ -z "$KEEP_REP" ]; then rm -f gpurun_out/step_${TAG}.ncu-rep gpurun_out/step_c5_${TAG}.ncu-rep; fi
fi
