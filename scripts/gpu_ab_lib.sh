# A/B of the in-tree library against build/libtcg_base.so on the default C3
# bench (alternating, REPS times each; "new34" = in-tree with 2^34 chunks),
# then the GPU tests with the in-tree library.
set -x
mkdir -p gpurun_out
for i in $(seq 1 ${REPS:-2}); do
  for v in base new new34; do
    unset TCG_LIBRARY TCG_CHUNK_INDEX_LOG2
    [ $v = base ] && export TCG_LIBRARY=build/libtcg_base.so
    [ $v = new34 ] && export TCG_CHUNK_INDEX_LOG2=34
    timeout 600 python bench.py --no-extra --no-cpu-baseline > gpurun_out/ab_$v$i.json 2> gpurun_out/ab_$v$i.err
    python -c "import json;d=json.load(open('gpurun_out/ab_$v$i.json'));print('$v', d['value'], d['ms_per_step'], d['parity_ok'], d['work_avoidance']['dedup_factor_per_rank'], d['roofline']['kernels_ms_per_step'])"
  done
done
unset TCG_LIBRARY TCG_CHUNK_INDEX_LOG2
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_ab2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ab2.log
fi
