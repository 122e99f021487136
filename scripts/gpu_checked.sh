# Bounds-checked library (-DTCG_CHECKED: device asserts, see tcg.cu) over the
# GPU test suite and the sanitizer targets; compute-sanitizer itself is closed
# on this GPU pool.  Expects build/libtcg_checked.so (built in the container).
mkdir -p gpurun_out
export TCG_LIBRARY=build/libtcg_checked.so
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/checked_pytest.log 2>&1; echo "checked pytest rc=$?"; tail -3 gpurun_out/checked_pytest.log
for f in batch enum sweep7 direct7 sweep8 sweep6 multi large split; do
  timeout 600 python scripts/sanitize.py $f > gpurun_out/checked_$f.log 2>&1; echo "checked $f rc=$? $(tail -1 gpurun_out/checked_$f.log)"
done
