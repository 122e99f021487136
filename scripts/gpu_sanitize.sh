# compute-sanitizer over every kernel family (scripts/sanitize.py), one small
# launch chain each; summaries to gpurun_out/sanitize/.
mkdir -p gpurun_out/sanitize
FAMS=${FAMS:-"batch enum sweep7 direct7 sweep8 sweep6 multi large"}
TOOLS=${TOOLS:-"memcheck racecheck synccheck initcheck"}
for f in $FAMS; do
  for t in $TOOLS; do
    extra=""
    [ "$t" = "racecheck" ] && extra="--racecheck-report all"
    [ "$t" = "memcheck" ] && extra="--leak-check no"
    timeout ${TMO:-900} compute-sanitizer --tool $t $extra --print-limit 30 python scripts/sanitize.py $f > gpurun_out/sanitize/${f}_${t}.log 2>&1
    rc=$?
    echo "$f $t rc=$rc :: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize target ok' gpurun_out/sanitize/${f}_${t}.log | tr '\n' ' ')"
  done
done
