# compute-sanitizer over every device entry point (tools/sanitize.py) on small
# problems; summaries into gpurun_out/sanitize_<tool>_<problem>.log
#   bash tools/sanitize.sh [problems...]
PROBS=${*:-"mixed c1 c3:0.1"}
for t in memcheck racecheck synccheck initcheck; do
  for p in $PROBS; do
    log=gpurun_out/sanitize_${t}_${p/:/_}.log
    timeout ${SAN_TIMEOUT:-900} compute-sanitizer --tool $t --error-exitcode 9 --print-limit 20 python tools/sanitize.py $p > $log 2>&1
    echo "$t $p rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize workload ok' $log | tr '\n' ' ')"
  done
done
