#!/usr/bin/env bash
# compute-sanitizer sweep over every kernel path (tools/sanitize.py cases), one process per
# (tool, case) so a failure is attributed; summaries into $OUT/sanitize_summary.txt.
#   gpurun --timeout 1800 -- 'bash tools/sanitize.sh gpurun_out/san'
OUT=${1:-gpurun_out/san}
mkdir -p "$OUT"
CS=${CS:-compute-sanitizer}
export VXQ_WAIT_TIMEOUT_S=120
SUM="$OUT/sanitize_summary.txt"
: > "$SUM"
if ! timeout 300 python tools/sanitize.py > "$OUT/plain.log" 2>&1; then
  echo "plain run failed" | tee -a "$SUM"; exit 1
fi
ALL=$(python tools/sanitize.py --list)
KEY="pa_resident pa_sparse pa_coop sbm_sparse pa_dense sbm_dense sa"
for tool in memcheck racecheck synccheck initcheck; do
  case $tool in memcheck) CASES=$ALL ;; initcheck) CASES="pa_sparse pa_dense sbm_dense sa" ;; *) CASES=$KEY ;; esac
  for c in $CASES; do
    log="$OUT/${tool}_${c}.log"
    timeout 300 $CS --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize.py --case $c > "$log" 2>&1
    rc=$?
    errs=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" "$log" | tail -1)
    echo "$tool $c rc=$rc $errs" | tee -a "$SUM"
  done
done
