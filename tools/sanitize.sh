#!/bin/bash
# compute-sanitizer over the -m gpu suite (GPU box):  bash tools/sanitize.sh [outdir]
# memcheck over everything except the n = 2^22 cases (instrumented 4M-row kernels
# take tens of minutes); racecheck / synccheck / initcheck over the parity, API,
# Newton and leverage tests at their small sizes.  One log per tool.
OUT=${1:-gpurun_out/sanitizer}
mkdir -p "$OUT"
CS="compute-sanitizer --print-limit 50 --error-exitcode 99 --target-processes all"
SMALL='not c4_full and not census and not dist and not dropin and not 4000 and not 10000 and not 8192 and not 6000 and not n5000'
run() {
  local tool=$1; shift
  local sel=$1; shift
  timeout ${TMO:-1500} $CS --tool $tool "$@" python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$sel" \
      > "$OUT/$tool.log" 2>&1
  echo "$tool rc=$?" | tee -a "$OUT/summary.txt"
  grep -E "ERROR SUMMARY|passed|failed" "$OUT/$tool.log" | tail -3 | tee -a "$OUT/summary.txt"
}
: > "$OUT/summary.txt"
run memcheck "not c4_full and not dist and not dropin"
run racecheck "$SMALL" --racecheck-report all
run synccheck "$SMALL"
run initcheck "$SMALL"
