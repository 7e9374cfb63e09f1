#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over tools/sanitize_probe.py -> $1
OUT=${1:-gpurun_out/sanitizer.txt}
echo "# compute-sanitizer on tools/sanitize_probe.py (model / structure cases, 2 kg_step + kg_score each, KG_NO_GRAPH=1, one B200)" > $OUT
for T in memcheck racecheck synccheck initcheck; do
  echo "## $T" >> $OUT
  timeout 900 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_probe.py >> $OUT 2>&1
  echo "exit $?" >> $OUT
done
