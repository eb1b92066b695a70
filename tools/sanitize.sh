#!/bin/bash
# One compute-sanitizer tool (memcheck | racecheck | synccheck) over the kernel families under
# every K4 variant (run under gpurun; one tool per call).  Logs into gpurun_out/san/.
set -u
TOOL=${1:-memcheck}
O=gpurun_out/san
mkdir -p $O
EXTRA=""
[ "$TOOL" = racecheck ] && EXTRA="--racecheck-report hazard"
for V in "default" "RSG_OLA2=5,12" "RSG_IP=9,14 RSG_IP_FORCE=1" "RSG_IP=0,0" "RSG_LARGE_MIN=6"; do
  n=$(echo "$V" | tr -dc "A-Za-z0-9_")
  ENVS=""; [ "$V" != default ] && ENVS="$V"
  env $ENVS timeout 300 python tools/sanitize_case.py > $O/${TOOL}_${n}_plain.log 2>&1 && \
  env $ENVS timeout 1200 compute-sanitizer --tool $TOOL $EXTRA --error-exitcode 9 python tools/sanitize_case.py > $O/${TOOL}_${n}.log 2>&1
  echo "$TOOL $V rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/${TOOL}_${n}.log | tail -1)"
done
