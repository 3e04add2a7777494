#!/bin/bash
# One `ncu --set full` capture per kernel regex of the C2 bench workload
# (first guided pass), reports into gpurun_out/ncu_<tag>.ncu-rep.
#   tools/ncu_capture.sh tag:regex[:skip] ... [-- extra bench args]
EXTRA=""
SPECS=()
while [ $# -gt 0 ]; do
  if [ "$1" = "--" ]; then shift; EXTRA="$*"; break; fi
  SPECS+=("$1"); shift
done
for spec in "${SPECS[@]}"; do
  IFS=: read -r tag rx skip <<< "$spec"
  ncu --set full --import-source on --clock-control none -k "regex:$rx" -s "${skip:-0}" -c 1 \
      -f -o "gpurun_out/ncu_$tag" python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
      --no-e2e $EXTRA > "gpurun_out/ncu_$tag.log" 2>&1
  echo "$tag rc=$?"
done
