#!/bin/bash
# One `ncu --set full` capture per kernel regex of the C2 bench workload
# (first guided pass); exports the raw metrics and the source/SASS page as CSV
# next to gpurun_out/ncu_<tag>.log and drops the report unless KEEP_REP=1.
#   tools/ncu_capture.sh tag:regex[:skip] ... [-- extra bench args]
EXTRA=""
SPECS=()
while [ $# -gt 0 ]; do
  if [ "$1" = "--" ]; then shift; EXTRA="$*"; break; fi
  SPECS+=("$1"); shift
done
for spec in "${SPECS[@]}"; do
  IFS=: read -r tag rx skip <<< "$spec"
  rep="/tmp/ncu_$tag"
  ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$rx" -s "${skip:-0}" -c 1 \
      -f -o "$rep" python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
      --no-e2e $EXTRA > "gpurun_out/ncu_$tag.log" 2>&1
  echo "$tag rc=$?"
  ncu -i "$rep.ncu-rep" --page raw --csv > "gpurun_out/ncu_${tag}_raw.csv" 2>/dev/null
  ncu -i "$rep.ncu-rep" --page source --csv --print-source cuda,sass > "gpurun_out/ncu_${tag}_sass.csv" 2>/dev/null
  [ "${KEEP_REP:-0}" = 1 ] && cp "$rep.ncu-rep" gpurun_out/
done
