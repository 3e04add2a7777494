#!/bin/bash
# Paper-settings relMSE sweep: SVO 128^3-256^3,
# l_min 4, c_ray 512, guided vs unguided at equal spp and equal time, C2 / C3 /
# cornell_enclosed at 1080p.  Appends JSON lines to $OUT.
OUT=${OUT:-gpurun_out/relmse_r2.jsonl}
SPP=${SPP:-64}
mkdir -p gpurun_out
for sc in c3 enclosed c2; do
  REF=/tmp/ref_${sc}.npy
  first=1
  for res in 128 256; do
    for mode in wfpg wfpg-product; do
      for k in 1 4; do
        extra="--ref-file $REF"
        [ $first = 1 ] && extra="--save-ref $REF"
        python tools/relmse.py --scene $sc --svo-res $res --lmin 4 --c-ray 512 --spp $SPP \
          --mode $mode --spp-per-pass $k --out $OUT $extra > /dev/null || echo "FAILED $sc $res $mode $k"
        first=0
      done
    done
  done
done
