#!/bin/bash
# Follow-up relMSE sweep: cheaper guided samples within the reference's
# semantics (k samples per render_pass share one set of fields; c_ray scaled
# with k keeps the bin count; N0 64 vs 128), 256 spp, R = 256, l_min 4.
OUT=${OUT:-gpurun_out/relmse_r2b.jsonl}
SPP=${SPP:-256}
mkdir -p gpurun_out
for sc in enclosed c3; do
  REF=/tmp/ref_${sc}.npy
  first=1
  for mode in wfpg wfpg-product; do
    for k in 1 4 16; do
      for n0 in 64 128; do
        cray=$((512 * k))
        extra="--ref-file $REF"
        [ $first = 1 ] && extra="--save-ref $REF"
        python tools/relmse.py --scene $sc --svo-res 256 --lmin 4 --c-ray $cray --spp $SPP \
          --mode $mode --spp-per-pass $k --field-res $n0 --out $OUT $extra > /dev/null \
          || echo "FAILED $sc $mode $k $n0"
        first=0
      done
    done
  done
done
