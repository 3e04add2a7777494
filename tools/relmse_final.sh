#!/bin/bash
# End-of-round re-run of the equal-time comparison with the final build:
# cornell_enclosed G = 1 / 2 (4 and 16 samples per pass, N0 64 / 128),
# C2 and C3 with the first bounce guided.  Same protocol as relmse_confirm.sh.
OUT=${OUT:-gpurun_out/relmse_final.jsonl}
mkdir -p gpurun_out
REF=/tmp/ref_enclosed_final.npy
first=1
for g in 1 2; do
  for k in 4 16; do
    for n0 in 64 128; do
      extra="--ref-file $REF"; [ $first = 1 ] && extra="--save-ref $REF"; first=0
      python tools/relmse.py --scene enclosed --svo-res 256 --lmin 4 --c-ray $((512 * k)) \
        --spp 256 --mode wfpg --spp-per-pass $k --field-res $n0 --guided-depths $g --seed 7 \
        --out $OUT $extra > /dev/null || echo "FAILED enclosed $g $k $n0"
    done
  done
done
for sc in c2 c3; do
  python tools/relmse.py --scene $sc --svo-res 256 --lmin 4 --c-ray 8192 --spp 256 \
    --mode wfpg --spp-per-pass 16 --field-res 128 --guided-depths 1 --out $OUT \
    > /dev/null || echo "FAILED $sc"
done
