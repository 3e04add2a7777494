#!/bin/bash
# Equal-time confirmation runs (round 2): guided first bounce only (G = 1),
# the winning settings of relmse_sweep3.sh, three seeds at 256 spp and one
# 1024 spp run on cornell_enclosed; G = 1 on C2 and C3 for comparison.
OUT=${OUT:-gpurun_out/relmse_confirm.jsonl}
mkdir -p gpurun_out
REF=/tmp/ref_enclosed.npy
first=1
for seed in 7 11 13; do
  for k in 4 16; do
    for n0 in 64 128; do
      extra="--ref-file $REF"; [ $first = 1 ] && extra="--save-ref $REF"; first=0
      python tools/relmse.py --scene enclosed --svo-res 256 --lmin 4 --c-ray $((512 * k)) \
        --spp 256 --mode wfpg --spp-per-pass $k --field-res $n0 --guided-depths 1 --seed $seed \
        --out $OUT $extra > /dev/null || echo "FAILED enclosed $seed $k $n0"
    done
  done
done
python tools/relmse.py --scene enclosed --svo-res 256 --lmin 4 --c-ray 8192 --spp 1024 \
  --mode wfpg --spp-per-pass 16 --field-res 128 --guided-depths 1 --out $OUT --ref-file $REF \
  > /dev/null || echo "FAILED enclosed 1024"
for sc in c2 c3; do
  python tools/relmse.py --scene $sc --svo-res 256 --lmin 4 --c-ray 8192 --spp 256 \
    --mode wfpg --spp-per-pass 16 --field-res 128 --guided-depths 1 --out $OUT \
    > /dev/null || echo "FAILED $sc"
done
