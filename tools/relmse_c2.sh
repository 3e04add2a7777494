#!/bin/bash
# C2 (BASELINE configs[1]: Cornell 1080p, guided vs unguided, SVO depth 10)
# equal-time relMSE with the first bounce guided: SVO 256^3 / 1024^3,
# k = 4 / 16 samples per pass, N0 = 64 / 128, 64 and 256 spp.
OUT=${OUT:-gpurun_out/relmse_c2.jsonl}
mkdir -p gpurun_out
REF=/tmp/ref_c2.npy
first=1
for spp in 64 256; do
  for r in 256 1024; do
    for k in 4 16; do
      for n0 in 64 128; do
        extra="--ref-file $REF"; [ $first = 1 ] && extra="--save-ref $REF"; first=0
        python tools/relmse.py --scene c2 --svo-res $r --lmin 4 --c-ray $((512 * k)) \
          --spp $spp --mode wfpg --spp-per-pass $k --field-res $n0 --guided-depths 1 \
          --out $OUT $extra > /dev/null || echo "FAILED $spp $r $k $n0"
      done
    done
  done
done
