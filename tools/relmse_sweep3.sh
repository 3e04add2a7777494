#!/bin/bash
# Round-2 follow-up relMSE sweep on cornell_enclosed (the scene where guiding
# wins at equal spp), after the guided-pass speedups: guided depths G = 1, 2,
# 4, k = 4 / 16 samples per render_pass (c_ray = 512 k), N0 = 64 / 128, plain
# guiding, SVO 256^3, l_min 4, 256 spp.
OUT=${OUT:-gpurun_out/relmse_r2c.jsonl}
SPP=${SPP:-256}
mkdir -p gpurun_out
REF=/tmp/ref_enclosed.npy
first=1
for g in 1 2 4; do
  for k in 4 16; do
    for n0 in 64 128; do
      cray=$((512 * k))
      extra="--ref-file $REF"
      [ $first = 1 ] && extra="--save-ref $REF"
      python tools/relmse.py --scene enclosed --svo-res 256 --lmin 4 --c-ray $cray --spp $SPP \
        --mode wfpg --spp-per-pass $k --field-res $n0 --guided-depths $g --out $OUT $extra \
        > /dev/null || echo "FAILED $g $k $n0"
      first=0
    done
  done
done
