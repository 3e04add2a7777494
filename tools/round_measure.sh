#!/bin/bash
# End-of-round measurements on one B200 -> gpurun_out/round/ (copy to profiles/ after):
# bench lines (C2 headline with CPU baseline, C3, product, 4K, tess, reference arm),
# the C2 launch list, and one ncu --set full capture of the depth-1 field kernel.
set -x
O=gpurun_out/round
mkdir -p $O
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --scene c3 > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --product --no-cpu-baseline > $O/bench_prod.json 2> $O/bench_prod.err
python bench.py --width 3840 --height 2160 --no-cpu-baseline > $O/bench_4k.json 2> $O/bench_4k.err
python bench.py --scene tess --no-cpu-baseline > $O/bench_tess.json 2> $O/bench_tess.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
    > $O/launches_c2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file $O/launches_c3.csv python bench.py --scene c3 --steps 2 --warmup 1 --no-cpu-baseline \
    --no-e2e > $O/launches_c3.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:fields<.int.128" -c 1 -f -o /tmp/f128 python bench.py --no-cpu-baseline --no-e2e \
    --steps 1 --warmup 0 > $O/ncu_f128.log 2>&1
ncu -i /tmp/f128.ncu-rep --page raw --csv > $O/ncu_f128_raw.csv 2>/dev/null
ncu -i /tmp/f128.ncu-rep --page source --csv --print-source cuda,sass > $O/ncu_f128_source.csv 2>/dev/null
python bench.py --impl reference > $O/bench_reference_c2.json 2> $O/bench_reference_c2.err
ls -la $O
python tools/bench_c5.py --check-n 1100000 > $O/c5.jsonl 2> $O/c5.err
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:k_shade" -s 4 -c 1 -f -o /tmp/shade python bench.py --no-cpu-baseline --no-e2e \
    --steps 1 --warmup 3 > $O/ncu_shade.log 2>&1
ncu -i /tmp/shade.ncu-rep --page raw --csv > $O/ncu_shade_raw.csv 2>/dev/null
