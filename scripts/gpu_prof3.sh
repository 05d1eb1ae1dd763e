#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
for c in 5 4; do for v in mb7 mb8; do
  EXPMC_B200_LIB=paper_1904_12759_b200/variants/lib_$v.so timeout 600 python bench.py --config $c --kernel-only --steps 3 --warmup 2 > $OUT/${v}_cfg$c.json 2>&1
done; done
timeout 300 python bench.py --kernel-only --steps 2 --warmup 1 > $OUT/plain5.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:entry_walk -s 1 -c 1 -o $OUT/prof_cfg5 python bench.py --kernel-only --steps 2 --warmup 1 > $OUT/ncu5.log 2>&1
