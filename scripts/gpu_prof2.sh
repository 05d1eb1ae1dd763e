#!/bin/bash
OUT=gpurun_out/r1s; mkdir -p $OUT
for c in 5; do EXPMC_B200_LIB=paper_1904_12759_b200/variants/lib_mb7.so timeout 600 python bench.py --config $c --kernel-only --steps 3 --warmup 2 > $OUT/mb7_cfg$c.json 2>&1; done
EXPMC_B200_LIB=paper_1904_12759_b200/variants/lib_mb7.so timeout 600 python bench.py --config 4 --scale 0.1 --kernel-only --steps 3 --warmup 2 > $OUT/mb7_cfg4s.json 2>&1
timeout 600 python bench.py --config 4 --scale 0.1 --kernel-only --steps 3 --warmup 2 > $OUT/def_cfg4s.json 2>&1
timeout 300 python bench.py --kernel-only --steps 2 --warmup 1 > $OUT/plain5.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:entry_walk -s 1 -c 1 -o $OUT/prof_cfg5 python bench.py --kernel-only --steps 2 --warmup 1 > $OUT/ncu5.log 2>&1
timeout 300 python bench.py --config 4 --scale 0.1 --kernel-only --steps 2 --warmup 1 > $OUT/plain4.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:entry_walk -s 1 -c 1 -o $OUT/prof_cfg4s python bench.py --config 4 --scale 0.1 --kernel-only --steps 2 --warmup 1 > $OUT/ncu4.log 2>&1
