#!/bin/bash
# ncu --set full of K3 for the default build and variants on one config:
# bash scripts/gpu_prof_ab.sh tag cfg scale variant...
TAG=$1; CFG=$2; SC=$3; shift 3
OUT=gpurun_out/$TAG; mkdir -p $OUT
run() {  # name lib
  EXPMC_B200_LIB=$2 timeout 300 python bench.py --config $CFG --scale $SC --kernel-only --no-cpu-baseline --no-ceiling --steps 2 --warmup 1 > $OUT/$1_cfg$CFG.json 2>&1
  EXPMC_B200_LIB=$2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:entry_walk -s 1 -c 1 \
    -o $OUT/prof_$1_cfg$CFG python bench.py --config $CFG --scale $SC --kernel-only --no-cpu-baseline --no-ceiling --steps 1 --warmup 1 > $OUT/ncu_$1.log 2>&1
}
run default paper_1904_12759_b200/libexpmc_b200.so
for v in "$@"; do run $v paper_1904_12759_b200/variants/lib_$v.so; done
echo done
