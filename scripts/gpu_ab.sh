#!/bin/bash
# kernel-only timing of the default build and variants, no tests:
# bash scripts/gpu_ab.sh tag "cfgs" variant...
TAG=$1; CFGS=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
for c in $CFGS; do
  timeout 600 python bench.py --config $c --kernel-only --steps 2 --warmup 1 > $OUT/default_cfg$c.json 2>&1
  for v in "$@"; do
    EXPMC_B200_LIB=paper_1904_12759_b200/variants/lib_$v.so timeout 600 python bench.py --config $c --kernel-only --steps 2 --warmup 1 > $OUT/${v}_cfg$c.json 2>&1
  done
done
