#!/bin/bash
# Correctness of the default build + timing of tuning variants.
# usage: bash scripts/gpu_variants.sh tag "cfgs" [variant names...]
TAG=$1; CFGS=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
for c in $CFGS; do
  timeout 600 python bench.py --config $c --kernel-only --steps 3 --warmup 2 > $OUT/default_cfg$c.json 2>&1
  for v in "$@"; do
    EXPMC_B200_LIB=paper_1904_12759_b200/variants/lib_$v.so timeout 600 python bench.py --config $c --kernel-only --steps 3 --warmup 2 > $OUT/${v}_cfg$c.json 2>&1
  done
done
echo done
