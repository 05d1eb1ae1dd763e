#!/bin/bash
# tests + kernel-only timing of the default build on configs given as args
OUT=gpurun_out/$1; shift; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
for c in "$@"; do
  timeout 900 python bench.py --config $c --kernel-only --steps 3 --warmup 2 > $OUT/default_cfg$c.json 2>&1
done
