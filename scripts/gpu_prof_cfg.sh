#!/bin/bash
# one ncu --set full capture (with source) of K3: tag cfg [scale]
OUT=gpurun_out/$1; CFG=${2:-5}; SC=${3:-1.0}; mkdir -p $OUT
timeout 300 python bench.py --config $CFG --scale $SC --kernel-only --steps 2 --warmup 1 > $OUT/plain$CFG.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:entry_walk -s 1 -c 1 \
  -o $OUT/prof_cfg$CFG python bench.py --config $CFG --scale $SC --kernel-only --steps 2 --warmup 1 > $OUT/ncu$CFG.log 2>&1
echo rc=$?
