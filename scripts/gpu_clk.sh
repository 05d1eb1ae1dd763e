#!/bin/bash
OUT=gpurun_out/r1r; mkdir -p $OUT
for c in 1 5; do
  timeout 600 python bench.py --config $c --kernel-only --steps 10 --warmup 3 > $OUT/nvml_cfg$c.json 2>&1
done
timeout 300 python scripts/diag_steps.py 5 > $OUT/diag5.log 2>&1
