#!/bin/bash
OUT=gpurun_out/r1q; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python scripts/diag_steps.py 1 > $OUT/diag1.log 2>&1
timeout 300 python scripts/diag_steps.py 5 > $OUT/diag5.log 2>&1
for c in 5 1 2 4; do
  timeout 600 python bench.py --config $c --kernel-only --steps 3 --warmup 2 > $OUT/default_cfg$c.json 2>&1
  for v in r4c256; do
    EXPMC_B200_LIB=paper_1904_12759_b200/variants/lib_$v.so timeout 600 python bench.py --config $c --kernel-only --steps 3 --warmup 2 > $OUT/${v}_cfg$c.json 2>&1
  done
done
