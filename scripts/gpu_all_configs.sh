#!/bin/bash
# Per-config bench lines (with the reference CPU baseline) + the accuracy leg.
# usage: bash scripts/gpu_all_configs.sh tag
TAG=${1:-all}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err
done
timeout 1800 python scripts/accuracy.py > $OUT/accuracy.jsonl 2> $OUT/accuracy.err
echo done
