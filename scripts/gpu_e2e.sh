#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench_cfg5.json 2> $OUT/bench_cfg5.err
timeout 900 python bench.py --config 4 --no-cpu-baseline --steps 3 > $OUT/bench_cfg4.json 2> $OUT/bench_cfg4.err
