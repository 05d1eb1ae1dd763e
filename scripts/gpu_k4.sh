#!/bin/bash
# K4 (vector / tc) tests + Theorem-2 throughput on configs 1-4 (GPU only)
TAG=${1:-k4}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_vector.py -x -q > $OUT/pytest_vec.log 2>&1; echo "rc=$?" >> $OUT/pytest_vec.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "vector or tc" > $OUT/pytest_par.log 2>&1; echo "rc=$?" >> $OUT/pytest_par.log
timeout 1200 python scripts/bench_vector.py --no-cpu --steps 2 > $OUT/vec.jsonl 2> $OUT/vec.err
echo done
