#!/bin/bash
# One gpurun call: GPU tests, smoke, bench (cfg 5 default + cfg 1), ncu launch
# list and one --set full capture of the walker kernel.  Outputs in gpurun_out/.
# usage: bash scripts/gpu_bench_profile.sh [tag] [skip_tests]
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt
if [ "$2" != "skip_tests" ]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke_rc=$?" >> $OUT/smoke.log
  timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
fi
timeout 900 python bench.py > $OUT/bench_cfg5.json 2> $OUT/bench_cfg5.err; echo "rc=$?" >> $OUT/bench_cfg5.err
timeout 300 python bench.py --config 1 --no-cpu-baseline > $OUT/bench_cfg1.json 2> $OUT/bench_cfg1.err
timeout 300 python bench.py --kernel-only --steps 2 --warmup 1 > $OUT/plain_k.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg5.csv python bench.py --kernel-only --steps 2 --warmup 1 > $OUT/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:entry_walk -s 1 -c 1 -o $OUT/prof_cfg5 python bench.py --kernel-only --steps 2 --warmup 1 > $OUT/ncu_full.log 2>&1
echo done
