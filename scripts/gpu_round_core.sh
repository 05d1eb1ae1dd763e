#!/bin/bash
# Core round artefacts: smoke, GPU tests, default bench (cfg 5), reference
# arm, launch list + one ncu --set full capture of the walker on cfg 5.
TAG=${1:-core}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi > $OUT/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke_rc=$?" >> $OUT/smoke.log
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for c in ${CONFIGS:-}; do
  st=10; [ $c = 4 ] && st=3
  timeout 1200 python bench.py --config $c --steps $st --warmup 3 > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/ref_cfg5.json 2> $OUT/ref_cfg5.err
timeout 300 python bench.py --kernel-only --steps 2 --warmup 1 > $OUT/plain_k.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg5.csv python bench.py --kernel-only --steps 2 --warmup 1 > $OUT/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:entry_walk -s 1 -c 1 -o $OUT/prof_cfg5 python bench.py --kernel-only --steps 2 --warmup 1 > $OUT/ncu_full.log 2>&1
echo done
