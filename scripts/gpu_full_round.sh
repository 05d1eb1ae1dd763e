#!/bin/bash
# Round artefacts: GPU tests, smoke, all-config bench lines (reference CPU
# baseline included), accuracy leg, launch list + ncu --set full of the
# walker on config 5.
TAG=${1:-full}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke_rc=$?" >> $OUT/smoke.log
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
for c in 5 1 2 3 4; do
  st=10; [ $c = 4 ] && st=3
  timeout 1200 python bench.py --config $c --steps $st --warmup 3 > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/ref_cfg5.json 2> $OUT/ref_cfg5.err
timeout 2400 python scripts/accuracy.py > $OUT/accuracy.jsonl 2> $OUT/accuracy.err
timeout 300 python bench.py --kernel-only --steps 2 --warmup 1 > $OUT/plain_k.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg5.csv python bench.py --kernel-only --steps 2 --warmup 1 > $OUT/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:entry_walk -s 1 -c 1 -o $OUT/prof_cfg5 python bench.py --kernel-only --steps 2 --warmup 1 > $OUT/ncu_full.log 2>&1
echo done
