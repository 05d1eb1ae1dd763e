#!/bin/bash
# K4 round artefacts: Theorem-2 bench with the CPU reference beside it,
# launch lists of one vector call (cfg 3, cfg 4) and one ncu --set full
# capture of the jumper walk (cfg 3 vector).
TAG=${1:-k4p}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1500 python scripts/bench_vector.py --steps 3 > $OUT/vec.jsonl 2> $OUT/vec.err
for c in 3 4; do
  timeout 600 python scripts/vec_once.py $c > $OUT/plain_cfg$c.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_vec_cfg$c.csv python scripts/vec_once.py $c > $OUT/ncu_launch_cfg$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vec_walk -s 1 -c 1 -o $OUT/prof_vec_cfg3 python scripts/vec_once.py 3 > $OUT/ncu_full.log 2>&1
echo done
