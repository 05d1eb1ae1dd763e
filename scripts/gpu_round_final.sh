#!/bin/bash
# Round artefacts after K4 v2: smoke, all GPU tests, bench lines cfg 1-5,
# reference arm, Theorem-2 bench with CPU reference, K3 launch list,
# ncu --set full of the K4 jumper walk (cfg 3 vector).
TAG=${1:-final}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi > $OUT/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke_rc=$?" >> $OUT/smoke.log
timeout 1200 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for c in 1 2 3 4; do
  st=10; [ $c = 4 ] && st=3
  timeout 1200 python bench.py --config $c --steps $st --warmup 3 > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/ref_cfg5.json 2> $OUT/ref_cfg5.err
timeout 1500 python scripts/bench_vector.py --steps 3 > $OUT/vec.jsonl 2> $OUT/vec.err
timeout 600 python scripts/vec_once.py 3 > $OUT/plain_vec3.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_vec_cfg3.csv python scripts/vec_once.py 3 > $OUT/ncu_launch_vec3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vec_walk -s 1 -c 1 -o $OUT/prof_vec_cfg3 python scripts/vec_once.py 3 > $OUT/ncu_full_vec.log 2>&1
echo done
