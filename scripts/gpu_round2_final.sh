#!/bin/bash
# Round-2 artefacts at one commit (one gpurun call, ~20 GPU-minutes):
#  1. ncu --set full of the walker on every config (full launches) condensed
#     into profiles/r02/ncu_cfg<i>.json, the measured L2 gather ceiling
#     (profiles/r02/l2_gather_peak.json) — bench.py's roofline reads both;
#  2. smoke, the whole GPU test suite;
#  3. bench lines for configs 5 (default), 1-4, the reference arm;
#  4. ncu launch list of the default bench command, the accuracy leg,
#     the self-checking build, one traced host call.
# bash scripts/gpu_round2_final.sh TAG
TAG=${1:-r2final}
OUT=gpurun_out/$TAG; mkdir -p $OUT profiles/r02
export EXPMC_CSR_CACHE=/tmp/expmc_csr_cache
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/smi.txt
# -- 1. captures (each only after the same command ran clean without ncu)
timeout 600 python scripts/l2_gather_peak.py profiles/r02/l2_gather_peak.json > $OUT/l2_peak.log 2>&1
for c in 5 3 2 1 4; do
  timeout 900 python bench.py --config $c --kernel-only --steps 2 --warmup 1 > $OUT/plain_cfg$c.log 2>&1 || { echo "plain cfg$c failed" >> $OUT/errors.txt; continue; }
  SRC=""; [ $c = 5 ] && SRC="--import-source on"
  timeout 1800 ncu --set full --clock-control none $SRC -k regex:entry_walk -s 1 -c 1 -o $OUT/prof_cfg$c \
      python bench.py --config $c --kernel-only --steps 2 --warmup 1 > $OUT/ncu_cfg$c.log 2>&1
  python scripts/ncu_to_profile.py $OUT/prof_cfg$c.ncu-rep $c profiles/r02/ncu_cfg$c.json \
      "ncu --set full --clock-control none, bench.py --config $c --kernel-only, full-size launch ($TAG)" > $OUT/ncu_to_profile_cfg$c.log 2>&1
  python scripts/ncu_summary.py $OUT/prof_cfg$c.ncu-rep > $OUT/ncu_summary_cfg$c.txt 2>&1
  [ $c != 5 ] && rm -f $OUT/prof_cfg$c.ncu-rep     # (64 MiB return limit: keep the headline report only)
done
cp profiles/r02/ncu_cfg*.json profiles/r02/l2_gather_peak.json $OUT/ 2>/dev/null
# -- 2. tests
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke_rc=$?" >> $OUT/smoke.log
timeout 2400 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
# -- 3. bench lines
timeout 900 python bench.py > $OUT/bench_cfg5.json 2> $OUT/bench_cfg5.err
for c in 1 2 3 4; do
  st=10; [ $c = 4 ] && st=3
  timeout 1200 python bench.py --config $c --steps $st --warmup 3 > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/ref_cfg5.json 2> $OUT/ref_cfg5.err
# -- 4. launch list, accuracy, checks build, traced call
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg5.csv \
    python bench.py --kernel-only --steps 2 --warmup 1 > $OUT/ncu_launch.log 2>&1
timeout 2400 python scripts/accuracy.py > $OUT/accuracy.jsonl 2> $OUT/accuracy.err
EXPMC_DEBUG=2 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-ceiling > $OUT/trace_call.json 2> $OUT/trace_call.err
[ -f paper_1904_12759_b200/variants/lib_checks.so ] && bash scripts/gpu_checks.sh $TAG/checks > $OUT/checks.log 2>&1
echo done
