#!/bin/bash
# Late-round artefacts: the torchrun (NCCL) launch path of bench.py at one
# rank, both arms, then the K4 (Theorem-2) bench with the CPU reference
# beside it, launch lists of one vector call (cfg 3, cfg 4) and one ncu
# --set full capture of the jumper walk (cfg 3 vector).
TAG=${1:-k4d}
OUT=gpurun_out/$TAG; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517"
timeout 900 $TR bench.py --gpus 1 --steps 5 --warmup 3 > $OUT/torchrun_bench.json 2> $OUT/torchrun_bench.err
timeout 600 $TR bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > $OUT/torchrun_ref.json 2> $OUT/torchrun_ref.err
bash scripts/gpu_k4_prof.sh $TAG
echo done
