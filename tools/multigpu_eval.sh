#!/usr/bin/env bash
# Multi-GPU evaluation for an 8 x B200 box (not runnable on the one-GPU boxes of
# round 1).  Writes everything under gpurun_out/multigpu/.
#   bash tools/multigpu_eval.sh [steps]
set -u
STEPS=${1:-200}
OUT=gpurun_out/multigpu
mkdir -p "$OUT"
NG=$(python -c 'import torch; print(torch.cuda.device_count())')
echo "GPUs: $NG"
python tools/p2p_probe.py > "$OUT/p2p.jsonl" 2>&1
PORT=29511
for N in 2 4 8; do
  [ "$N" -le "$NG" ] || continue
  for FL in tmaws tma ws reg; do
    for AG in sm ce nccl; do
      PORT=$((PORT + 1))
      TM_STAGED_KERNEL=$FL TM_ALLGATHER=$AG timeout 600 python -m torch.distributed.run --nnodes=1 \
        --nproc-per-node "$N" --master-addr 127.0.0.1 --master-port "$PORT" bench.py --gpus "$N" \
        --steps "$STEPS" --warmup 10 --no-e2e > "$OUT/bench_n${N}_${FL}_${AG}.json" 2> "$OUT/bench_n${N}_${FL}_${AG}.err"
      echo "N=$N $FL $AG rc=$?"
    done
  done
  for S in asa ar; do
    PORT=$((PORT + 1))
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
      --master-port "$PORT" bench.py --gpus "$N" --strategy "$S" --steps "$STEPS" --warmup 10 --no-e2e \
      > "$OUT/bench_n${N}_${S}.json" 2> "$OUT/bench_n${N}_${S}.err"
  done
done
timeout 3600 python -m pytest tests/test_gpu_multiprocess.py -x -q > "$OUT/pytest_multiprocess.txt" 2>&1
echo "done: $OUT"
