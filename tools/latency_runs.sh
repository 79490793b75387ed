#!/usr/bin/env bash
# Latency tables (r02): k ranks in one process, and k processes concurrent under MPS.
set -u
OUT=gpurun_out/lat
mkdir -p "$OUT"
timeout 900 python tools/latency.py > "$OUT/single_process.jsonl" 2> "$OUT/single_process.err"
echo "single rc=$?"
export CUDA_MPS_PIPE_DIRECTORY=/tmp/tm_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/tm_mps_log
mkdir -p "$CUDA_MPS_PIPE_DIRECTORY" "$CUDA_MPS_LOG_DIRECTORY"
nvidia-cuda-mps-control -d || { echo "MPS daemon did not start"; exit 0; }
PORT=29711
for K in 8 2; do
  PORT=$((PORT + 1))
  TM_PROCS_PER_GPU=$K timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $K \
    --master-addr 127.0.0.1 --master-port $PORT tools/latency_mp.py > "$OUT/mps_k$K.jsonl" 2> "$OUT/mps_k$K.err"
  echo "mps k=$K rc=$?"
done
echo quit | nvidia-cuda-mps-control
