#!/usr/bin/env bash
# The multi-process exchange (one process per rank, CUDA IPC peer mappings,
# system-scope flags) measured with k processes running CONCURRENTLY on one GPU
# under CUDA MPS: the closest one-GPU stand-in for the one-process-per-GPU
# deployment (every byte moves through this GPU's HBM instead of NVLink).
#   bash tools/mps_multiprocess_bench.sh [k] [steps]
set -u
K=${1:-8}
STEPS=${2:-100}
OUT=gpurun_out/mps
mkdir -p "$OUT"
export CUDA_MPS_PIPE_DIRECTORY=/tmp/tm_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/tm_mps_log
mkdir -p "$CUDA_MPS_PIPE_DIRECTORY" "$CUDA_MPS_LOG_DIRECTORY"
nvidia-cuda-mps-control -d || { echo "MPS daemon did not start"; exit 0; }
PORT=29611
for FL in tmaws tma ws reg; do
  PORT=$((PORT + 1))
  TM_PROCS_PER_GPU=$K TM_STAGED_KERNEL=$FL TM_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run \
    --nnodes=1 --nproc-per-node "$K" --master-addr 127.0.0.1 --master-port "$PORT" bench.py --gpus "$K" \
    --steps "$STEPS" --warmup 5 --no-e2e > "$OUT/bench_k${K}_${FL}.json" 2> "$OUT/bench_k${K}_${FL}.err"
  echo "$FL rc=$?"
done
echo quit | nvidia-cuda-mps-control
