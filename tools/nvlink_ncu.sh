#!/usr/bin/env bash
# NVLink bytes of the exchange kernel on a multi-GPU box, from ncu's NVLink
# counters (NVML's byte counters report NOT_SUPPORTED on this pool's B200s,
# tools/nvml_nvlink_probe.py): rank 0 runs bench.py under ncu with one-pass
# metrics (no kernel replay, which would re-run one rank's kernel without its
# peers), ranks 1..N-1 run plain; the ranks are started by hand with the
# torch.distributed environment variables.  Output: CSV of
# nvltx/nvlrx user bytes and duration per launch of the staged kernel.
#   bash tools/nvlink_ncu.sh N [outdir]
set -u
N=${1:-8}
OUT=${2:-gpurun_out/multigpu}
mkdir -p "$OUT"
PORT=29650
export MASTER_ADDR=127.0.0.1 MASTER_PORT=$PORT WORLD_SIZE=$N
for R in $(seq 1 $((N - 1))); do
  RANK=$R LOCAL_RANK=$R timeout 900 python bench.py --gpus "$N" --steps 10 --warmup 3 --no-e2e \
    --no-cpu-baseline --no-nccl-compare > "$OUT/nvlink_ncu_rank$R.log" 2>&1 &
done
RANK=0 LOCAL_RANK=0 timeout 900 ncu --metrics gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum \
  --replay-mode application -k regex:tm_exchange -c 8 --csv --log-file "$OUT/nvlink_ncu_n$N.csv" \
  python bench.py --gpus "$N" --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-nccl-compare \
  > "$OUT/nvlink_ncu_rank0.log" 2>&1
echo "rank0 rc=$?"
wait
