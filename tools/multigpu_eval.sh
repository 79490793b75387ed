#!/usr/bin/env bash
# Multi-GPU evaluation for an 8 x B200 box (the one-GPU boxes of rounds 1-2
# cannot run it).  Writes everything under gpurun_out/multigpu/:
#   p2p.jsonl                 peer copy bandwidth of every pair (tools/p2p_probe.py)
#   bench_n{N}_{wl}_{fl}_ag{ag}.json   bench.py at N = 2, 4, 8 per staged flavour and
#                             allgather mode (each line: north-star block, NVML
#                             NVLink bytes vs algorithmic, oracle parity of every rank)
#   bench_n{N}_{strategy}.json         ASA fp32 and AR (NCCL) at AlexNet size
#   ag_table.txt              the allgather decision table (tools/ag_decide.py)
#   nsys_n8.*                 an nsys capture with NVLink GPU metrics, if nsys exists
#   pytest_multiprocess.txt   the multi-process GPU tests with one GPU per rank
#   pytest_multiprocess_cas128_peer.txt   their concurrent-EASGD cases with the
#                             128-bit CAS forced on peer memory (TM_EASGD_CAS128=2)
#   bash tools/multigpu_eval.sh [steps]
set -u
STEPS=${1:-200}
OUT=gpurun_out/multigpu
mkdir -p "$OUT"
NG=$(python -c 'import torch; print(torch.cuda.device_count())')
echo "GPUs: $NG"
python tools/p2p_probe.py > "$OUT/p2p.jsonl" 2>&1
PORT=29511
run() {  # N out-name extra-args...
  local N=$1 NAME=$2; shift 2
  PORT=$((PORT + 1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
    --master-port "$PORT" bench.py --gpus "$N" --steps "$STEPS" --warmup 10 "$@" > "$OUT/$NAME.json" 2> "$OUT/$NAME.err"
  echo "$NAME rc=$?"
}
for N in 2 4 8; do
  [ "$N" -le "$NG" ] || continue
  run "$N" "bench_n${N}_default" --no-e2e
  for WL in alexnet googlenet 1m; do
    for FL in tmaws tma oneshot reg ll ll2; do
      for AG in sm ce nccl; do
        case "$FL" in ll|ll2|oneshot) [ "$AG" = sm ] || continue ;; esac  # no separate allgather phase
        TM_STAGED_KERNEL=$FL TM_ALLGATHER=$AG run "$N" "bench_n${N}_${WL}_${FL}_ag${AG}" --workload "$WL" --no-e2e \
          --no-cpu-baseline --no-nccl-compare
      done
    done
  done
  for S in asa ar; do
    run "$N" "bench_n${N}_${S}" --strategy "$S" --no-e2e
  done
done
python tools/ag_decide.py "$OUT" > "$OUT/ag_table.txt"
# small-message latency per flavour over NVLink (64 exchanges per graph): the
# data for the LL / LL2 / one-shot / two-phase thresholds, which were set from
# one-GPU (MPS) tables
for N in 2 4 8; do
  [ "$N" -le "$NG" ] || continue
  PORT=$((PORT + 1))
  timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
    --master-port "$PORT" tools/latency_mp.py --flavours default,ll,ll2,oneshot,reg,tma,tmaws \
    --P 2048,32768,131072,524288,1048576,2097152,4194304 > "$OUT/latency_flavours_n$N.jsonl" 2> "$OUT/latency_flavours_n$N.err"
  echo "latency N=$N rc=$?"
done
# config 5: message-size sweep 64 KB .. 1 GB (fp32 bytes per rank), ASA16 vs NCCL's allreduce
for N in 2 4 8; do
  [ "$N" -le "$NG" ] || continue
  PORT=$((PORT + 1))
  timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
    --master-port "$PORT" tools/latency_mp.py --nccl --flavours default \
    --P 16384,65536,262144,1048576,4194304,16777216,67108864,268435456 --inner 8 --reps 10 \
    > "$OUT/sweep_n$N.jsonl" 2> "$OUT/sweep_n$N.err"
  echo "sweep N=$N rc=$?"
done
if command -v nsys > /dev/null && [ "$NG" -ge 8 ]; then
  nsys profile --gpu-metrics-devices=all -o "$OUT/nsys_n8" --force-overwrite true \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29599 \
    bench.py --gpus 8 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > "$OUT/nsys_n8.log" 2>&1
  echo "nsys rc=$?"
else
  echo "nsys not installed: NVLink bytes come from the NVML counters in each bench line" > "$OUT/nsys_n8.log"
fi
[ "$NG" -ge 8 ] && bash tools/nvlink_ncu.sh 8 "$OUT"
timeout 3600 python -m pytest tests/test_gpu_multiprocess.py -x -q > "$OUT/pytest_multiprocess.txt" 2>&1
# exact concurrent EASGD with the 128-bit CAS forced on peer GPUs' centre shards
# (over NVLink; the default keeps the 32-bit CAS there): if this passes, the
# 128-bit CAS can be allowed on peer memory too
TM_EASGD_CAS128=2 timeout 900 python -m pytest tests/test_gpu_multiprocess.py -q -k "concurrent" \
  > "$OUT/pytest_multiprocess_cas128_peer.txt" 2>&1
echo "done: $OUT"
