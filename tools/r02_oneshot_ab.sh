#!/usr/bin/env bash
# One-shot kernel A/B: per-CTA chunk 256 / 512 / 1024, one process (k = 8) and
# 8 processes under MPS.
set -u
O=gpurun_out/oneshot_ab
mkdir -p $O
for CH in 256 512 1024; do
  TM_ONESHOT_CHUNK=$CH python tools/latency.py --flavours oneshot --k 2,8 --P 2048,32768,131072 > $O/single_ch$CH.jsonl 2>&1
done
export CUDA_MPS_PIPE_DIRECTORY=/tmp/tm_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/tm_mps_log
mkdir -p "$CUDA_MPS_PIPE_DIRECTORY" "$CUDA_MPS_LOG_DIRECTORY"
nvidia-cuda-mps-control -d
P=29700
for CH in 256 512 1024; do
  P=$((P+1))
  TM_ONESHOT_CHUNK=$CH TM_PROCS_PER_GPU=8 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 \
    --master-addr 127.0.0.1 --master-port $P tools/latency_mp.py --flavours oneshot --P 2048,32768,131072 > $O/mps8_ch$CH.jsonl 2> $O/mps8_ch$CH.err
done
echo quit | nvidia-cuda-mps-control
for f in $O/*.jsonl; do echo "== $f"; python -c "
import json,sys
for l in open('$f'):
    try: r=json.loads(l)
    except Exception: continue
    print(r['P'], r['k'], r.get('C'), round(r.get('us', r.get('us_max_over_ranks', 0)),2))"; done
