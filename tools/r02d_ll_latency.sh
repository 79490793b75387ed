# Latency of the LL flavour against one-shot / register / TMA: k ranks in one
# process, and k processes concurrent under MPS (64 exchanges per graph).
set -u
O=gpurun_out/r02d/ll_lat
mkdir -p $O
P=2048,8192,32768,65536,131072,262144,524288,1048576
timeout 900 python tools/latency.py --k 2,4,8 --P $P --flavours default,oneshot,reg,ll > $O/single_process.jsonl 2> $O/single_process.err
echo "single rc=$?"
export CUDA_MPS_PIPE_DIRECTORY=/tmp/tm_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/tm_mps_log
mkdir -p "$CUDA_MPS_PIPE_DIRECTORY" "$CUDA_MPS_LOG_DIRECTORY"
nvidia-cuda-mps-control -d
for K in 2 4 8; do
TM_PROCS_PER_GPU=$K timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $K --master-addr 127.0.0.1 \
  --master-port 2977$K tools/latency_mp.py --P $P --flavours default,oneshot,reg,ll > $O/mps_k$K.jsonl 2> $O/mps_k$K.err
echo "mps k=$K rc=$?"
done
echo quit | nvidia-cuda-mps-control
python - <<'PY'
import json, collections, glob
for f in sorted(glob.glob("gpurun_out/r02d/ll_lat/*.jsonl")):
    t = collections.defaultdict(dict)
    for line in open(f):
        try: r = json.loads(line)
        except Exception: continue
        if r.get("path") == "direct": t[(r["k"], r["P"])]["direct"] = r["us"]; continue
        t[(r["k"], r["P"])][r.get("flavour") or "default"] = r["us"]
    print("==", f)
    for key in sorted(t):
        print(key, {k: round(v, 1) for k, v in t[key].items()})
PY
