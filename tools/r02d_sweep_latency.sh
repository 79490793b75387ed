# Refresh after the LL default: the one-GPU config sweep (configs 2-5) and the
# small-size latency tables (default flavour vs the others, single process and
# k processes under MPS).
set -u
O=gpurun_out/r02d/sweep
mkdir -p $O
timeout 1800 python tools/sweep.py --md $O/sweep_graph.md > $O/sweep_graph.jsonl 2> $O/sweep.err; echo "sweep rc=$?"
P=2048,8192,32768,65536,131072,262144,524288,1048576,2097152
timeout 900 python tools/latency.py --k 2,4,8 --P $P --flavours default,ll,oneshot,reg,tma,tmaws > $O/latency_single.jsonl 2> $O/latency_single.err; echo "lat rc=$?"
export CUDA_MPS_PIPE_DIRECTORY=/tmp/tm_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/tm_mps_log
mkdir -p "$CUDA_MPS_PIPE_DIRECTORY" "$CUDA_MPS_LOG_DIRECTORY"
nvidia-cuda-mps-control -d
for K in 2 4 8; do
TM_PROCS_PER_GPU=$K timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $K --master-addr 127.0.0.1 \
  --master-port 2987$K tools/latency_mp.py --P $P --flavours default,ll,oneshot,reg,tma,tmaws > $O/latency_mps_k$K.jsonl 2> $O/latency_mps_k$K.err
echo "mps k=$K rc=$?"
done
echo quit | nvidia-cuda-mps-control
