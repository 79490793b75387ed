# LL2 (two-shot LL): correctness (fuzz, BSP, stress, variants, multi-process) and
# latency against the other flavours, single process and k processes under MPS.
set -u
O=gpurun_out/r02d/ll2
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_bsp.py tests/test_gpu_stress.py tests/test_gpu_variants.py -q -p no:cacheprovider -x -k "ll2 or fuzz" > $O/pytest_sp.txt 2>&1
echo "single-process rc=$?"; tail -2 $O/pytest_sp.txt
timeout 1500 python -m pytest tests/test_gpu_multiprocess.py -q -p no:cacheprovider -x -k "ll2 or fuzz" > $O/pytest_mp.txt 2>&1
echo "multi-process rc=$?"; tail -2 $O/pytest_mp.txt
P=32768,65536,131072,262144,524288,1048576,2097152,4194304
timeout 900 python tools/latency.py --k 2,4,8 --P $P --flavours default,ll,ll2,oneshot,reg,tma,tmaws > $O/latency_single.jsonl 2> $O/latency_single.err; echo "lat rc=$?"
export CUDA_MPS_PIPE_DIRECTORY=/tmp/tm_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/tm_mps_log
mkdir -p "$CUDA_MPS_PIPE_DIRECTORY" "$CUDA_MPS_LOG_DIRECTORY"
nvidia-cuda-mps-control -d
for K in 2 4 8; do
TM_PROCS_PER_GPU=$K timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $K --master-addr 127.0.0.1 \
  --master-port 2997$K tools/latency_mp.py --P $P --flavours default,ll,ll2,oneshot,reg,tma,tmaws > $O/latency_mps_k$K.jsonl 2> $O/latency_mps_k$K.err
echo "mps k=$K rc=$?"
done
echo quit | nvidia-cuda-mps-control
