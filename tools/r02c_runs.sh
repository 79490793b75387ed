set -u
mkdir -p gpurun_out/r02c
python -m pytest tests/test_gpu_exchange.py -q -x -k "range_cta_budget or default_staged" > gpurun_out/r02c/pytest.txt 2>&1; tail -2 gpurun_out/r02c/pytest.txt
timeout 600 python tools/overlap.py > gpurun_out/r02c/overlap.json 2>&1; echo "overlap rc=$?"
timeout 600 python tools/overlap.py --priority > gpurun_out/r02c/overlap_priority.json 2>&1; echo "overlap prio rc=$?"
export CUDA_MPS_PIPE_DIRECTORY=/tmp/tm_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/tm_mps_log
mkdir -p "$CUDA_MPS_PIPE_DIRECTORY" "$CUDA_MPS_LOG_DIRECTORY"
nvidia-cuda-mps-control -d
for N in 8 4 2; do
TM_PROCS_PER_GPU=$N timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$N bench.py --gpus $N --steps 50 --warmup 5 --no-e2e > gpurun_out/r02c/bench_mps_n$N.json 2> gpurun_out/r02c/bench_mps_n$N.err; echo "mps bench n$N rc=$?"
done
echo quit | nvidia-cuda-mps-control
