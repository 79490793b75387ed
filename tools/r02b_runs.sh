set -u
mkdir -p gpurun_out/r02b
python -m pytest tests/test_gpu_exchange.py -q -x -k "default_staged or oneshot or binding" > gpurun_out/r02b/pytest_small.txt 2>&1; tail -2 gpurun_out/r02b/pytest_small.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02b/bench_n1.json 2> gpurun_out/r02b/bench_n1.err; echo "n1 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02b/bench_n2_nccl.json 2> gpurun_out/r02b/bench_n2_nccl.err; echo "n2 nccl rc=$?"
TM_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e > gpurun_out/r02b/bench_n2_gloo.json 2> gpurun_out/r02b/bench_n2_gloo.err; echo "n2 gloo rc=$?"
export CUDA_MPS_PIPE_DIRECTORY=/tmp/tm_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/tm_mps_log
mkdir -p "$CUDA_MPS_PIPE_DIRECTORY" "$CUDA_MPS_LOG_DIRECTORY"
nvidia-cuda-mps-control -d
TM_PROCS_PER_GPU=4 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29557 tools/latency_mp.py > gpurun_out/r02b/mps_k4.jsonl 2> gpurun_out/r02b/mps_k4.err; echo "mps4 rc=$?"
TM_PROCS_PER_GPU=2 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29558 tools/latency_mp.py --P 4194304,8388608,16777216,60965224 --flavours oneshot,tmaws,tma --reps 3 --inner 8 > gpurun_out/r02b/mps_k2_large.jsonl 2> gpurun_out/r02b/mps_k2_large.err; echo "mps2 large rc=$?"
echo quit | nvidia-cuda-mps-control
