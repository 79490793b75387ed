#!/usr/bin/env bash
# The multi-process GPU tests with the processes CONCURRENT on the one GPU under
# CUDA MPS (TM_TEST_MPS=1: each process keeps 1/k of the co-resident CTAs), and
# the random-delay stress at 1,000 exchanges per rank for every staged flavour.
set -u
O=gpurun_out/mps_suite
mkdir -p $O
export CUDA_MPS_PIPE_DIRECTORY=/tmp/tm_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/tm_mps_log
mkdir -p "$CUDA_MPS_PIPE_DIRECTORY" "$CUDA_MPS_LOG_DIRECTORY"
nvidia-cuda-mps-control -d || { echo "MPS daemon did not start"; exit 0; }
TM_TEST_MPS=1 timeout 3000 python -m pytest tests/test_gpu_multiprocess.py -q > $O/pytest_multiprocess_under_mps.txt 2>&1
echo "suite rc=$?"; tail -3 $O/pytest_multiprocess_under_mps.txt
TM_TEST_MPS=1 TM_STRESS_ITERS=1000 timeout 3000 python -m pytest tests/test_gpu_multiprocess.py -q -k stress > $O/pytest_stress_1000_under_mps.txt 2>&1
echo "stress rc=$?"; tail -3 $O/pytest_stress_1000_under_mps.txt
echo quit | nvidia-cuda-mps-control
