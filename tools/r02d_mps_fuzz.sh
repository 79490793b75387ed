# The multi-process suite (incl. the fuzz at 48 cases per k) with the processes
# concurrent under CUDA MPS.
set -u
O=gpurun_out/r02d/mps
mkdir -p $O
export CUDA_MPS_PIPE_DIRECTORY=/tmp/tm_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/tm_mps_log
mkdir -p "$CUDA_MPS_PIPE_DIRECTORY" "$CUDA_MPS_LOG_DIRECTORY"
nvidia-cuda-mps-control -d || { echo "MPS daemon did not start"; exit 0; }
TM_TEST_MPS=1 TM_MP_FUZZ_CASES=48 timeout 3000 python -m pytest tests/test_gpu_multiprocess.py -q -p no:cacheprovider > $O/pytest_multiprocess_under_mps.txt 2>&1
echo "suite rc=$?"; tail -3 $O/pytest_multiprocess_under_mps.txt
echo quit | nvidia-cuda-mps-control
