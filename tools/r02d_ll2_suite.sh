set -u
O=gpurun_out/r02d/ll2_suite
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "suite rc=$?"; tail -3 $O/pytest_gpu.txt
for T in memcheck racecheck synccheck; do
  TM_STAGED_KERNEL=ll2 timeout 1500 compute-sanitizer --tool $T --error-exitcode 9 python tests/sanitize_driver.py > $O/san_ll2_$T.txt 2>&1
  echo "san ll2 $T rc=$?"
done
export CUDA_MPS_PIPE_DIRECTORY=/tmp/tm_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/tm_mps_log
mkdir -p "$CUDA_MPS_PIPE_DIRECTORY" "$CUDA_MPS_LOG_DIRECTORY"
nvidia-cuda-mps-control -d
TM_TEST_MPS=1 timeout 3000 python -m pytest tests/test_gpu_multiprocess.py -q -p no:cacheprovider > $O/pytest_mp_under_mps.txt 2>&1
echo "mps suite rc=$?"; tail -2 $O/pytest_mp_under_mps.txt
TM_TEST_MPS=1 TM_STRESS_ITERS=1000 timeout 3000 python -m pytest tests/test_gpu_multiprocess.py -q -p no:cacheprovider -k "stress and (ll or ll2)" > $O/pytest_stress1000_ll_mps.txt 2>&1
echo "mps stress rc=$?"; tail -2 $O/pytest_stress1000_ll_mps.txt
echo quit | nvidia-cuda-mps-control
