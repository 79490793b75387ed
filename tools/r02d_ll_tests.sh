set -u
mkdir -p gpurun_out/r02d/ll
timeout 1200 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_bsp.py tests/test_gpu_stress.py tests/test_gpu_variants.py -q -p no:cacheprovider -x -k "ll or fuzz" > gpurun_out/r02d/ll/pytest_sp.txt 2>&1
echo "single-process rc=$?"; tail -3 gpurun_out/r02d/ll/pytest_sp.txt
timeout 1500 python -m pytest tests/test_gpu_multiprocess.py -q -p no:cacheprovider -x -k "ll or fuzz" > gpurun_out/r02d/ll/pytest_mp.txt 2>&1
echo "multi-process rc=$?"; tail -3 gpurun_out/r02d/ll/pytest_mp.txt
