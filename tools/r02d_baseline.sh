set -u
mkdir -p gpurun_out/r02d
nvidia-smi -L > gpurun_out/r02d/gpus.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02d/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02d/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02d/smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r02d/bench_n1.json 2> gpurun_out/r02d/bench_n1.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/r02d/bench_n1.json
