# Repeats the multi-process fuzz to catch the intermittent self-check fallback.
set -u
mkdir -p gpurun_out/r02d/screpro
for it in $(seq 1 15); do
TM_DEBUG=1 timeout 300 python -m pytest tests/test_gpu_multiprocess.py -q -p no:cacheprovider -x -k "fuzz and 2" -s > gpurun_out/r02d/screpro/k2_$it.txt 2>&1
echo "k2 it $it rc=$? $(grep -c 'self-check' gpurun_out/r02d/screpro/k2_$it.txt)"
done
for it in $(seq 1 5); do
TM_DEBUG=1 timeout 300 python -m pytest tests/test_gpu_multiprocess.py -q -p no:cacheprovider -x -k "fuzz and 3" -s > gpurun_out/r02d/screpro/k3_$it.txt 2>&1
echo "k3 it $it rc=$? $(grep -c 'self-check' gpurun_out/r02d/screpro/k3_$it.txt)"
done
grep -h "\[tm\]" gpurun_out/r02d/screpro/*.txt | sort | uniq -c | head -20
