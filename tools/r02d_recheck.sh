set -u
O=gpurun_out/r02d/recheck
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_bsp.py tests/test_gpu_fuzz.py -q -p no:cacheprovider > $O/pytest_bsp_fuzz.txt 2>&1; echo "bsp+fuzz rc=$?"; tail -2 $O/pytest_bsp_fuzz.txt
timeout 900 python tools/latency.py --k 2,4,8 --P 2048,32768,65536,131072,262144,524288 --flavours default,ll,ll2 > $O/latency_single.jsonl 2> $O/latency_single.err; echo "lat rc=$?"
