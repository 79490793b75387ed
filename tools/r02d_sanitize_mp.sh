# compute-sanitizer (memcheck, synccheck, racecheck) on every worker process of
# the multi-process fuzz (TM_TEST_SANITIZER): IPC peer loads, system-scope flags.
set -u
O=gpurun_out/r02d/san_mp
mkdir -p $O
export TM_MP_FUZZ_CASES=8
for T in memcheck synccheck racecheck; do
  for K in 2 3; do
    rm -rf /tmp/tm_san_$T$K; mkdir -p /tmp/tm_san_$T$K
    TM_TEST_SANITIZER=$T timeout 2400 python -m pytest tests/test_gpu_multiprocess.py -q -p no:cacheprovider -x \
      -k "fuzz and $K" --basetemp=/tmp/tm_san_$T$K > $O/pytest_$T$K.txt 2>&1
    echo "$T k=$K rc=$? $(tail -1 $O/pytest_$T$K.txt)"
    for f in $(find /tmp/tm_san_$T$K -name "san_*rank*.txt"); do cp $f $O/$(basename $f .txt)_k$K.txt; done
    grep -h "ERROR SUMMARY\|RACECHECK SUMMARY" $O/san_${T}_rank*_k$K.txt | sort | uniq -c
  done
done
