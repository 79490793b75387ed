# compute-sanitizer over a slice of the single-process fuzz (exchange, BSP and
# EASGD cases; every flavour appears) -- memcheck, racecheck, synccheck, initcheck.
set -u
O=gpurun_out/r02d/san_fuzz
mkdir -p $O
export TM_FUZZ_CASES=48 TM_FUZZ_BSP_CASES=12 TM_FUZZ_EASGD_CASES=12
for T in memcheck racecheck synccheck initcheck; do
  timeout 2400 compute-sanitizer --tool $T --error-exitcode 9 --target-processes all \
    python -m pytest tests/test_gpu_fuzz.py -q -p no:cacheprovider -x > $O/san_fuzz_$T.txt 2>&1
  echo "$T rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' $O/san_fuzz_$T.txt | tail -2 | tr '\n' ' ')"
done
