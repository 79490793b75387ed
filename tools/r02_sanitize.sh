#!/usr/bin/env bash
# compute-sanitizer over every kernel (tests/sanitize_driver.py, a parity run too):
# the default flavours (one-shot for the driver's small sizes) and the
# warp-specialised TMA flavour (incl. the momentum exchange, nvec = 2).
set -u
O=gpurun_out/san_r02
mkdir -p $O
for FL in default tmaws tma; do
  for T in memcheck racecheck synccheck; do
    if [ "$FL" = default ]; then E=""; else E="TM_STAGED_KERNEL=$FL"; fi
    env $E timeout 1500 compute-sanitizer --tool $T --error-exitcode 9 python tests/sanitize_driver.py > $O/san_${FL}_${T}.txt 2>&1
    echo "$FL $T rc=$?"
  done
done
