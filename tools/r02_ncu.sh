#!/usr/bin/env bash
# Round-2 ncu evidence: the bench's launch list and one --set full capture of
# each round-2 kernel (reports under gpurun_out/ncu_r02, CSV pages copied to profiles/r02/ncu).
set -u
O=gpurun_out/ncu_r02
mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > $O/bench_under_ncu.log 2>&1
echo "launch list rc=$?"
cap() {  # name kernel-regex skip env... -- one_call args
  local name=$1 kre=$2 skip=$3; shift 3
  env "$@" timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$kre" -s $skip -c 1 \
    -o $O/$name -f python tools/one_call.py ${CALL} 3 > $O/$name.log 2>&1
  echo "$name rc=$?"
  ncu -i $O/$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>/dev/null
  ncu -i $O/$name.ncu-rep --page details --csv > $O/${name}_details.csv 2>/dev/null
  rm -f $O/$name.ncu-rep  # the CSV pages travel back; the report is too large for gpurun_out
}
CALL=exchange-direct cap direct_tma tm_direct_tma_kernel 1 X=1
CALL=bsp-staged-mom cap staged_bsp_mom tm_exchange_tma_kernel 1 X=1
CALL=exchange-staged cap staged_tmaws tm_exchange_tmaws_kernel 1 TM_STAGED_KERNEL=tmaws
CALL=exchange-staged cap oneshot_small tm_exchange_oneshot_kernel 1 TM_ONE_CALL_P=131072
CALL=exchange-staged cap oneshot_k2_2m tm_exchange_oneshot_kernel 1 TM_ONE_CALL_P=2097152 TM_ONE_CALL_K=2
