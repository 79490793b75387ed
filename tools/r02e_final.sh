#!/usr/bin/env bash
# Round-2 final evidence (session e) with the round's last binary: the GPU suite, smoke, the
# N = 1 bench line, the bench's ncu launch list and one --set full capture of the
# headline kernel, and the N > 1 bench lines with 2 and 8 processes concurrent on
# the one GPU under MPS.
set -u
O=gpurun_out/r02e/final
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.txt
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02e/final/bench_n1.json").read().strip().splitlines()[-1])
print("bench", round(d["ms_per_step"] * 1e3, 1), "us frac", round(d["roofline"]["frac"], 4), "parity", d["parity"]["parity"],
      "e2e", round(d["e2e"]["ms_per_step"], 2), "clocks", d["clocks"])
PY
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_under_ncu.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:tm_direct_tma_kernel" -s 1 -c 1 \
  -o $O/direct_tma -f python tools/one_call.py exchange-direct 3 > $O/direct_tma.log 2>&1
echo "ncu full rc=$?"
ncu -i $O/direct_tma.ncu-rep --page raw --csv > $O/direct_tma_raw.csv 2>/dev/null
ncu -i $O/direct_tma.ncu-rep --page details --csv > $O/direct_tma_details.csv 2>/dev/null
rm -f $O/direct_tma.ncu-rep
export CUDA_MPS_PIPE_DIRECTORY=/tmp/tm_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/tm_mps_log
mkdir -p "$CUDA_MPS_PIPE_DIRECTORY" "$CUDA_MPS_LOG_DIRECTORY"
nvidia-cuda-mps-control -d
for N in 8 2; do
TM_PROCS_PER_GPU=$N timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port 2967$N bench.py --gpus $N --steps 50 --warmup 5 > $O/bench_mps_n$N.json 2> $O/bench_mps_n$N.err
echo "mps bench n$N rc=$?"
done
echo quit | nvidia-cuda-mps-control
timeout 300 python tools/sweep.py --only easgd > $O/easgd_sweep.jsonl 2> $O/easgd_sweep.err; echo "easgd sweep rc=$?"
