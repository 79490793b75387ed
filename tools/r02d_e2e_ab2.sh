# A/B of the e2e leg: per-rank copies vs one 2-D copy per range, pipeline depth, H2D streams.
# (The --e2e-copy 2d option was removed after this A/B: no gain; see profiles/r02/ab/README.md.)
set -u
mkdir -p gpurun_out/r02d/e2e2
for cp in 2d per-rank; do
for ch in 2 4 8 16; do
for ns in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-staged --no-cpu-baseline --e2e-copy $cp --e2e-chunks $ch --e2e-h2d-streams $ns --e2e-steps 8 \
  > gpurun_out/r02d/e2e2/${cp}_c${ch}_s${ns}.json 2> gpurun_out/r02d/e2e2/${cp}_c${ch}_s${ns}.err
python -c "import json; d=json.loads(open('gpurun_out/r02d/e2e2/${cp}_c${ch}_s${ns}.json').read().strip().splitlines()[-1]); print('$cp chunks $ch streams $ns', round(d['e2e']['ms_per_step'],3), 'ms', d['e2e']['sampled_result_equals_first_exchange'])" || tail -5 gpurun_out/r02d/e2e2/${cp}_c${ch}_s${ns}.err
done
done
done
