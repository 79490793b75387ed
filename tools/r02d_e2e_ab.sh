# A/B of the e2e pipeline depth (bench --e2e-chunks) and H2D stream count.
set -u
mkdir -p gpurun_out/r02d/e2e
for ch in 8 16 32 64; do
for ns in 1 2 4; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-staged --no-cpu-baseline --e2e-chunks $ch --e2e-h2d-streams $ns --e2e-steps 8 \
  > gpurun_out/r02d/e2e/c${ch}_s${ns}.json 2> gpurun_out/r02d/e2e/c${ch}_s${ns}.err
python -c "import json; d=json.loads(open('gpurun_out/r02d/e2e/c${ch}_s${ns}.json').read().strip().splitlines()[-1]); print('chunks $ch streams $ns', round(d['e2e']['ms_per_step'],3), 'ms', d['e2e']['sampled_result_equals_first_exchange'])"
done
done
