# A/B of the L2 eviction-priority hint on the direct TMA kernel (TM_L2_HINT:
# 0 none, 1 evict_first loads, 2 evict_first stores, 3 both), bench headline
# config, two interleaved passes.
set -u
mkdir -p gpurun_out/r02d/l2hint
for pass in 1 2; do
for h in 0 1 2 3; do
TM_L2_HINT=$h timeout 300 python bench.py --steps 100 --warmup 10 --no-e2e --no-staged --no-cpu-baseline \
  > gpurun_out/r02d/l2hint/h${h}_p${pass}.json 2> gpurun_out/r02d/l2hint/h${h}_p${pass}.err
python -c "import json,sys; d=json.loads(open('gpurun_out/r02d/l2hint/h${h}_p${pass}.json').read().strip().splitlines()[-1]); print('hint $h pass $pass', round(d['ms_per_step']*1e3,1), 'us', d['parity']['parity'], d['ms_per_step_loops']['min'])"
done
done
