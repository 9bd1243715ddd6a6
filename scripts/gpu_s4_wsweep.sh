# Walk staging variants (WAMGPU_WALK_VARIANT: 0 = (D16,NS1) default, 1 = (8,2), 2 = (16,2), 3 = (32,1), 4 = (4,2))
# with warp-private staging: cfg2 expand ms per run.
mkdir -p gpurun_out/s4s
for v in 0 1 2 3 4 0; do
WAMGPU_WALK_VARIANT=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s4s/v$v.json 2> gpurun_out/s4s/v$v.err
python -c "
import json; d=json.load(open('gpurun_out/s4s/v$v.json')); print('variant $v', round(d['value'],1), 'expand', round(d['kernels']['per_step_ms']['expand'],2), d['final_objective'], d['clocks']['sm_mhz'])"
done
