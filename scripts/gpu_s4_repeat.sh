# Run-to-run spread of the default bench line on one box (cfg2, 4 runs, no CPU baseline).
mkdir -p gpurun_out/rep
for i in 1 2 3 4; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/rep/cfg2_$i.json 2> gpurun_out/rep/cfg2_$i.err
python -c "
import json; d=json.load(open('gpurun_out/rep/cfg2_$i.json')); print('run $i', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'ms', round(d['ms_per_step'],2), 'fwd', round(d['kernels']['fwd_avg_ms'],4), 'back', round(d['kernels']['back_avg_ms'],4), 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], 'expand', round(d['kernels']['per_step_ms']['expand'],2), d['final_objective'])"
done
