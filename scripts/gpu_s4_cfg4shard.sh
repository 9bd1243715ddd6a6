# cfg4 detached shard at R=8 (views only) with the session-4 build.
mkdir -p gpurun_out/c4
timeout 1500 python bench.py --config cfg4 --shard 8 --view-groups 8 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c4/cfg4_R8_v8.json 2> gpurun_out/c4/cfg4_R8_v8.err; echo "rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/c4/cfg4_R8_v8.json')); print(d['ms_per_step'], d['shard']['projected_ms_per_step'], {k: round(v,1) for k,v in d['kernels']['per_step_ms'].items()}, d['clocks'])"
