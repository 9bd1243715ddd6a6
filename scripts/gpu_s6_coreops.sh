# session 6: the standalone predicted_means / i_divergence ops, then the full suite and smoke with the rebuilt library
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_core_ops.py -m gpu -q > gpurun_out/s6_coreops.log 2>&1; tail -15 gpurun_out/s6_coreops.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s6_pytest2.log 2>&1; tail -3 gpurun_out/s6_pytest2.log
timeout 300 python __graft_entry__.py > gpurun_out/s6_smoke2.log 2>&1; tail -1 gpurun_out/s6_smoke2.log
timeout 900 python bench.py > gpurun_out/s6_cfg4_2.log 2>&1; tail -1 gpurun_out/s6_cfg4_2.log | cut -c1-300
