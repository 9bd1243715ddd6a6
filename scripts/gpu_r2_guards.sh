mkdir -p gpurun_out/guards
timeout 1500 python -m pytest tests/test_gpu_guards.py -x -q > gpurun_out/guards/pytest.log 2>&1; echo "rc=$?"; tail -n 30 gpurun_out/guards/pytest.log
