set -x
python -m pytest tests/test_gpu_wamh.py tests/test_gpu_cpp_shim.py -x -q -s > gpurun_out/s2_wamh.log 2>&1; echo wamh rc=$?
python -m pytest tests/test_gpu_parity_big.py -x -q -s > gpurun_out/s2_big.log 2>&1; echo big rc=$?
python -m pytest tests -m gpu -x -q > gpurun_out/s2_pytest_gpu.log 2>&1; echo all rc=$?
tail -3 gpurun_out/s2_*.log
