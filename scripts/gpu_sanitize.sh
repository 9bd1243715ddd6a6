# compute-sanitizer, ONE tool per gpurun call (B200_PROFILING.md): the small
# 2D/3D parity cases, the sharded 3D rank groups and the fused all-reduce
# protocol emulation.  Usage: bash scripts/gpu_sanitize.sh memcheck|racecheck|synccheck|initcheck
tool=$1
sel="tests/test_gpu_parity.py::test_wam_parity_tree_bit_exact[tiny] tests/test_gpu_parity.py::test_am_parity[tiny] \
tests/test_gpu_parity.py::test_root_only_iterations_use_phi_a tests/test_gpu_parity3d.py::test_wam3d_parity_tree_bit_exact[tiny3d] \
tests/test_gpu_parity3d.py::test_am3d_parity[tiny3d] tests/test_gpu_parity3d.py::test_wam3d_separable_haar_parity[tiny3d16] \
tests/test_gpu_fused_ar.py::test_fused_allreduce_protocol[257-2] tests/test_gpu_fused_ar.py::test_fused_allreduce_protocol[4103-4] \
tests/test_gpu_fused_ar.py::test_fused_back_producer_shards tests/test_gpu_parity3d.py::test_on_the_fly_tma_forward[tiny3d24]"
extra=""
[ "$tool" = "memcheck" ] && extra="--leak-check no"
[ "$tool" = "initcheck" ] && extra="--track-unused-memory no"
python -m pytest $sel -x -q > gpurun_out/san_plain.log 2>&1; echo plain rc=$?
timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 --target-processes all \
    python -m pytest $sel -x -q -p no:cacheprovider > gpurun_out/san_$tool.log 2>&1
echo sanitizer $tool rc=$?
tail -15 gpurun_out/san_$tool.log
