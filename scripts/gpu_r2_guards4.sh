export WAMGPU_GUARD=1 WAMGPU_FWD_BAND_MB=0.004
ALL="tiny,0,,0 tiny,0,am,0 small_lug,0,,0 tiny3d,0,,0 tiny3d,0,am,0 tiny3d16,3,,0 small3d,3,,0 tiny3d24,3,,1 small3d,0,am,1"
r() { echo "== $1"; shift; timeout 200 python scripts/guard_case.py "$@" 2>&1 | tail -n 3 | cut -c1-250; echo "rc=${PIPESTATUS[0]}"; }
r "full" $ALL
r "full again" $ALL
CUDA_LAUNCH_BLOCKING=1 r "full blocking" $ALL
r "3D only" tiny3d,0,,0 tiny3d,0,am,0 tiny3d16,3,,0 small3d,3,,0 tiny3d24,3,,1 small3d,0,am,1
r "3D no tiny3d24" tiny3d,0,,0 tiny3d,0,am,0 tiny3d16,3,,0 small3d,3,,0 small3d,0,am,1
r "last three" small3d,3,,0 tiny3d24,3,,1 small3d,0,am,1
r "3D stored only" tiny3d,0,,0 tiny3d,0,am,0 tiny3d16,3,,0 small3d,3,,0 small3d,0,am,0
