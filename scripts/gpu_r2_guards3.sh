
export WAMGPU_GUARD=1 WAMGPU_FWD_BAND_MB=0.004 WAMGPU_SYNC_CHECK=1
echo "== only small3d am tma"; timeout 120 python scripts/guard_case.py small3d,0,am,1 2>&1 | tail -n 4 | cut -c1-300
echo "== small3d am stored"; timeout 120 python scripts/guard_case.py small3d,0,am,0 2>&1 | tail -n 4 | cut -c1-300
echo "== tiny3d24 tma then small3d am tma"; timeout 120 python scripts/guard_case.py tiny3d24,3,,1 small3d,0,am,1 2>&1 | tail -n 4 | cut -c1-300
echo "== small3d h3 then small3d am tma"; timeout 120 python scripts/guard_case.py small3d,3,,0 small3d,0,am,1 2>&1 | tail -n 4 | cut -c1-300
unset WAMGPU_FWD_BAND_MB
echo "== no band: small3d h3 then small3d am tma"; timeout 120 python scripts/guard_case.py small3d,3,,0 small3d,0,am,1 2>&1 | tail -n 4 | cut -c1-300
