cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python tools/solve_profile.py 5 256 idrs 2>&1 | head -20
python tools/solve_profile.py 5 256 2>&1 | grep -E "solve|schur"
python tools/ladder.py 128 2>&1 | tail -12
for v in 2 3 4 5; do echo "short var $v"; AMG_LANE_VAR_SHORT=$v python tools/solve_profile.py 5 256 2>&1 | grep -E "solve|smooth_b3_f32xf32 +5956|residual_b3_f32xf32 +5352|spmv_b3_f32xf32 +2928|schur|apply_M_b3_f32xf32 +1006"; done
