cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_dist.py tests/test_capi.py -x -q 2>&1 | tail -2
for c in "3 64" "1 16" "4 128" "5 256"; do python tools/solve_profile.py $c 2>&1 | grep "solve"; done
for c in "3 64" "1 16"; do AMG_NO_GRAPH=1 python tools/solve_profile.py $c 2>&1 | grep "solve"; done
