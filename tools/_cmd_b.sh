cd $GRAFT_REPO_ROOT
python tools/solve_profile.py 4 128 2>&1 | head -12
python tools/solve_profile.py 3 64 2>&1 | head -14
python tools/solve_profile.py 1 16 2>&1 | head -10
