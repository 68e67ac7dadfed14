cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python tools/solve_profile.py 5 256 idrs 2>&1 | head -20
python tools/solve_profile.py 5 256 2>&1 | grep -E "solve|schur"
python tools/ladder.py 128 2>&1 | tail -12
