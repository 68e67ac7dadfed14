cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in "4 1 0" "3 1 0" "4 0 0" "3 0 0" "4 1 1" "3 1 1"; do python tools/spmv_probe.py $v 20; done 2>&1 | grep GBs
python tools/solve_profile.py 5 256 > gpurun_out/prof5.txt 2>&1; head -30 gpurun_out/prof5.txt
