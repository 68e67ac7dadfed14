cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_dist.py -x -q 2>&1 | tail -2
python tools/solve_profile.py 5 256 > gpurun_out/prof5.txt 2>&1; head -5 gpurun_out/prof5.txt | tail -1
grep -E "^(mdot|cgs)" gpurun_out/prof5.txt | sort -t_ -k3 | awk '{printf "%s:%s ", $1, $6}'; echo
AMG_CGS_WIDE=9 python tools/solve_profile.py 5 256 > gpurun_out/prof5w9.txt 2>&1; head -5 gpurun_out/prof5w9.txt | tail -1
grep -E "^(mdot|cgs)" gpurun_out/prof5w9.txt | sort -t_ -k3 | awk '{printf "%s:%s ", $1, $6}'; echo
