cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_solver.py -x -q 2>&1 | tail -2
for v in "4 1 0" "3 1 0" "4 0 0" "3 0 0" "4 1 1" "3 1 1"; do python tools/spmv_probe.py $v 20; done 2>&1 | grep GBs
for var in 0 2 4; do echo "7pt var $var"; AMG_LANE_VAR=$var PROBE_7PT=256 python tools/spmv_probe.py 3 1 1 20 | grep GBs; done
python tools/solve_profile.py 5 256 > gpurun_out/prof5.txt 2>&1; head -30 gpurun_out/prof5.txt
