cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_spmv.py -q -x -k "interleaved or lane_variants or sliced or plan" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_solver.py -q -x -k "interleaved or forced" 2>&1 | tail -2
AMG_SELLR=0 timeout 600 python tools/solve_profile.py 5 256 > gpurun_out/sp_sellr0.txt 2>&1
timeout 600 python tools/solve_profile.py 5 256 > gpurun_out/sp_sellr1.txt 2>&1
for a in "0 0" "0 1"; do timeout 600 python tools/level_probe.py 256 $a 10 2>&1 | grep -v Warn | grep "level\|None\|var    2\|var    4\|var    7\|8w"; done
