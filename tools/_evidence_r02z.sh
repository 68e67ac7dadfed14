# final round-2 evidence (run r02z): bench line, ncu launch list of one timed step, the ladder,
# per-kernel solve profiles of cfg 3 and cfg 5
cd $GRAFT_REPO_ROOT
TAG=${1:-r02z}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
python bench.py > gpurun_out/${TAG}_bench.log 2>&1 || { tail -20 gpurun_out/${TAG}_bench.log; exit 1; }
tail -c 400 gpurun_out/${TAG}_bench.log
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-spmv \
  --no-alt --no-other > /tmp/ncu_l.log 2>&1
tail -1 /tmp/ncu_l.log
python tools/solve_profile.py 5 256 > gpurun_out/${TAG}_solve_profile_cfg5.txt 2>&1
python tools/solve_profile.py 3 64 > gpurun_out/${TAG}_solve_profile_cfg3.txt 2>&1
python tools/solve_profile.py 1 16 > gpurun_out/${TAG}_solve_profile_cfg1.txt 2>&1
python tools/ladder.py 128 256 > gpurun_out/${TAG}_ladder.txt 2>&1
tail -12 gpurun_out/${TAG}_ladder.txt
