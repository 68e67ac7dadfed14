# round-2 closing check on a fresh box: smoke, the whole GPU suite, the default bench line,
# and a short reference-arm run (3 timed oracle iterations at 256^3)
cd $GRAFT_REPO_ROOT
TAG=${1:-r02f}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
python __graft_entry__.py --smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/${TAG}_smoke.log
python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc $?"
tail -n 1 gpurun_out/${TAG}_bench.log > gpurun_out/${TAG}_bench.json; tail -c 600 gpurun_out/${TAG}_bench.json
timeout 3000 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_ref.log 2>&1; echo "ref rc $?"
tail -n 1 gpurun_out/${TAG}_ref.log
