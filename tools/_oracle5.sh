cd $GRAFT_REPO_ROOT
free -g
ulimit -v 180000000
( while true; do free -g | awk 'NR==2{print $3}' >> gpurun_out/oracle5_mem.txt; sleep 30; done ) &
MON=$!
timeout 3300 python tools/oracle_reference_runs.py 5 > gpurun_out/oracle5.log 2>&1
echo "rc=$?" >> gpurun_out/oracle5.log
kill $MON
cp tests/golden/oracle_full_size.json gpurun_out/oracle_full_size.json
tail -3 gpurun_out/oracle5.log
