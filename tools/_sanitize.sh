# compute-sanitizer over the reduced solves (tools/sanitize.py); summaries to gpurun_out/r2/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
out=gpurun_out/r2/sanitizer.txt
: > $out
for tool in memcheck racecheck synccheck initcheck; do
  for c in cfg3 cfg4 cfg5 cg idrs dist2; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize.py $c \
      > gpurun_out/r2/san_${tool}_$c.log 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/r2/san_${tool}_$c.log | tail -1)" >> $out
  done
done
cat $out
