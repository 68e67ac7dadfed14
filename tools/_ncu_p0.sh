# ncu --set full of the level-0 prolongation (interleaved copy, 8-byte vectors) and smoother
cd $GRAFT_REPO_ROOT
rm -f /tmp/p0.ncu-rep /tmp/sm.ncu-rep
ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_bsr_sellr<\(int\)3, \(int\)3, \(int\)2, float, float, \(bool\)1, amgb::LEpiSpmv<float>>" -s 1 -c 1 -o /tmp/p0 python tools/solve_profile.py 5 256 > /tmp/ncu_p0.log 2>&1
tail -1 /tmp/ncu_p0.log
ncu -i /tmp/p0.ncu-rep --page details --csv > gpurun_out/p0_details.csv
ncu -i /tmp/p0.ncu-rep --page raw --csv > gpurun_out/p0_raw.csv
