# ncu --set full of the two-pass orthogonalisation's update pass (k = 30, wide kernel) and of
# the level-1 smoother (interleaved copy, 16-byte vectors)
cd $GRAFT_REPO_ROOT
rm -f /tmp/o.ncu-rep /tmp/l1.ncu-rep
ncu -f --set full --clock-control none --kernel-name-base demangled -k "regex:k_cgs_wide<\(int\)4, \(int\)3>" -s 20 -c 1 -o /tmp/o python tools/solve_profile.py 5 256 > /tmp/ncu_o.log 2>&1
tail -1 /tmp/ncu_o.log
ncu -i /tmp/o.ncu-rep --page details --csv > gpurun_out/ortho_details.csv
ncu -f --set full --clock-control none --kernel-name-base demangled -k "regex:k_bsr_sellr<\(int\)3, \(int\)3, \(int\)4, float, float, \(bool\)1, amgb::LEpiSmooth" -c 1 -o /tmp/l1 python tools/solve_profile.py 5 256 > /tmp/ncu_l1.log 2>&1
tail -1 /tmp/ncu_l1.log
ncu -i /tmp/l1.ncu-rep --page details --csv > gpurun_out/l1_smooth_details.csv
