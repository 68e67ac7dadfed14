cd $GRAFT_REPO_ROOT
rm -f /tmp/s.ncu-rep
ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_bsr_sellr.*LEpiSmooth<float, float>" -s 1 -c 1 -o /tmp/s python tools/solve_profile.py 5 256 > /tmp/ncu_s.log 2>&1
tail -2 /tmp/ncu_s.log
ncu -i /tmp/s.ncu-rep --page details --csv > gpurun_out/sellr_smooth_details.csv
ncu -i /tmp/s.ncu-rep --page raw --csv > gpurun_out/sellr_smooth_raw.csv
ncu -i /tmp/s.ncu-rep --page source --csv --print-source sass > gpurun_out/sellr_smooth_sass.csv 2>/dev/null
