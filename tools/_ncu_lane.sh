cd $GRAFT_REPO_ROOT
python tools/solve_profile.py 4 128 > gpurun_out/plain4.log 2>&1 || exit 1
rm -f /tmp/prof_res.ncu-rep; ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:LEpiResidual<float>" -c 1 -o /tmp/prof_res python tools/solve_profile.py 4 128 > /tmp/ncu_res.log 2>&1
tail -3 /tmp/ncu_res.log
ncu -i /tmp/prof_res.ncu-rep --page details --csv > gpurun_out/ncu_lane_res_details.csv
ncu -i /tmp/prof_res.ncu-rep --page raw --csv > gpurun_out/ncu_lane_res_raw.csv
ncu -i /tmp/prof_res.ncu-rep --page source --csv > gpurun_out/ncu_lane_res_source.csv
ls -la gpurun_out/*.csv
