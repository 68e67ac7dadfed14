cd $GRAFT_REPO_ROOT
TAG=r01d
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-spmv --no-alt --no-other > gpurun_out/${TAG}_plain2.log 2>&1 || exit 1
rm -f /tmp/smooth.ncu-rep
ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_bsr_lane.*LEpiSmooth<float, float>" -c 1 -o /tmp/smooth python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-spmv --no-alt --no-other > /tmp/ncu_smooth.log 2>&1
tail -2 /tmp/ncu_smooth.log
ncu -i /tmp/smooth.ncu-rep --page details --csv > gpurun_out/${TAG}_ncu_smooth_details.csv
ncu -i /tmp/smooth.ncu-rep --page raw --csv > gpurun_out/${TAG}_ncu_smooth_raw.csv
