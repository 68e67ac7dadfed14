# round evidence: full bench line, ncu launch list of the timed region, ncu --set full of the
# dominant solve kernel and of the cfg-2 SpMV kernel (CSV exported on the box)
cd $GRAFT_REPO_ROOT
TAG=${1:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
python bench.py > gpurun_out/${TAG}_bench.log 2>&1 || { tail -20 gpurun_out/${TAG}_bench.log; exit 1; }
tail -1 gpurun_out/${TAG}_bench.log
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-spmv > gpurun_out/${TAG}_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-spmv > /tmp/ncu_l.log 2>&1
tail -2 /tmp/ncu_l.log
rm -f /tmp/top.ncu-rep /tmp/spmv.ncu-rep
ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_bsr_sellr<\(int\)4.*double, float.*LEpiSpmv<double>" -c 1 -o /tmp/top python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-spmv > /tmp/ncu_top.log 2>&1
tail -2 /tmp/ncu_top.log
ncu -i /tmp/top.ncu-rep --page details --csv > gpurun_out/${TAG}_ncu_top_details.csv
ncu -i /tmp/top.ncu-rep --page raw --csv > gpurun_out/${TAG}_ncu_top_raw.csv
rm -f /tmp/smooth.ncu-rep
ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_bsr_sellr<\(int\)3, \(int\)3, \(int\)2, float, float, \(bool\)1, amgb::LEpiSmooth<float, float>>" -c 1 -o /tmp/smooth python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-spmv > /tmp/ncu_smooth.log 2>&1
tail -2 /tmp/ncu_smooth.log
ncu -i /tmp/smooth.ncu-rep --page details --csv > gpurun_out/${TAG}_ncu_smooth_details.csv
ncu -i /tmp/smooth.ncu-rep --page raw --csv > gpurun_out/${TAG}_ncu_smooth_raw.csv
python tools/spmv_probe.py 4 1 0 5 > gpurun_out/${TAG}_spmv_plain.log 2>&1 || exit 1
ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_bsr_sellr" -s 2 -c 1 -o /tmp/spmv python tools/spmv_probe.py 4 1 0 5 > /tmp/ncu_spmv.log 2>&1
tail -2 /tmp/ncu_spmv.log
ncu -i /tmp/spmv.ncu-rep --page details --csv > gpurun_out/${TAG}_ncu_spmv_details.csv
ncu -i /tmp/spmv.ncu-rep --page raw --csv > gpurun_out/${TAG}_ncu_spmv_raw.csv
ls -la gpurun_out | grep $TAG
