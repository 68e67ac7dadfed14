# round-2 evidence: the bench line, the ncu launch list of one timed step, and ncu --set full
# captures of the dominant kernel and of the kernels VERDICT r01 asked about (CSV on the box)
cd $GRAFT_REPO_ROOT
TAG=${1:-r02a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
python bench.py > gpurun_out/${TAG}_bench.log 2>&1 || { tail -20 gpurun_out/${TAG}_bench.log; exit 1; }
tail -c 600 gpurun_out/${TAG}_bench.log
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-spmv \
  --no-alt --no-other > /tmp/ncu_l.log 2>&1
tail -1 /tmp/ncu_l.log
cap() {  # name regex skip
  rm -f /tmp/$1.ncu-rep
  ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$2" -s $3 -c 1 \
    -o /tmp/$1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-spmv --no-alt --no-other > /tmp/ncu_$1.log 2>&1
  tail -1 /tmp/ncu_$1.log
  ncu -i /tmp/$1.ncu-rep --page details --csv > gpurun_out/${TAG}_ncu_$1_details.csv
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/${TAG}_ncu_$1_raw.csv
}
cap top 'k_bsr_sellr<\(int\)4.*double, float.*LEpiSpmv<double>' 0
cap smooth 'k_bsr_sellr<\(int\)3, \(int\)3, \(int\)2, float, float, \(bool\)1, amgb::LEpiSmooth<float, float>>' 0
cap resid 'k_bsr_sellr<\(int\)3, \(int\)3, \(int\)2, float, float, \(bool\)1, amgb::LEpiResidual<float>>' 0
cap p0 'k_bsr_sellr<\(int\)3, \(int\)3, \(int\)2, float, float, \(bool\)1, amgb::LEpiSpmvPre<float>>' 1
cap r0m 'LEpiSpmvM' 0
cap splitm 'k_split4_M' 0
cap schurum 'EpiSchurUM' 0
cap schurp 'LEpiSchurP' 0
cap mdot16 'k_mdot16_wide<\(int\)4>' 2
cap update 'k_cgs_wide<\(int\)4, \(int\)3, double, __half>' 2
cap smoothjoin 'LEpiSmoothJoin' 0
python tools/spmv_probe.py 4 1 0 5 > gpurun_out/${TAG}_spmv_plain.log 2>&1 || exit 1
rm -f /tmp/spmv.ncu-rep
ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_bsr_sellr" -s 2 -c 1 \
  -o /tmp/spmv python tools/spmv_probe.py 4 1 0 5 > /tmp/ncu_spmv.log 2>&1
ncu -i /tmp/spmv.ncu-rep --page details --csv > gpurun_out/${TAG}_ncu_spmv_details.csv
ncu -i /tmp/spmv.ncu-rep --page raw --csv > gpurun_out/${TAG}_ncu_spmv_raw.csv
ls gpurun_out | grep $TAG
