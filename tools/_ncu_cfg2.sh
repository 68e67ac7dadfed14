set -e
cd $GRAFT_REPO_ROOT
export AMG_TMA_GROUP=1
python tools/spmv_probe.py 4 1 0 5 > gpurun_out/plain_g.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bsr -s 2 -c 1 -o /tmp/prof_g python tools/spmv_probe.py 4 1 0 5 > /tmp/ncu_g.log 2>&1
ncu -i /tmp/prof_g.ncu-rep --page details --csv > gpurun_out/ncu_cfg2_group_details.csv
ncu -i /tmp/prof_g.ncu-rep --page raw --csv > gpurun_out/ncu_cfg2_group_raw.csv
ncu -i /tmp/prof_g.ncu-rep --page source --csv > gpurun_out/ncu_cfg2_group_source.csv || true
unset AMG_TMA_GROUP
python tools/spmv_probe.py 4 1 0 5 > gpurun_out/plain_s.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bsr -s 2 -c 1 -o /tmp/prof_s python tools/spmv_probe.py 4 1 0 5 > /tmp/ncu_s.log 2>&1
ncu -i /tmp/prof_s.ncu-rep --page details --csv > gpurun_out/ncu_cfg2_seg_details.csv
ncu -i /tmp/prof_s.ncu-rep --page raw --csv > gpurun_out/ncu_cfg2_seg_raw.csv
ncu -i /tmp/prof_s.ncu-rep --page source --csv > gpurun_out/ncu_cfg2_seg_source.csv || true
ls -la gpurun_out
