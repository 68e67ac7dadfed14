# ncu --set full of the pass-1 multi-dot on the fp32 shadow basis (gmres_ortho = 2) vs the fp64
# one (default), wide kernel at k ~ 25 (cfg 5)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for v in 2 1; do
  rm -f /tmp/md$v.ncu-rep
  ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:k_cgs_wide<\(int\)4, \(int\)0" -s 4 -c 1 -o /tmp/md$v \
    python tools/solve_profile.py 5 256 gmres_ortho=$v > /tmp/ncu_md$v.log 2>&1
  tail -1 /tmp/ncu_md$v.log
  ncu -i /tmp/md$v.ncu-rep --page details --csv > gpurun_out/r2/ncu_mdot_o$v.csv
done
