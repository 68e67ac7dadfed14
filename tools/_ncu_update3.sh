# ncu --set full of the update pass's three-vectors-per-warp kernel at its new launch shape
# (three blocks per SM, 80 registers; run r02o) -- the 8th launch of the solve (k = 24 region)
cd $GRAFT_REPO_ROOT
rm -f /tmp/u3.ncu-rep
ncu -f --set full --clock-control none --kernel-name-base demangled -k "regex:k_cgs_wide<\(int\)3, \(int\)3" -s 7 -c 1 -o /tmp/u3 python tools/solve_profile.py 5 256 > /tmp/ncu_u3.log 2>&1
tail -1 /tmp/ncu_u3.log
ncu -i /tmp/u3.ncu-rep --page details --csv > gpurun_out/r02o_ncu_update3_details.csv
grep -E "DRAM Throughput|Registers Per Thread|Theoretical Occupancy|Achieved Occupancy|Duration|No Eligible|Grid Size|Local" gpurun_out/r02o_ncu_update3_details.csv | cut -d, -f12- | head -20
