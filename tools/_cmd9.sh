for tr in 64 128 256; do for ns in 2 3; do echo "tr $tr ns $ns"; AMG_TMA_ROWS_TR=$tr AMG_TMA_NS=$ns PROBE_7PT=256 python tools/spmv_probe.py 3 1 1 20 2>&1 | tail -1; done; done
