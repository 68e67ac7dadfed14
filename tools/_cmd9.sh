for tr in 64 128; do for ns in 3 4; do echo "tr $tr ns $ns"; AMG_TMA_NS=$ns AMG_TMA_ROWS_TR=$tr PROBE_7PT=256 python tools/spmv_probe.py 3 1 1 20 2>&1 | tail -1; done; done
python -m pytest tests/test_gpu_spmv.py tests/test_gpu_solver.py -x -q 2>&1 | tail -2
python bench.py --cfg 5 --steps 2 --warmup 1 --no-cpu-baseline --no-spmv 2>&1 | tail -1
