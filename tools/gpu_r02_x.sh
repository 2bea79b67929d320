# SpMV A.1 / unscheduled on the warp-per-row kernel: parity suites + cfg5 timings
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_acceptance.py tests/test_gpu_irpath.py tests/test_gpu_generic.py tests/test_gpu_fullscale.py -q -x 2>&1 | tail -2
timeout 900 python tools/bench_configs.py --cfg 5 --only A1,SPMV0,A7 2>&1 | grep '"ms"' | cut -c1-200
timeout 900 python tools/bench_configs.py --cfg 1 --only A1,SPMV0,A7 2>&1 | grep '"ms"' | cut -c1-200
echo done
