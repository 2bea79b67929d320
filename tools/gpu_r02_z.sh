# serial schedules on the nnz-split kernels: determinism + parity, then cfg2 A10/A11 timings
timeout 1800 python -m pytest tests/test_gpu_serial.py tests/test_gpu_parity.py tests/test_gpu_acceptance.py tests/test_gpu_irpath.py tests/test_gpu_edge.py -q -x 2>&1 | tail -2
timeout 900 python tools/bench_configs.py --cfg 2 --only A10,A11 2>&1 | grep '"ms"' | cut -c1-160
echo done
