# A.3 heavy-row kernel at 2 CTAs/SM, 8 rows in flight (the new default): tests + cfg2
timeout 1500 python -m pytest tests/test_gpu_spmm_heavy.py tests/test_gpu_edge.py tests/test_gpu_parity.py -q -x -k "spmm or A3 or heavy" 2>&1 | tail -1
timeout 600 python tools/bench_configs.py --cfg 2 --only A3 2>&1 | grep '"ms"' | cut -c1-200
