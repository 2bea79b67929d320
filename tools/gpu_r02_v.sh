# K9 slice-split with heavy-slice cut (A.5 / MTTKRP0) vs warp-per-slice (K9): parity + cfg4 timings
timeout 900 python -m pytest tests/test_gpu_mttkrp_slice.py tests/test_gpu_mttkrp_quarter.py tests/test_gpu_edge.py -q -x -k "mttkrp or MTTKRP or slice" 2>&1 | tail -3
timeout 900 python tools/bench_configs.py --cfg 4 --only A5,K9,MTTKRP0,A6 2>&1 | tail -4 | cut -c1-260
echo done
