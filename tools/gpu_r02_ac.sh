# A.3 heavy-row path (cut 512, row kernel at 2 CTAs/SM when cutting): tests + cfg2
timeout 900 python -m pytest tests/test_gpu_spmm_heavy.py tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x 2>&1 | tail -1
timeout 600 python tools/bench_configs.py --cfg 2 --only A3,K5 2>&1 | grep '"ms"' | cut -c1-200
echo done
