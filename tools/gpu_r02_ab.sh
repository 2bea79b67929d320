# A.3 (CPU-tagged SpMM rows) with the heavy-row CTA path: parity + cfg2 timing
timeout 1500 python -m pytest tests/test_gpu_spmm_heavy.py -x -q 2>&1 | grep -E "Error|error|assert|FAIL|passed|failed" | head -20
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_acceptance.py -q -x 2>&1 | tail -2
timeout 900 python tools/bench_configs.py --cfg 2 --only A3,K5 2>&1 | grep '"ms"' | cut -c1-170
echo done
