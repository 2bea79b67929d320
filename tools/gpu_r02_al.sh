# A.1 (CPU-tagged SpMV rows) with the heavy-row CTA path: tests + cfg5 timing
timeout 1500 python -m pytest tests/test_gpu_spmm_heavy.py tests/test_gpu_edge.py tests/test_gpu_parity.py tests/test_gpu_acceptance.py -q -x -rf 2>&1 | grep -E "FAILED|^E |passed|failed" | head
timeout 900 python tools/bench_configs.py --cfg 5 --only A1,A8 2>&1 | grep '"ms"' | cut -c1-200
echo done
