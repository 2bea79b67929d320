# extra parity cases: K9 cut at ranks 48 / 8 / 1, A.3 heavy rows at N = 1, TTV0 small tensors
timeout 1500 python -m pytest tests/test_gpu_mttkrp_slice.py tests/test_gpu_spmm_heavy.py tests/test_gpu_serial.py -q -rf 2>&1 | grep -E "FAILED|^E |passed|failed" | head -20
echo done
