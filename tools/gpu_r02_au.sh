# K9 cut at rank 32 fp32 on the quarter kernel (UNIT mode: units in one slice, quarter fold, plain stores)
timeout 1500 python -m pytest tests/test_gpu_mttkrp_slice.py tests/test_gpu_mttkrp_quarter.py tests/test_gpu_parity.py tests/test_gpu_acceptance.py tests/test_gpu_serial.py -q -x -rf 2>&1 | grep -E "FAILED|^E |passed|failed" | head
for rep in 1 2; do timeout 600 python tools/bench_configs.py --cfg 4 --only A5,MTTKRP0,A6 2>&1 | grep '"ms"' | cut -c1-200; done
echo done
