# K9 cut at rank 32 fp32 on the quarter kernel with deterministic head/tail slots + ordered fold
timeout 1500 python -m pytest tests/test_gpu_mttkrp_slice.py tests/test_gpu_mttkrp_quarter.py tests/test_gpu_parity.py tests/test_gpu_acceptance.py tests/test_gpu_fullscale.py -q -x -rf -k "mttkrp or MTTKRP or A5 or A6 or K9 or slice or cfg4" 2>&1 | grep -E "FAILED|^E |passed|failed" | head
for rep in 1 2; do timeout 600 python tools/bench_configs.py --cfg 4 --only A5,MTTKRP0,A6 2>&1 | grep '"ms"' | cut -c1-230; done
echo done
