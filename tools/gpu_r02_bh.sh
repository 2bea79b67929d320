# K5 row walk with the next-batch B-row L1 prefetch (product now); A.3's cut / heavy kernels without it
timeout 1500 python -m pytest tests/test_gpu_spmm_heavy.py tests/test_gpu_edge.py tests/test_gpu_parity.py -q -x -k "spmm or K5 or A3" 2>&1 | tail -1
for rep in 1 2; do timeout 600 python tools/bench_configs.py --cfg 2 --only K5,A3 2>&1 | grep '"ms"' | cut -c1-200; done
echo done
