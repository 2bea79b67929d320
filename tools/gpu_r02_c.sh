# IR path (generic lowering honouring the schedule) + MTTKRP quarter kernel.
timeout 1200 python -m pytest tests/test_gpu_irpath.py -q -x 2>&1 | tail -25
timeout 900 python -m pytest tests/test_gpu_mttkrp_quarter.py tests/test_gpu_edge.py tests/test_gpu_generic.py -q -x 2>&1 | tail -5
timeout 600 python tools/bench_configs.py --cfg 4 --only A6 2>&1 | tail -1 | cut -c1-300
for w in 128 512 1024; do timeout 300 python tools/bench_configs.py --cfg 4 --only A6 --no-parity --params NNZ_PER_TB=$((w*8)),NNZ_PER_WARP=$w 2>&1 | tail -1 | cut -c1-200; done
