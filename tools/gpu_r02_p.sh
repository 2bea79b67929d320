python -c "from paper_2001_00532_b200 import build as b; b.build_variant('h0', 'spx_spmv.cu', ['-DSPX_SPMV_HIST=0'])"
timeout 900 python -m pytest tests/test_gpu_edge.py tests/test_gpu_parity.py tests/test_gpu_fullscale.py -q -x -k "spmv or A2 or A9 or cfg5 or cfg1" 2>&1 | tail -2
timeout 900 python tools/bench_configs.py --cfg 5 --only A2 2>&1 | tail -1 | cut -c1-250
SPX_LIB=tools/variants/libspx_h0.so timeout 600 python tools/bench_configs.py --cfg 5 --only A2 --no-parity 2>&1 | tail -1 | cut -c1-200
timeout 900 python tools/bench_configs.py --cfg 5 --only A2 --no-parity 2>&1 | tail -1 | cut -c1-200
timeout 600 python tools/bench_configs.py --cfg 1 --only A2 2>&1 | tail -1 | cut -c1-200
