python -c "from paper_2001_00532_b200 import build as b; b.build_variant('cv50', 'spx_spmv.cu', ['-DSPX_SPMV_CARVEOUT=50']); b.build_variant('cvm1', 'spx_spmv.cu', ['-DSPX_SPMV_CARVEOUT=-1'])"
timeout 900 python -m pytest tests/test_gpu_edge.py tests/test_gpu_parity.py tests/test_gpu_ttv_stream.py -q -x -k "spmv or ttv or A2 or A9" 2>&1 | tail -2
timeout 900 python tools/bench_configs.py --cfg 5 --only A2 2>&1 | tail -1 | cut -c1-250
for v in cv50 cvm1; do echo "variant $v"; SPX_LIB=tools/variants/libspx_$v.so timeout 600 python tools/bench_configs.py --cfg 5 --only A2 --no-parity 2>&1 | tail -1 | cut -c1-200; done
timeout 600 python tools/bench_configs.py --cfg 1 --only A2 2>&1 | tail -1 | cut -c1-200
timeout 600 ncu --set full --clock-control none -k regex:spmv_nnz -c 1 -o gpurun_out/l_k3 -f python tools/bench_configs.py --reps 1 --warm 1 --no-parity --cfg 5 --only A2 > gpurun_out/l_k3.log 2>&1
echo done
