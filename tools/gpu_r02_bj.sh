# K1 thread-per-row SpMV (A.7 as written): L2 prefetch of the thread's crd / vals lines ahead (SPX_SPMV_ROW_PF steps)
python -c "from paper_2001_00532_b200 import build as b; b.build_variant('rpf4', 'spx_spmv.cu', ['-DSPX_SPMV_ROW_PF=4']); b.build_variant('rpf16', 'spx_spmv.cu', ['-DSPX_SPMV_ROW_PF=16'])"
SPX_LIB=tools/variants/libspx_rpf4.so timeout 900 python -m pytest tests/test_gpu_edge.py -q -x -k "spmv_row" 2>&1 | tail -1
for rep in 1 2; do for v in prod rpf4 rpf16; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 5 --only A7 --no-parity 2>&1 | grep '"ms"' | cut -c1-90; done; done
echo done
