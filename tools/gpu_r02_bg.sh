# warp-per-row SpMM walk (K5 as written, A.3's cut / heavy kernels): next-batch L1 prefetch of B rows (SPX_SPMM_ROW_PF)
python -c "from paper_2001_00532_b200 import build as b; b.build_variant('rpf', 'spx_spmm.cu', ['-DSPX_SPMM_ROW_PF=1'])"
SPX_LIB=tools/variants/libspx_rpf.so timeout 900 python -m pytest tests/test_gpu_spmm_heavy.py tests/test_gpu_edge.py -q -x -k "spmm" 2>&1 | tail -1
for rep in 1 2; do for v in prod rpf; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 2 --only K5,A3 --no-parity 2>&1 | grep '"ms"' | cut -c1-90; done; done
echo done
