# SpMV A.2 cfg5: smaller per-warp pos slices (SPX_SPMV_WARP_POS) so the carveout leaves more L1 to the x gathers
python -c "
from paper_2001_00532_b200 import build as b
b.build_variant('p32c2', 'spx_spmv.cu', ['-DSPX_SPMV_WARP_POS=32', '-DSPX_SPMV_CARVEOUT=2'])
b.build_variant('p64c0', 'spx_spmv.cu', ['-DSPX_SPMV_WARP_POS=64', '-DSPX_SPMV_CARVEOUT=0'])
b.build_variant('p64c4', 'spx_spmv.cu', ['-DSPX_SPMV_WARP_POS=64', '-DSPX_SPMV_CARVEOUT=4'])"
SPX_LIB=tools/variants/libspx_p32c2.so timeout 900 python -m pytest tests/test_gpu_edge.py -q -x -k "spmv" 2>&1 | tail -1
for rep in 1 2; do for v in prod p64c4 p64c0 p32c2; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 5 --only A2 --no-parity 2>&1 | grep '"ms"' | cut -c1-100; done; done
echo done
