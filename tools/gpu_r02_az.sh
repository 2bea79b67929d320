# A.3 heavy-row kernel occupancy vs B rows in flight (SPX_SPMM_HEAVY_MINB / SPX_SPMM_HEAVY_UDIV)
python -c "
from paper_2001_00532_b200 import build as b
b.build_variant('hm2u2', 'spx_spmm.cu', ['-DSPX_SPMM_HEAVY_MINB=2', '-DSPX_SPMM_HEAVY_UDIV=2'])
b.build_variant('hm2u4', 'spx_spmm.cu', ['-DSPX_SPMM_HEAVY_MINB=2', '-DSPX_SPMM_HEAVY_UDIV=4'])
b.build_variant('hm1u2', 'spx_spmm.cu', ['-DSPX_SPMM_HEAVY_UDIV=2'])"
SPX_LIB=tools/variants/libspx_hm2u4.so timeout 900 python -m pytest tests/test_gpu_spmm_heavy.py -q -x 2>&1 | tail -1
for rep in 1 2; do for v in prod hm2u2 hm2u4 hm1u2; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 2 --only A3 --no-parity 2>&1 | grep '"ms"' | cut -c1-100; done; done
echo done
