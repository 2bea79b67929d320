# A.3 cut row kernel: occupancy vs B rows in flight (SPX_SPMM_CUT_MINB / SPX_SPMM_CUT_UDIV)
python -c "
from paper_2001_00532_b200 import build as b
b.build_variant('cm3u2', 'spx_spmm.cu', ['-DSPX_SPMM_CUT_MINB=3', '-DSPX_SPMM_CUT_UDIV=2'])
b.build_variant('cm3u4', 'spx_spmm.cu', ['-DSPX_SPMM_CUT_MINB=3', '-DSPX_SPMM_CUT_UDIV=4'])
b.build_variant('cm4u2', 'spx_spmm.cu', ['-DSPX_SPMM_CUT_MINB=4', '-DSPX_SPMM_CUT_UDIV=2'])"
SPX_LIB=tools/variants/libspx_cm3u2.so timeout 900 python -m pytest tests/test_gpu_spmm_heavy.py -q -x 2>&1 | tail -1
for rep in 1 2; do for v in cm3u2 cm3u4 cm4u2; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 2 --only A3 --no-parity 2>&1 | grep '"ms"' | cut -c1-100; done; done
echo done
