# occupancy sweeps: TTV K7 (SPX_TTV_MINB), warp-per-row SpMV A.8 (SPX_SPMV_WARP_MINB / _STEPS)
python -c "
from paper_2001_00532_b200 import build as b
b.build_variant('t5', 'spx_csf.cu', ['-DSPX_TTV_MINB=5'])
b.build_variant('t8', 'spx_csf.cu', ['-DSPX_TTV_MINB=8'])
b.build_variant('w3', 'spx_spmv.cu', ['-DSPX_SPMV_WARP_MINB=3'])
b.build_variant('w4s4', 'spx_spmv.cu', ['-DSPX_SPMV_WARP_MINB=4', '-DSPX_SPMV_WARP_STEPS=4'])"
for rep in 1 2; do
for v in prod t5 t8; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 4 --only K7 --no-parity 2>&1 | grep '"ms"' | cut -c1-90; done
for v in prod w3 w4s4; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 5 --only A8 --no-parity 2>&1 | grep '"ms"' | cut -c1-90; done
done
echo done
