# SDDMM K6: occupancy (SPX_SDDMM_MINB) vs D rows in flight (SPX_SDDMM_UN)
python -c "
from paper_2001_00532_b200 import build as b
b.build_variant('s3u2', 'spx_sddmm.cu', ['-DSPX_SDDMM_MINB=3'])
b.build_variant('s3u1', 'spx_sddmm.cu', ['-DSPX_SDDMM_MINB=3', '-DSPX_SDDMM_UN=1'])
b.build_variant('s4u1', 'spx_sddmm.cu', ['-DSPX_SDDMM_MINB=4', '-DSPX_SDDMM_UN=1'])"
for rep in 1 2; do for v in prod s3u2 s3u1 s4u1; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 3 --only K6 --no-parity 2>&1 | grep '"ms"' | cut -c1-100; done; done
echo done
