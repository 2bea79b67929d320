# K9 cut (A.5 / MTTKRP0 at cfg4): smaller leaf ranges (SPX_SLICE_PART_MIN / SPX_SLICE_UNITS) against warp-quantisation
python -c "
from paper_2001_00532_b200 import build as b
b.build_variant('p1k', 'spx_csf.cu', ['-DSPX_SLICE_PART_MIN=1024', '-DSPX_SLICE_UNITS=65536'])
b.build_variant('p2k', 'spx_csf.cu', ['-DSPX_SLICE_PART_MIN=2048', '-DSPX_SLICE_UNITS=32768'])
b.build_variant('p512', 'spx_csf.cu', ['-DSPX_SLICE_PART_MIN=512', '-DSPX_SLICE_UNITS=131072'])"
SPX_LIB=tools/variants/libspx_p1k.so timeout 900 python -m pytest tests/test_gpu_mttkrp_slice.py -q -x 2>&1 | tail -1
for rep in 1 2; do for v in prod p2k p1k p512; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 4 --only A5 --no-parity 2>&1 | grep '"ms"' | cut -c1-100; done; done
echo done
