# A.3 heavy-row kernel: CTA width (SPX_SPMM_HEAVY_WARPS, full occupancy at 64 registers) x cut
python -c "
from paper_2001_00532_b200 import build as b
b.build_variant('h4', 'spx_spmm.cu', ['-DSPX_SPMM_HEAVY_WARPS=4'])
b.build_variant('h8', 'spx_spmm.cu', ['-DSPX_SPMM_HEAVY_WARPS=8'])
b.build_variant('h8c256', 'spx_spmm.cu', ['-DSPX_SPMM_HEAVY_WARPS=8', '-DSPX_SPMM_CUT_MIN=256', '-DSPX_SPMM_CUT_DIV=262144'])
b.build_variant('h4c1k', 'spx_spmm.cu', ['-DSPX_SPMM_HEAVY_WARPS=4', '-DSPX_SPMM_CUT_MIN=1024', '-DSPX_SPMM_CUT_DIV=65536'])"
SPX_LIB=tools/variants/libspx_h4.so timeout 900 python -m pytest tests/test_gpu_spmm_heavy.py -q -x 2>&1 | tail -1
for v in prod h4 h8 h8c256 h4c1k; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 2 --only A3 --no-parity 2>&1 | grep '"ms"' | cut -c1-110; done
echo done
