# K9 split path (MTTKRP0 / A.5 at cfg4): unit count (SPX_SLICE_UNITS) with the SPLIT kernel at 2 CTAs/SM, G = 4
python -c "
from paper_2001_00532_b200 import build as b
for u in (4096, 16384, 32768): b.build_variant(f'u{u}', 'spx_csf.cu', [f'-DSPX_SLICE_UNITS={u}'])"
timeout 900 python -m pytest tests/test_gpu_mttkrp_slice.py -q -x 2>&1 | tail -1
for v in prod u4096 u16384 u32768; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 4 --only MTTKRP0,K9 --no-parity 2>&1 | grep '"ms"' | cut -c1-120; done
echo done
