# warp-per-row SpMV (A.8 / A.1): predicated tail steps of PT x 32 positions (SPX_SPMV_WARP_PTAIL = 2 / 4 / 8; 0 = one at a time)
python -c "
from paper_2001_00532_b200 import build as b
for t in (0, 4, 8): b.build_variant(f'pt{t}', 'spx_spmv.cu', [f'-DSPX_SPMV_WARP_PTAIL={t}'])"
timeout 900 python -m pytest tests/test_gpu_edge.py tests/test_gpu_parity.py -q -x -k "spmv or A8 or A1" 2>&1 | tail -1
for rep in 1 2; do for v in prod pt0 pt4 pt8; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 5,1 --only A8,A1 --no-parity 2>&1 | grep '"ms"' | cut -c1-100; done; done
echo done
