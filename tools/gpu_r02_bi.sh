# K10 warp-per-row SDDMM: next-batch L1 prefetch of D rows (SPX_SDDMM_ROW_PF)
python -c "from paper_2001_00532_b200 import build as b; b.build_variant('srpf', 'spx_sddmm.cu', ['-DSPX_SDDMM_ROW_PF=1'])"
SPX_LIB=tools/variants/libspx_srpf.so timeout 900 python -m pytest tests/test_gpu_edge.py tests/test_gpu_parity.py -q -x -k "sddmm or K10" 2>&1 | tail -1
for rep in 1 2; do for v in prod srpf; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 3 --only K10 --no-parity 2>&1 | grep '"ms"' | cut -c1-90; done; done
echo done
