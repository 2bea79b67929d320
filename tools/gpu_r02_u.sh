# SDDMM K6 cfg3: D-row prefetch -- SPX_SDDMM_PF=1 (next batch's rows into L2), =2 (next group's rows into L1) -- vs the product
python -c "from paper_2001_00532_b200 import build as b; b.build_variant('spf1', 'spx_sddmm.cu', ['-DSPX_SDDMM_PF=1']); b.build_variant('spf2', 'spx_sddmm.cu', ['-DSPX_SDDMM_PF=2'])"
for v in spf1 spf2; do SPX_LIB=tools/variants/libspx_$v.so timeout 600 python -m pytest tests/test_gpu_edge.py tests/test_gpu_parity.py -q -x -k "sddmm or K6 or SDDMM" 2>&1 | tail -1; done
for rep in 1 2; do
for v in prod spf1 spf2; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 3 --only K6 --no-parity 2>&1 | tail -1 | cut -c1-120; done; done
echo done
