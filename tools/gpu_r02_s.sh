# MTTKRP A.6 cfg4: L1 prefetch of D rows -- PF=1 next batch (ring 3 / 4), PF=2 this batch's later groups (ring 2) -- vs the product
python -c "from paper_2001_00532_b200 import build as b; b.build_variant('pf3', 'spx_csf.cu', ['-DSPX_MQ_PF=1','-DSPX_MQ_RING=3']); b.build_variant('pf2', 'spx_csf.cu', ['-DSPX_MQ_PF=2']); b.build_variant('pf4', 'spx_csf.cu', ['-DSPX_MQ_PF=1','-DSPX_MQ_RING=4'])"
SPX_LIB=tools/variants/libspx_pf2.so timeout 600 python -m pytest tests/test_gpu_mttkrp_quarter.py -q -x 2>&1 | tail -2
for rep in 1 2; do
for v in prod pf2 pf3 pf4; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 4 --only A6 --no-parity 2>&1 | tail -1 | cut -c1-120; done; done
echo done
