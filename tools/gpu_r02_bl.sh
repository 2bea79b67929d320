# quarter walk: D-row L1 prefetch PFD batches ahead, the leaf index read one batch earlier (SPX_MQUAD_PFD)
python -c "from paper_2001_00532_b200 import build as b; b.build_variant('pd3', 'spx_csf.cu', ['-DSPX_MQUAD_PFD=3']); b.build_variant('pd8', 'spx_csf.cu', ['-DSPX_MQUAD_PFD=8'])"
SPX_LIB=tools/variants/libspx_pd3.so timeout 900 python -m pytest tests/test_gpu_mttkrp_slice.py -q -x 2>&1 | tail -1
for rep in 1 2; do for v in prod pd3 pd8; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 4 --only K9,A5 --no-parity 2>&1 | grep '"ms"' | cut -c1-90; done; done
echo done
