# quarter walk (K9 warp-per-slice, K9 cut, K8 non-quarter shapes): next-batch L1 prefetch of D rows (SPX_MQUAD_PF)
python -c "from paper_2001_00532_b200 import build as b; b.build_variant('qpf', 'spx_csf.cu', ['-DSPX_MQUAD_PF=1'])"
SPX_LIB=tools/variants/libspx_qpf.so timeout 900 python -m pytest tests/test_gpu_mttkrp_slice.py tests/test_gpu_edge.py -q -x -k "mttkrp or slice" 2>&1 | tail -1
for rep in 1 2; do for v in prod qpf; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 4 --only K9,A5 --no-parity 2>&1 | grep '"ms"' | cut -c1-100; done; done
echo done
