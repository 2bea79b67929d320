# quarter kernel slow path as a runtime loop (SPX_MQ_SLOWLOOP, half the code) -- A.6 (red.add) and A.5 (deterministic slots)
python -c "from paper_2001_00532_b200 import build as b; b.build_variant('sl1', 'spx_csf.cu', ['-DSPX_MQ_SLOWLOOP=1'])"
SPX_LIB=tools/variants/libspx_sl1.so timeout 900 python -m pytest tests/test_gpu_mttkrp_slice.py tests/test_gpu_mttkrp_quarter.py -q -x 2>&1 | tail -1
for rep in 1 2; do for v in prod sl1; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 4 --only A6,A5 --no-parity 2>&1 | grep '"ms"' | cut -c1-100; done; done
echo done
