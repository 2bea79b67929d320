# MTTKRP quarter kernel: reorderable C++ shared loads of the leaf slots (SPX_MQ_CLDS) vs asm volatile ld.shared
python -c "from paper_2001_00532_b200 import build as b; b.build_variant('clds', 'spx_csf.cu', ['-DSPX_MQ_CLDS=1'])"
SPX_LIB=tools/variants/libspx_clds.so timeout 600 python -m pytest tests/test_gpu_mttkrp_quarter.py -q -x 2>&1 | tail -1
for rep in 1 2; do for v in prod clds; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 4 --only A6 --no-parity 2>&1 | grep '"ms"' | cut -c1-110; done; done
echo done
