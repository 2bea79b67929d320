# MTTKRP A.6 cfg4: dynamic chunk counter (SPX_MQ_DYN) vs grid-stride, 1 GPU and 8 weighted leaf-exact shards
python -c "from paper_2001_00532_b200 import build as b; b.build_variant('dyn', 'spx_csf.cu', ['-DSPX_MQ_DYN=1'])"
SPX_LIB=tools/variants/libspx_dyn.so timeout 600 python -m pytest tests/test_gpu_mttkrp_quarter.py tests/test_gpu_shards.py -q -x 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_mttkrp_quarter.py -q -x 2>&1 | tail -2
for rep in 1 2; do
for v in prod dyn; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 4 --only A6 --no-parity 2>&1 | tail -1 | cut -c1-120; done; done
for v in prod dyn; do echo "shards $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 900 python tools/bench_shards.py --cfg 4 --exact --fiber-weight 8 2>&1 | tail -4 | cut -c1-260; done
echo done
