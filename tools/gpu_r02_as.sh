# quarter kernel: group-loop unroll (SPX_MQ_HUNROLL 4 = product / 2 / 1) -- code size vs per-group overhead
python -c "
from paper_2001_00532_b200 import build as b
b.build_variant('hu2', 'spx_csf.cu', ['-DSPX_MQ_HUNROLL=2']); b.build_variant('hu1', 'spx_csf.cu', ['-DSPX_MQ_HUNROLL=1'])"
SPX_LIB=tools/variants/libspx_hu2.so timeout 900 python -m pytest tests/test_gpu_mttkrp_quarter.py -q -x 2>&1 | tail -1
for rep in 1 2; do for v in prod hu2 hu1; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 4 --only A6 --no-parity 2>&1 | grep '"ms"' | cut -c1-100; done; done
echo done
