# SpMV A.2 cfg5: x gathers with L1::evict_last (SPX_SPMV_X_EL) vs the product
python -c "from paper_2001_00532_b200 import build as b; b.build_variant('xel', 'spx_spmv.cu', ['-DSPX_SPMV_X_EL=1'])"
for rep in 1 2; do for v in prod xel; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 5 --only A2 --no-parity 2>&1 | grep '"ms"' | cut -c1-100; done; done
echo done
