# SDDMM K6: L1::no_allocate on the 256-bit D-row gathers (SPX_LD256_NA) vs the product
python -c "from paper_2001_00532_b200 import build as b; b.build_variant('na_sddmm', 'spx_sddmm.cu', ['-DSPX_LD256_NA=1'])"
for rep in 1 2; do for v in prod na_sddmm; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 3 --only K6 --no-parity 2>&1 | grep '"ms"' | cut -c1-110; done; done
echo done
