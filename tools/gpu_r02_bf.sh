# quarter walk (K9 cut for A.5, K9 warp per slice): leaf-ring depth (SPX_LEAF_RING 4 = product / 3 / 6 / 8)
python -c "
from paper_2001_00532_b200 import build as b
for r in (3, 6, 8): b.build_variant(f'lr{r}', 'spx_csf.cu', [f'-DSPX_LEAF_RING={r}'])"
SPX_LIB=tools/variants/libspx_lr6.so timeout 900 python -m pytest tests/test_gpu_mttkrp_slice.py -q -x 2>&1 | tail -1
for rep in 1 2; do for v in prod lr3 lr6 lr8; do echo "variant $v"; if [ $v = prod ]; then L=; else L=tools/variants/libspx_$v.so; fi
SPX_LIB=$L timeout 600 python tools/bench_configs.py --cfg 4 --only A5,K9 --no-parity 2>&1 | grep '"ms"' | cut -c1-90; done; done
echo done
