timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python tools/bench_configs.py --cfg 2 --only A4 2>&1 | grep -v "^#"
SPX_SPMM_RING=-1 timeout 900 python tools/bench_configs.py --cfg 2 --only A4 2>&1 | grep -v "^#"
NCU="ncu --set full --clock-control none --import-source on -c 1"
BC="python tools/bench_configs.py --reps 1 --warm 0 --no-parity"
SPX_SPMM_RING=-1 timeout 600 $NCU -k regex:spmm_nnz_kernel -o gpurun_out/r1_spmm_reg2 -f $BC --cfg 2 --only A4 > gpurun_out/p_spmm2.log 2>&1
