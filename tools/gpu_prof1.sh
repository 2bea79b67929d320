# one ncu --set full capture per kernel family (tooling; results under gpurun_out/)
NCU="ncu --set full --clock-control none --import-source on -c 1"
BC="python tools/bench_configs.py --reps 1 --warm 0 --no-parity"
timeout 600 $NCU -k regex:spmv_nnz_kernel -o gpurun_out/r1_spmv_nnz -f $BC --cfg 5 --only A2 > gpurun_out/p_spmv.log 2>&1
SPX_SPMM_RING=-1 timeout 600 $NCU -k regex:spmm_nnz_kernel -o gpurun_out/r1_spmm_reg -f $BC --cfg 2 --only A4 > gpurun_out/p_spmm.log 2>&1
timeout 600 $NCU -k regex:mttkrp_nnz_kernel -o gpurun_out/r1_mttkrp_nnz -f $BC --cfg 4 --only A6 > gpurun_out/p_mttkrp.log 2>&1
timeout 600 $NCU -k regex:ttv_fiber -o gpurun_out/r1_ttv -f $BC --cfg 4 --only K7 > gpurun_out/p_ttv.log 2>&1
timeout 600 $NCU -k regex:sddmm_nnz -o gpurun_out/r1_sddmm_nnz -f $BC --cfg 3 --only K6 > gpurun_out/p_sddmm.log 2>&1
ls -la gpurun_out/
