NCU="ncu --set full --clock-control none --import-source on -c 1"
BC="python tools/bench_configs.py --reps 1 --warm 0 --no-parity"
timeout 600 $NCU -k regex:spmv_nnz_atomic_kernel -o gpurun_out/r1_spmv3 -f $BC --cfg 5 --only A2 > gpurun_out/p_spmv2.log 2>&1
