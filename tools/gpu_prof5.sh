timeout 900 python -m pytest tests/test_gpu_edge.py -x -q -k mttkrp 2>&1 | tail -2
NCU="ncu --set full --clock-control none --import-source on -c 1"
BC="python tools/bench_configs.py --reps 1 --warm 0 --no-parity"
timeout 600 $NCU -k regex:mttkrp_nnz_kernel -o gpurun_out/r1_mttkrp4 -f $BC --cfg 4 --only A6 > gpurun_out/p_mttkrp4.log 2>&1
