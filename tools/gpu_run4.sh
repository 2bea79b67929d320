timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python tools/bench_configs.py --cfg 4 --only A6,K7 2>&1 | grep -v "^#"
NCU="ncu --set full --clock-control none --import-source on -c 1"
BC="python tools/bench_configs.py --reps 1 --warm 0 --no-parity"
timeout 600 $NCU -k regex:mttkrp_nnz_kernel -o gpurun_out/r1_mttkrp3 -f $BC --cfg 4 --only A6 > gpurun_out/p_mttkrp3.log 2>&1
