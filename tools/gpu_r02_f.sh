# Round-2 ncu captures of the kernels round 1 left unprofiled (VERDICT missing #8) + stats test.
timeout 600 python -m pytest tests/test_gpu_irpath.py -q -x -k "stats or tail or divide" 2>&1 | tail -3
P="--set full --clock-control none --import-source on -c 1"
BC="python tools/bench_configs.py --reps 1 --warm 1 --no-parity"
timeout 600 ncu $P -k regex:spmv_row -o gpurun_out/f_k1 -f $BC --cfg 5 --only A7 > gpurun_out/f_k1.log 2>&1
timeout 600 ncu $P -k regex:spmv_warp -o gpurun_out/f_k2 -f $BC --cfg 5 --only A8 > gpurun_out/f_k2.log 2>&1
timeout 600 ncu $P -k regex:spmm_row -o gpurun_out/f_k5 -f $BC --cfg 2 --only K5 > gpurun_out/f_k5.log 2>&1
timeout 600 ncu $P -k regex:sddmm_row -o gpurun_out/f_k10 -f $BC --cfg 3 --only K10 > gpurun_out/f_k10.log 2>&1
timeout 600 ncu $P -k regex:ttv_stream -o gpurun_out/f_k11 -f $BC --cfg 4 --only K11 > gpurun_out/f_k11.log 2>&1
timeout 600 ncu $P -k regex:mttkrp_quarter -o gpurun_out/f_k8 -f $BC --cfg 4 --only A6 > gpurun_out/f_k8.log 2>&1
timeout 600 ncu $P -k regex:sddmm_nnz -o gpurun_out/f_k6 -f $BC --cfg 3 --only K6 > gpurun_out/f_k6.log 2>&1
timeout 600 ncu $P -k regex:spmv_nnz -o gpurun_out/f_k3 -f $BC --cfg 5 --only A2 > gpurun_out/f_k3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/bench_pack.py --cfg 2 --reps 1 > gpurun_out/f_pack.csv 2> gpurun_out/f_pack.err
ls -la gpurun_out/ | grep f_
