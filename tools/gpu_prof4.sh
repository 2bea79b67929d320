BC="python tools/bench_configs.py --reps 2 --warm 0 --no-parity"
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none -k regex:"spmv|chunk" $BC --cfg 5 --only A2 > gpurun_out/p_spmv3.txt 2>&1
grep -E "spmv|chunk|duration|warps_active|registers" gpurun_out/p_spmv3.txt | head -40
