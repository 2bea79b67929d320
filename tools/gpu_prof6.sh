NCU="ncu --set full --clock-control none --import-source on -c 1"
BC="python tools/bench_configs.py --reps 1 --warm 0 --no-parity"
timeout 600 $NCU -k regex:ttv_fiber -o gpurun_out/r1_ttv3 -f $BC --cfg 4 --only K7 > gpurun_out/p_ttv3.log 2>&1
