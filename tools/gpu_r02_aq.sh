# ncu of the deterministic quarter K9 kernel (cfg4 A.5)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mttkrp_quarter -c 1 -o gpurun_out/aq_det -f python tools/bench_configs.py --reps 1 --warm 1 --no-parity --cfg 4 --only A5 > gpurun_out/aq.log 2>&1; echo "rc=$?"
