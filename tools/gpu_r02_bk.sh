# ncu of K9's warp-per-slice walk (cfg4): where the lone heavy-slice warp waits
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mttkrp_slice -c 1 -o gpurun_out/bk_k9 -f python tools/bench_configs.py --reps 1 --warm 1 --no-parity --cfg 4 --only K9 > gpurun_out/bk.log 2>&1; echo rc=$?
