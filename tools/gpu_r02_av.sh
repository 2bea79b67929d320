# UNIT-mode quarter kernel profile (cfg4 A.5): launch list + ncu of the quarter kernel
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/av_launch.csv python tools/bench_configs.py --reps 2 --warm 1 --no-parity --cfg 4 --only A5 > gpurun_out/av.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mttkrp_quarter -c 1 -o gpurun_out/av_unit -f python tools/bench_configs.py --reps 1 --warm 1 --no-parity --cfg 4 --only A5 > gpurun_out/av2.log 2>&1; echo rc=$?
