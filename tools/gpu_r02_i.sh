# Round-2 measurement pass: every config and schedule with at-scale parity and the CPU
# restatement timed (-march=native, all host threads); bench line; launch list.
timeout 600 python -m pytest tests/test_gpu_irpath.py -q -x -k "stats" 2>&1 | tail -2
timeout 2400 python tools/bench_configs.py --cpu-time > gpurun_out/i_configs.jsonl 2> gpurun_out/i_configs.err; tail -3 gpurun_out/i_configs.err
timeout 900 python bench.py > gpurun_out/i_bench.json 2> gpurun_out/i_bench.err; tail -c 600 gpurun_out/i_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/i_launches.csv python bench.py --steps 2 --warmup 1 --profile > gpurun_out/i_bench_under_ncu.log 2>&1
echo done
