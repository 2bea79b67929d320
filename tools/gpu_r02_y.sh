# full GPU suite after the unscheduled / CPU-tagged remaps, then every config (parity + timings)
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 2400 python tools/bench_configs.py --cfg 1,5,2,3,4 > gpurun_out/y_configs.jsonl 2> gpurun_out/y_configs.err
grep -c '"ms"' gpurun_out/y_configs.jsonl
echo done
