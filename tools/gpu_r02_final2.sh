# round-2 final check (2): full suite, smoke, reference arm, bench line, and the per-config records
bash tools/gpu_r02_final.sh
timeout 3000 python tools/bench_configs.py --cfg 1,5,2,3,4 --cpu-time > gpurun_out/fin_configs.jsonl 2> gpurun_out/fin_configs.err; grep -c '"ms"' gpurun_out/fin_configs.jsonl
