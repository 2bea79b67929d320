# final per-config records (every schedule incl. the serial / CPU-tagged remaps) with the CPU restatement timed
timeout 3000 python tools/bench_configs.py --cfg 1,5,2,3,4 --cpu-time > gpurun_out/ag_configs.jsonl 2> gpurun_out/ag_configs.err
grep -c '"ms"' gpurun_out/ag_configs.jsonl; tail -2 gpurun_out/ag_configs.err
timeout 1800 python tools/bench_shards.py --cfg 2,5 > gpurun_out/ag_shards.jsonl 2>&1; tail -1 gpurun_out/ag_shards.jsonl | cut -c1-200
timeout 1800 python tools/bench_shards.py --cfg 4 --exact --fiber-weight 8 > gpurun_out/ag_shards4.jsonl 2>&1; tail -1 gpurun_out/ag_shards4.jsonl | cut -c1-200
echo done
