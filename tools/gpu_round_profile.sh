# Round profile: GPU tests, smoke, bench, launch list + full ncu capture of the
# dominant kernel, every config.  Outputs land in gpurun_out/ (scratch);
# summaries are copied into profiles/ after review.
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/rp_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rp_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/rp_bench.json 2> gpurun_out/rp_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/rp_launches.csv python bench.py --steps 2 --warmup 1 --profile > gpurun_out/rp_bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_nnz_kernel -s 2 -c 1 -o gpurun_out/rp_spmm -f python bench.py --profile --steps 2 --warmup 1 > gpurun_out/rp_ncu_full.log 2>&1
timeout 1200 python tools/bench_configs.py > gpurun_out/rp_configs.jsonl 2> gpurun_out/rp_configs.err
timeout 600 python tools/bench_loadbal.py > gpurun_out/rp_loadbal.jsonl 2> gpurun_out/rp_loadbal.err
timeout 900 python tools/bench_shards.py > gpurun_out/rp_shards.jsonl 2> gpurun_out/rp_shards.err
timeout 600 python tools/bench_shards.py --cfg 4 --fiber-weight 25 > gpurun_out/rp_shards_weighted.jsonl 2>> gpurun_out/rp_shards.err
cat gpurun_out/rp_pytest.txt gpurun_out/rp_smoke.txt gpurun_out/rp_bench.json
