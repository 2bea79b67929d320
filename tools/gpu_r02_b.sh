# Round-2 re-entry pass: GPU suite, smoke, bench (primary + secondaries), launch list.
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/b_pytest.txt 2>&1; tail -15 gpurun_out/b_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/b_smoke.txt 2>&1; cat gpurun_out/b_smoke.txt | tail -3
timeout 900 python bench.py > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err; tail -c 4000 gpurun_out/b_bench.json; tail -5 gpurun_out/b_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/b_launches.csv python bench.py --steps 2 --warmup 1 --profile > gpurun_out/b_bench_under_ncu.log 2>&1
echo done
