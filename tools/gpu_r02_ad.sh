# checkpoint: full GPU suite, smoke, reference arm, bench (port bound + PCIe link), launch list, ncu of the new kernels
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/ad_pytest.txt 2>&1; tail -2 gpurun_out/ad_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --impl reference > gpurun_out/ad_ref.json 2> gpurun_out/ad_ref.err; tail -c 300 gpurun_out/ad_ref.json
timeout 900 python bench.py > gpurun_out/ad_bench.json 2> gpurun_out/ad_bench.err; python -c "
import json; d=json.load(open('gpurun_out/ad_bench.json')); print(d['value'], d['ms_per_step'], d['clocks'], d['e2e']['value'], d['e2e'].get('link'), d['roofline']['frac'], d['roofline'].get('port_bound'), d['parity']['ok'], [ (s['workload'][:5], s['ms_per_step'], s['value']) for s in d['secondary']])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ad_launches.csv python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu --e2e-steps 0 > gpurun_out/ad_bench_under_ncu.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp_quarter -c 1 -o gpurun_out/ad_k8 -f python tools/bench_configs.py --reps 1 --warm 1 --no-parity --cfg 4 --only A6 > gpurun_out/ad_k8.log 2>&1; echo "k8 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp_slice -c 1 -o gpurun_out/ad_k9s -f python tools/bench_configs.py --reps 1 --warm 1 --no-parity --cfg 4 --only A5 > gpurun_out/ad_k9s.log 2>&1; echo "k9 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_row -c 1 -o gpurun_out/ad_k5c -f python tools/bench_configs.py --reps 1 --warm 1 --no-parity --cfg 2 --only A3 > gpurun_out/ad_k5c.log 2>&1; echo "k5 rc=$?"
echo done
