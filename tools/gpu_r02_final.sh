# round-2 final check: build from source, full GPU suite, smoke, reference arm, bench line, launch list
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fin_build.txt 2>&1; echo "build rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/fin_pytest.txt 2>&1; tail -2 gpurun_out/fin_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --impl reference > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err; tail -c 200 gpurun_out/fin_ref.json
timeout 900 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; python -c "
import json; d=json.load(open('gpurun_out/fin_bench.json')); print(d['value'], d['ms_per_step'], d['clocks'], d['e2e']['value'], d['e2e'].get('link',{}).get('frac'), d['roofline']['frac'], d['roofline'].get('port_bound',{}).get('frac'), d['parity']['ok'], d['gpu_launches'], [ (s['workload'][:5], s['ms_per_step'], s['value']) for s in d['secondary']])"
echo done
