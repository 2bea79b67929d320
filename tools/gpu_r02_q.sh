timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/q_pytest.txt 2>&1; tail -3 gpurun_out/q_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --impl reference > gpurun_out/q_ref.json 2> gpurun_out/q_ref.err; tail -c 700 gpurun_out/q_ref.json
timeout 900 python bench.py > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; python -c "
import json; d=json.load(open('gpurun_out/q_bench.json')); print(d['value'], d['ms_per_step'], d['clocks'], d['e2e']['value'], d['roofline']['frac'], d['parity']['ok'], [ (s['workload'][:5], s['ms_per_step'], s['value']) for s in d['secondary']])"
