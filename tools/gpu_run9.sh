timeout 900 python -m pytest tests/test_gpu_pack.py -x -q 2>&1 | tail -15
timeout 900 python tools/bench_pack.py 2>&1 | tail -5
