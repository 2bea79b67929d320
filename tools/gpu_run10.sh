timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python tools/bench_configs.py --cfg 4,2,3 --only A6,K7,A4,K6 2>&1 | grep -v "^#"
