timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python tools/bench_configs.py --cfg 3 2>&1 | grep -v "^#"
