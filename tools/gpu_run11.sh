timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python tools/bench_fileio.py 2>&1 | tail -2
