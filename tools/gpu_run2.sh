timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 900 python tools/bench_configs.py --cfg 1,5,2 2>&1 | grep -v "^#"
SPX_SPMM_RING=-1 timeout 600 python tools/bench_configs.py --cfg 2 --no-parity 2>&1 | grep -v "^#"
