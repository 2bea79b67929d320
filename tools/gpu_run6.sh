for mb in 3 2 4; do
  SPX_NVCC_EXTRA="-DSPX_SPMM_MINB=$mb" python -c "from paper_2001_00532_b200 import build as b; b.build(force=True)"
  echo "MINB=$mb"; timeout 900 python tools/bench_configs.py --cfg 2 --only A4 --no-parity 2>&1 | grep -v "^#"
done
python -c "from paper_2001_00532_b200 import build as b; b.build(force=True)"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
