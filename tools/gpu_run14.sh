for flag in "" "-DSPX_GATHER_L1_NOALLOC"; do
  SPX_NVCC_EXTRA="$flag" python -c "from paper_2001_00532_b200 import build as b; b.build(force=True)"
  echo "flag=$flag"; timeout 900 python tools/bench_configs.py --cfg 2 --only A4 --no-parity 2>&1 | grep -v "^#"
done
