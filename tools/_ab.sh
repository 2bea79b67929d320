for v in "-DSPX_MTTKRP_SLICE_G=4 -DSPX_MTTKRP_SLICE_MINB=2" ""; do
  SPX_NVCC_EXTRA="$v" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD FAIL
  echo "variant [$v] $(python tools/bench_configs.py --cfg 4 --only K9 --no-parity 2>&1 | grep -o '"ms": [0-9.]*\|Error.*' | head -2)"
done
python -m pytest tests -m gpu -q -x -k "mttkrp or K9 or A5 or MTTKRP" 2>&1 | tail -1
