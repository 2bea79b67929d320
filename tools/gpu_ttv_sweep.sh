for v in "" tools/variants/libspx_ttvnopf.so; do
  echo "== variant ${v:-default}"
  SPX_LIB=$v timeout 300 python tools/bench_configs.py --cfg 4 --only K11 --no-parity 2>&1 | grep -o '"schedule": "[^"]*".*"ms": [0-9.]*' | sed 's/"kernel".*"ms"/ms/'
done
timeout 300 python -m pytest tests/test_gpu_ttv_stream.py -q -x 2>&1 | tail -2
