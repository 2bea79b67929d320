timeout 600 python -m pytest tests/test_gpu_ttv_stream.py -q -x 2>&1 | tail -2
timeout 500 python tools/bench_configs.py --cfg 4 --only K11 2>&1 | tail -5 | cut -c1-200
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_ttv.py 8192 512 16 2>/dev/null | grep -E "ttv_" | tail -2 | awk -F'","' '{print substr($5,1,40), $NF}'
