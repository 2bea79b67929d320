# edge matrices x the CPU-tagged / serial schedules
timeout 1500 python -m pytest tests/test_gpu_edge.py -q -x -rf 2>&1 | grep -E "FAILED|^E |passed|failed" | head -20
echo done
