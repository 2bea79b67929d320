# pack with the single-pass decoupled look-back scan: bit-exact tests + kernel launch list at cfg2
timeout 1500 python -m pytest tests/test_gpu_pack.py tests/test_gpu_coo.py -q -x -rf 2>&1 | grep -E "FAILED|^E |passed|failed|rror" | head -10
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ai_pack.csv python tools/bench_pack.py --cfg 2 > gpurun_out/ai_pack.log 2>&1; echo "ncu rc=$?"
echo done
