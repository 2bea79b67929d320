python -c "from paper_2001_00532_b200 import build as b; b.build_variant('seg0', 'spx_csf.cu', ['-DSPX_MQ_SEGLOOP=0'])"
timeout 600 python -m pytest tests/test_gpu_mttkrp_quarter.py tests/test_gpu_shards.py -q -x 2>&1 | tail -2
timeout 600 python tools/bench_configs.py --cfg 4 --only A6 2>&1 | tail -1 | cut -c1-250
SPX_LIB=tools/variants/libspx_seg0.so timeout 600 python tools/bench_configs.py --cfg 4 --only A6 --no-parity 2>&1 | tail -1 | cut -c1-200
timeout 600 python tools/bench_configs.py --cfg 4 --only A6 --no-parity 2>&1 | tail -1 | cut -c1-200
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp_quarter -c 1 -o gpurun_out/n_k8 -f python tools/bench_configs.py --reps 1 --warm 1 --no-parity --cfg 4 --only A6 > gpurun_out/n_k8.log 2>&1
echo done
