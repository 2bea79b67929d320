python -c "from paper_2001_00532_b200 import build as b; b.build_variant('hot0', 'spx_sddmm.cu', ['-DSPX_SDDMM_HOT=0']); b.build_variant('smw0', 'spx_csf.cu', ['-DSPX_MQ_SMWIN=0'])"
timeout 600 python -m pytest tests/test_gpu_irpath.py -q -x -k "stats" 2>&1 | grep -E "Error|error|assert|passed|failed" | head -20
timeout 600 python -m pytest tests/test_gpu_sddmm_hot.py tests/test_gpu_mttkrp_quarter.py -q -x 2>&1 | tail -3
timeout 600 python tools/bench_configs.py --cfg 3 --only K6 2>&1 | tail -1 | cut -c1-300
SPX_LIB=tools/variants/libspx_hot0.so timeout 600 python tools/bench_configs.py --cfg 3 --only K6 --no-parity 2>&1 | tail -1 | cut -c1-200
for f in 40 80; do python -c "from paper_2001_00532_b200 import build as b; b.build_variant('hf$f', 'spx_sddmm.cu', ['-DSPX_SDDMM_HOT_FRAC=$f'])"; SPX_LIB=tools/variants/libspx_hf$f.so timeout 600 python tools/bench_configs.py --cfg 3 --only K6 --no-parity 2>&1 | tail -1 | cut -c1-200; done
timeout 600 python tools/bench_configs.py --cfg 4 --only A6 --no-parity 2>&1 | tail -1 | cut -c1-200
SPX_LIB=tools/variants/libspx_smw0.so timeout 600 python tools/bench_configs.py --cfg 4 --only A6 --no-parity 2>&1 | tail -1 | cut -c1-200
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sddmm_nnz -c 1 -o gpurun_out/g_k6 -f python tools/bench_configs.py --reps 1 --warm 1 --no-parity --cfg 3 --only K6 > gpurun_out/g_k6.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp_quarter -c 1 -o gpurun_out/g_k8 -f python tools/bench_configs.py --reps 1 --warm 1 --no-parity --cfg 4 --only A6 > gpurun_out/g_k8.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/bench_configs.py --reps 1 --warm 0 --no-parity --cfg 3 --only K6 2>/dev/null | grep -E "col_degree|degree_hist|hot_thresh|hot_mask|sddmm_nnz|chunk_seg" > gpurun_out/g_k6_launches.csv
echo done
