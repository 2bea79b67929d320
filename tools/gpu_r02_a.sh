# Round-2 first GPU pass: full GPU suite (incl. full-scale cfg2-5 parity),
# bench (primary + secondaries), gather-path counters for the SpMM ceiling.
M="l1tex__m_xbar2l1tex_read_bytes.sum,l1tex__m_xbar2l1tex_read_bytes.sum.per_second,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_bytes.sum.per_second,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg,sm__cycles_elapsed.avg.per_second,gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__t_bytes.sum.per_second,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,lts__t_sector_hit_rate.pct,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed"
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/a_pytest.txt 2>&1; tail -15 gpurun_out/a_pytest.txt
timeout 900 python bench.py > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err; tail -c 3000 gpurun_out/a_bench.json; tail -5 gpurun_out/a_bench.err
timeout 600 ncu --metrics $M --clock-control none -k regex:spmm_nnz_kernel -s 2 -c 1 --csv python bench.py --profile --steps 2 --warmup 1 --no-secondary > gpurun_out/a_ncu_spmm.csv 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:g_reg -c 4 --csv python tools/gbench2.py > gpurun_out/a_ncu_greg.csv 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:"g_g4|g_dsm" -c 3 --csv python tools/gbench3.py > gpurun_out/a_ncu_g3.csv 2>&1
echo done
