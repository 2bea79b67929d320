# round-2 sanitizer pass over every kernel (incl. the new ones) + ncu --set full of the bench's SpMM
for t in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_smoke.py > gpurun_out/o_san_$t.log 2>&1; echo "$t rc=$?"; tail -3 gpurun_out/o_san_$t.log
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_nnz_kernel -s 2 -c 1 -o gpurun_out/o_spmm -f python bench.py --profile --steps 2 --warmup 1 --no-secondary > gpurun_out/o_ncu.log 2>&1; tail -2 gpurun_out/o_ncu.log
