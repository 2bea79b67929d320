# sanitizers over every kernel incl. the K9 heavy-slice cut and the serial-schedule nnz paths
python tools/sanitize_smoke.py 2>&1 | tail -3
for t in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_smoke.py > gpurun_out/aa_san_$t.log 2>&1; echo "$t rc=$?"; tail -2 gpurun_out/aa_san_$t.log
done
