cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
for t in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_case.py cfg2 > gpurun_out/san_${t}_cfg2.log 2>&1; echo rc=$? >> gpurun_out/san_${t}_cfg2.log
done
timeout 900 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_case.py cfg4 > gpurun_out/san_racecheck_cfg4.log 2>&1; echo rc=$? >> gpurun_out/san_racecheck_cfg4.log
timeout 600 compute-sanitizer --tool synccheck --print-limit 50 python tools/sanitize_case.py cfg4 > gpurun_out/san_synccheck_cfg4.log 2>&1; echo rc=$? >> gpurun_out/san_synccheck_cfg4.log
RIGA_TRACE=1 timeout 300 python tools/slice_timeline.py cfg3 16 2 > gpurun_out/timeline_cfg3.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/solve_launches_cfg3.csv python tools/one_solve.py --config cfg3 --solves 2 > gpurun_out/ncu_solve.log 2>&1
