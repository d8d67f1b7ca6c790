set -x
timeout 300 python -m pytest tests/test_gpu_sparsela.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout 200 python tools/one_factor.py cfg5 2>&1 | tail -1; done
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_dmma.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2_factor_launches_cfg5_s4g.csv python tools/one_factor.py cfg5 > /dev/null 2>&1
