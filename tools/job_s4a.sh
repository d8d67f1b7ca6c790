set -x
python tools/one_factor.py cfg5 > gpurun_out/of.log 2>&1 || exit 1
# launches 330.. are the upper levels (wide K=512 trails); skip the first 300 launches of the profiled region
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:'k_trail128|k_trsm128|k_diag128|k_extend_add' -s 200 -c 14 -o /tmp/r2_factor_cfg5_full python tools/one_factor.py cfg5 > gpurun_out/ncu_f.log 2>&1
ncu -i /tmp/r2_factor_cfg5_full.ncu-rep --page raw --csv > gpurun_out/r2_factor_cfg5_full_raw.csv
ncu -i /tmp/r2_factor_cfg5_full.ncu-rep --page details > gpurun_out/r2_factor_cfg5_full_details.txt
ncu -i /tmp/r2_factor_cfg5_full.ncu-rep --page source --csv -k regex:k_trail128 -c 1 > gpurun_out/r2_trail128_source.csv
ls -la /tmp/r2_factor_cfg5_full.ncu-rep
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_s4.json 2> gpurun_out/bench_s4.err
