set -x
RIGA_SYM_TIME=1 python tools/one_factor.py cfg3 2>&1 | grep -i "symbolic_create\|factor ms"
RIGA_SYM_TIME=1 python tools/one_factor.py cfg5 2>&1 | grep -i "symbolic_create\|factor ms"
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:'k_trail128' -s 150 -c 4 -o /tmp/tr python tools/one_factor.py cfg5 > /dev/null 2>&1
ncu -i /tmp/tr.ncu-rep --page details > gpurun_out/r2_trail128_full_details_s4.txt
ncu -i /tmp/tr.ncu-rep --page raw --csv > gpurun_out/r2_trail128_full_raw_s4.csv
python tools/one_solve.py --config cfg3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_sub_|k_rest_|k_inv_' -c 40 -o /tmp/sv python tools/one_solve.py --config cfg3 --solves 1 > /dev/null 2>&1
ncu -i /tmp/sv.ncu-rep --page details > gpurun_out/r2_solve_cfg3_full_details_s4.txt
ncu -i /tmp/sv.ncu-rep --page raw --csv > gpurun_out/r2_solve_cfg3_full_raw_s4.csv
python tools/concurrency_probe.py --steps 300 --what solve 2>&1 | tail -2
