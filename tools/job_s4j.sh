set -x
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:'k_trail128' -s 57 -c 1 -f -o /tmp/tr2 python tools/one_factor.py cfg5 > /dev/null 2>&1
ncu -i /tmp/tr2.ncu-rep --page details > gpurun_out/r2_trail128_full_details_final.txt
ncu -i /tmp/tr2.ncu-rep --page source --csv > gpurun_out/r2_trail128_source_final.csv
