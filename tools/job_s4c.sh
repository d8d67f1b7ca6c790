set -x
ncu --set full --clock-control none --import-source on -k regex:syrk_tiles128 -c 1 -o /tmp/dg tools/bench_dmma/dgemm_bench 8192 512 > /dev/null 2>&1
ncu -i /tmp/dg.ncu-rep --page source --csv > gpurun_out/dg_source.csv
ncu -i /tmp/dg.ncu-rep --page details > gpurun_out/dg_details.txt
