set -x
timeout 60 tools/bench_dmma/dgemm_bench 4096 2048 | tail -2
timeout 60 tools/bench_dmma/dgemm_bench 8192 512 | tail -2
timeout 60 tools/bench_dmma/dgemm_bench 1000 100 | tail -2
timeout 300 python -m pytest tests/test_gpu_sparsela.py -x -q 2>&1 | tail -3
timeout 200 python tools/one_factor.py cfg5 2>&1 | tail -1
timeout 200 python tools/one_factor.py cfg4 2>&1 | tail -1
timeout 200 python tools/one_factor.py cfg3 2>&1 | tail -1
