set -x
tools/bench_dmma/dgemm_bench 4096 2048
tools/bench_dmma/dgemm_bench 4096 512
python -m pytest tests/test_gpu_sparsela.py -x -q 2>&1 | tail -5
python tools/one_factor.py cfg5 2>&1 | tail -1
RIGA_FACTOR_LOOKAHEAD=0 python tools/one_factor.py cfg5 2>&1 | tail -1
