set -x
python -m pytest tests/test_gpu_sparsela.py -x -q 2>&1 | tail -3
python tools/one_factor.py cfg5 2>&1 | tail -1
RIGA_FACTOR_NB2=256 python tools/one_factor.py cfg5 2>&1 | tail -1
python tools/one_factor.py cfg4 2>&1 | tail -1
