set -x
timeout 600 python -m pytest tests/test_gpu_sparsela.py tests/test_gpu_eigensolver.py -x -q 2>&1 | tail -3
timeout 300 python tools/time_solve.py cfg3 50 2>&1 | tail -1
timeout 300 python tools/time_solve.py cfg5 20 2>&1 | tail -1
timeout 300 python tools/concurrency_probe.py --steps 300 --what solve 2>&1 | tail -2
RIGA_SUB_PC=0 timeout 300 python tools/concurrency_probe.py --steps 300 --what solve 2>&1 | tail -2
