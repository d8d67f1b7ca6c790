#!/bin/bash
# A/B the library builds in variants/*.so: isolated solve, aggregate solves, slice timeline
for v in "$@"; do
  echo "== $v"
  RIGA_LIB=$PWD/variants/$v.so timeout 300 python tools/profile_ops.py --config cfg3 --reps 30 2>&1 | grep -A1 '"solve": {' | tail -1
  RIGA_LIB=$PWD/variants/$v.so timeout 300 python tools/concurrency_probe.py --steps 300 --what solve | tail -1
  RIGA_LIB=$PWD/variants/$v.so OPENBLAS_NUM_THREADS=1 timeout 300 python tools/slice_timeline.py cfg3 16 3 2>&1 | grep total | tail -2
done
