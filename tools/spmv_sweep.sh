#!/bin/bash
# Sweep CSR SpMV lanes-per-row x elements-per-lane on the cfg pencils (L2 flushed per launch).
cd "$(dirname "$0")/.."
for cfg in ${CFGS:-cfg3 cfg4}; do
  python tools/spmv_probe.py $cfg
  for L in 8 16 32; do for U in 4 6 8; do
    RIGA_SPMV_LANES=$L RIGA_SPMV_U=$U python tools/spmv_probe.py $cfg
  done; done
done
