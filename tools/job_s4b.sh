set -x
for la in 1 0; do RIGA_FACTOR_LOOKAHEAD=$la python tools/one_factor.py cfg5 2>&1 | tail -1; done
for nb in 384 640 768; do RIGA_FACTOR_NB2=$nb python tools/one_factor.py cfg5 2>&1 | tail -1; done
