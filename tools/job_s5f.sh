#!/bin/bash
for h in 0 2 4 6 11; do
  echo "== RIGA_PRIO_HIGH=$h"
  RIGA_PRIO_HIGH=$h timeout 600 python tools/slice_timeline.py cfg3 16 5 2>&1 | grep "^total" | tail -3
done
