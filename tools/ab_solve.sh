#!/bin/bash
# aggregate solve throughput (16 threads x 16 streams) of library variants, interleaved repeats
for rep in 1 2 3; do
  for v in "$@"; do
    IFS=: read name envs <<< "$v"
    echo -n "$name $envs: "
    env RIGA_LIB=$PWD/variants/$name.so $envs timeout 300 python tools/concurrency_probe.py --steps 400 --what solveg --threads 16 | tail -1
  done
done
