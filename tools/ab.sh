#!/bin/bash
# A/B timing of library builds in ab/*.so on the same box: tools/ab.sh c3 [c2 ...]
for round in 1 2; do
  for lib in ab/*.so; do
    echo "== $lib round $round"
    TS_B200_LIB=$lib python tools/bench_all.py "$@" --no-cpu 2>&1 | grep "^| c"
  done
done
