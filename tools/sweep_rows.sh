#!/bin/bash
# Times the batched micro PCG for each strip height R (TS_PCG_ROWS) on the given configs.
for cfg in "$@"; do
  for R in ${ROWS:-2 3 4 5 7 9 13 17 22}; do
    out=$(TS_PCG_ROWS=$R timeout 300 python tools/probe.py $cfg 2>&1 | tail -1)
    echo "$cfg R=$R $(echo "$out" | python -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); print("rate=%.3e micro_ms=%.1f macro_ms=%.1f sweeps=%d" % (d["rate"], d["micro_ms"], d["macro_ms"], d["sweeps"]))
except Exception as e: print("fail", e)')"
  done
done
