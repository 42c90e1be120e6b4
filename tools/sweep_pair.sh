#!/bin/bash
# Column-pair kernel strip heights (TS_PCG_PAIR) vs the single-column kernel (0).
for cfg in "$@"; do
  for R in ${PAIRS:-0 5 6 7}; do
    out=$(TS_PCG_PAIR=$R timeout 300 python tools/probe.py $cfg 2>&1 | tail -1)
    echo "$cfg PAIR=$R $(echo "$out" | python -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); print("rate=%.3e micro_ms=%.1f macro_ms=%.1f sweeps=%d" % (d["rate"], d["micro_ms"], d["macro_ms"], d["sweeps"]))
except Exception as e: print("fail", e)')"
  done
done
