"""Sum ncu --csv gpu__time_duration per kernel name from stdin (development aid)."""
import collections
import csv
import sys

tot, cnt = collections.Counter(), collections.Counter()
for row in csv.reader(line for line in sys.stdin if line.startswith('"')):
    if len(row) < 3 or row[0] == "ID" or not row[-1].replace(",", "").replace(".", "").isdigit():
        continue
    name = row[4].split("(")[0]
    scale = {"ns": 1e-6, "nsecond": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(row[-2], 1.0)
    tot[name] += float(row[-1].replace(",", "")) * scale
    cnt[name] += 1
for k, v in tot.most_common():
    print(f"{v:10.3f} ms  n={cnt[k]:4d}  {k}")
