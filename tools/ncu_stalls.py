"""Stall-reason totals (sampling) of one kernel from
`ncu -i REP --page source --csv --print-source cuda,sass -k KERNEL` output:
    python tools/ncu_stalls.py dump.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot = collections.Counter()
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or r[0].strip() or len(r) != len(hdr):
        continue
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                tot[h] += int(r[i] or 0)
            except ValueError:
                pass
s = sum(tot.values()) or 1
for k, v in tot.most_common(12):
    print(f"{k:28s} {100 * v / s:5.1f}%")
