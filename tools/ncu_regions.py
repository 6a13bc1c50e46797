"""Instruction / stall shares of line ranges from the same dump as ncu_lines.py:
    python tools/ncu_regions.py dump.csv file:lo-hi=name ..."""
import collections
import csv
import sys


def main(path, specs):
    rows = list(csv.reader(open(path)))
    cur_file, cur_line = "", 0
    ex, smp = collections.Counter(), collections.Counter()
    iex = ismp = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            iex = r.index("Instructions Executed")
            ismp = r.index("Warp Stall Sampling (All Samples)")
            continue
        if iex is None or len(r) <= iex:
            continue
        if r[0].strip():
            try:
                cur_line = int(r[0])
            except ValueError:
                pass
            continue
        try:
            e = int(r[iex] or 0)
            s = int(r[ismp] or 0)
        except ValueError:
            continue
        ex[(cur_file, cur_line)] += e
        smp[(cur_file, cur_line)] += s
    te, ts = sum(ex.values()) or 1, sum(smp.values()) or 1
    regions = []
    for sp in specs:
        loc, name = sp.split("=")
        f, rng = loc.split(":")
        lo, hi = (int(x) for x in rng.split("-"))
        regions.append((f, lo, hi, name))
    acc_e, acc_s = collections.Counter(), collections.Counter()
    for (f, ln), e in ex.items():
        name = "other"
        for rf, lo, hi, nm in regions:
            if f == rf and lo <= ln <= hi:
                name = nm
                break
        acc_e[name] += e
        acc_s[name] += smp[(f, ln)]
    print(f"total warp-instr {te:.3e}")
    for nm in sorted(acc_e, key=lambda k: -acc_e[k]):
        print(f"{nm:14s} instr {100 * acc_e[nm] / te:5.1f}%  ({acc_e[nm]:.3e})  stall {100 * acc_s[nm] / ts:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
