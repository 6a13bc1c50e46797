"""Per-SASS-instruction hot spots from `ncu --page source --print-source sass --csv`:
prints instruction-executed counts and stall samples grouped into regions
between branch targets so loops are visible."""
import csv
import sys


def main(path, top=60):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iex = hdr.index("Instructions Executed")
    isamp = hdr.index("Warp Stall Sampling (All Samples)")
    recs = []
    for r in rows[2:]:
        if len(r) <= iex:
            continue
        try:
            ex = int(r[iex].replace(",", "") or 0)
            sm = int(r[isamp].replace(",", "") or 0)
        except ValueError:
            continue
        recs.append((r[ia], r[isrc], ex, sm))
    tot_ex = sum(x[2] for x in recs) or 1
    tot_sm = sum(x[3] for x in recs) or 1
    print(f"total warp-instr {tot_ex:.3e}, samples {tot_sm}")
    # print contiguous instructions with their share
    for a, s, ex, sm in recs:
        if ex / tot_ex > 0.002 or sm / tot_sm > 0.004:
            print(f"{a:>6} {100*ex/tot_ex:5.2f}% ex {100*sm/tot_sm:5.2f}% smp  {s[:70]}")


if __name__ == "__main__":
    main(sys.argv[1])
