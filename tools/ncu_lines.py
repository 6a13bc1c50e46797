"""Per-CUDA-source-line instruction and stall shares from
`ncu -i REP -k KERNEL --page source --csv --print-source cuda,sass`:
    python tools/ncu_lines.py dump.csv [top]"""
import collections
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    cur_file, cur_line, cur_src = "", 0, ""
    ex = collections.Counter()
    smp = collections.Counter()
    text = {}
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
        if r[0].strip():  # a CUDA line row: "line", "source", ...
            try:
                cur_line = int(r[0])
            except ValueError:
                continue
            cur_src = r[1]
            text[(cur_file, cur_line)] = cur_src.strip()
        try:
            e = int(r[iex].replace(",", "") or 0)
            s = int(r[ismp].replace(",", "") or 0)
        except ValueError:
            continue
        if not r[0].strip():  # SASS rows under the current CUDA line
            ex[(cur_file, cur_line)] += e
            smp[(cur_file, cur_line)] += s
    te = sum(ex.values()) or 1
    ts = sum(smp.values()) or 1
    print(f"total warp-instr {te:.3e}  stall samples {ts}")
    for k, v in sorted(ex.items(), key=lambda kv: -kv[1] - smp[kv[0]] * te / ts)[:top]:
        print(f"{k[0]}:{k[1]:<5} ex {100 * v / te:5.1f}%  stall {100 * smp[k] / ts:5.1f}%  "
              f"{text.get(k, '')[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
