"""Write profiles/ summaries from ncu outputs (run here, no GPU needed):
  python tools/ncu_digest.py launches <launches.csv> <out.md> ["<command / note>"]
  python tools/ncu_digest.py kernels <report.ncu-rep> <out.md>"""
import collections
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active lanes / instruction"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__sass_thread_inst_executed_op_ffma2_pred_on.sum", "FFMA2 thread instructions"),
    ("sm__sass_thread_inst_executed_op_fmul2_pred_on.sum", "FMUL2 thread instructions"),
    ("sm__sass_thread_inst_executed_op_fadd2_pred_on.sum", "FADD2 thread instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__sass_thread_inst_executed_op_ffma_pred_on.sum", "thread FFMA"),
    ("sm__sass_thread_inst_executed_op_fadd_pred_on.sum", "thread FADD"),
    ("sm__sass_thread_inst_executed_op_fmul_pred_on.sum", "thread FMUL"),
]


def launches(path, out, what="`tools/profile_step.py --steps 2` (2x128^3, c2)"):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in data:
        name = r[ki].split("(")[0]
        v = float(r[vi].replace(",", ""))
        if r[ui] == "msecond":
            v *= 1e6
        elif r[ui] == "usecond":
            v *= 1e3
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list: {path}\n\n`ncu --metrics gpu__time_duration.sum "
                f"--clock-control none` over {what}; "
                "cold-cache serialised launches: compare shares.\n\n")
        f.write(f"Total {T / 1e6:.3f} ms over {len(data)} launches.\n\n")
        f.write("| kernel | launches | total ms | share |\n|---|---|---|---|\n")
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            f.write(f"| `{k}` | {cnt[k]} | {v / 1e6:.3f} | {100 * v / T:.1f}% |\n")


def kernels(path, out):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    with open(out, "w") as f:
        f.write(f"# ncu --set full digest: {path}\n\n")
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            u = dict(zip(hdr, units))
            f.write(f"## `{d.get('Kernel Name', '?')}`\n\n| metric | value |\n|---|---|\n")
            for k, lab in KEYS:
                if k in d:
                    f.write(f"| {lab} (`{k}`) | {d[k]} {u.get(k, '')} |\n")
            f.write("\n")


if __name__ == "__main__":
    {"launches": launches, "kernels": kernels}[sys.argv[1]](*sys.argv[2:])
