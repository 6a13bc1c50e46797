"""Summarise an ncu report (--page raw) for the kernels in it: time, DRAM
bytes, issue/pipe utilisation, lane efficiency, warp stall reasons."""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time_ms", 1e-6),
    ("dram__bytes_read.sum", "dram_read_MB", 1e-6),
    ("dram__bytes_write.sum", "dram_write_MB", 1e-6),
    ("smsp__inst_executed.sum", "warp_inst_G", 1e-9),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "lanes_per_inst", 1),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma_pipe_pct", 1),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu_pipe_pct", 1),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_pipe_pct", 1),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_pipe_pct", 1),
    ("sm__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct", 1),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts", 1),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts", 1),
    ("sm__sass_thread_inst_executed_op_ffma_pred_on.sum", "thread_ffma_G", 1e-9),
    ("sm__sass_thread_inst_executed_op_fadd_pred_on.sum", "thread_fadd_G", 1e-9),
    ("sm__sass_thread_inst_executed_op_fmul_pred_on.sum", "thread_fmul_G", 1e-9),
    ("sm__sass_thread_inst_executed_op_ffma2_pred_on.sum", "thread_ffma2_G", 1e-9),
    ("sm__sass_thread_inst_executed_op_fadd2_pred_on.sum", "thread_fadd2_G", 1e-9),
    ("sm__sass_thread_inst_executed_op_fmul2_pred_on.sum", "thread_fmul2_G", 1e-9),
    ("launch__registers_per_thread", "regs", 1),
]
STALL = "smsp__average_warp_latency_issue_stalled_"


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "?")[:60]
        print(f"== {name}")
        for k, lab, sc in KEYS:
            if k in d and d[k] not in ("", "n/a"):
                try:
                    print(f"   {lab:22s} {float(d[k].replace(',', '')) * sc:12.4f}")
                except ValueError:
                    pass
        stalls = []
        for k, v in d.items():
            if k.startswith(STALL) and k.endswith(".ratio"):
                try:
                    stalls.append((float(v.replace(",", "")), k[len(STALL):-6]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("   top stalls:", ", ".join(f"{n}={v:.2f}" for v, n in stalls[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
