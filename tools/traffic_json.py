"""Turn an ncu CSV of k_gravity (tools/gpu/r2_ncu_c4g.sh / r2_ncu_c2g.sh) into
profiles/traffic_<config>.json, the ncu evidence bench.py attaches to its
roofline: DRAM bytes per launch and executed FP32 operations by the paper's
rule (fadd + fmul + 2 ffma), with Blackwell's packed FP32x2
instructions counted per element (FADD2 / FMUL2 = 2, FFMA2 = 4 operations).

    python tools/traffic_json.py gpurun_out/ncu_c4g.csv c4 > profiles/traffic_c4.json
"""
import csv
import json
import sys

OPS = {  # metric suffix -> FP32 operations per thread instruction
    "fadd": 1, "fmul": 1, "ffma": 2, "fadd2": 2, "fmul2": 2, "ffma2": 4}


def main(path, config):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h, rows = rows[0], rows[1:]
    iK, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    m, kernel = {}, None
    for r in rows:
        if "k_gravity" not in r[iK]:
            continue
        kernel = kernel or r[iK]
        m[r[iM]] = float(r[iV].replace(",", ""))
    thread = {k: m.get(f"sm__sass_thread_inst_executed_op_{k}_pred_on.sum", 0.0) for k in OPS}
    ops = sum(OPS[k] * v for k, v in thread.items())
    rd, wr = m.get("dram__bytes_read.sum", 0.0), m.get("dram__bytes_write.sum", 0.0)
    out = {
        "config": config,
        "source": f"ncu --metrics (few-pass) over tools/profile_step.py --config {config} --steps 2, "
                  f"first k_gravity launch; CSV {path}",
        "kernel": kernel,
        "gravity_dram_bytes_per_launch": int(rd + wr),
        "gravity_dram_read_bytes": int(rd),
        "gravity_dram_write_bytes": int(wr),
        "gravity_fp32_ops_per_launch": int(ops),
        "fp32_rule": "fadd + fmul + 2 ffma + 2 fadd2 + 2 fmul2 + 4 ffma2 thread instructions "
                     "(PAPER.md:238, packed FP32x2 per element); no MUFU on the table path",
        **{f"thread_{k}": int(v) for k, v in thread.items()},
        "warp_instructions": int(m.get("smsp__inst_executed.sum", 0.0)),
        "duration_ns_under_ncu": int(m.get("gpu__time_duration.sum", 0.0)),
    }
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
