"""Summarise an `ncu --set full` report of the hot-path kernels.

python tools/ncu_summary.py REPORT.ncu-rep OUT.md [--traffic profiles/traffic.json]

Writes a markdown table per kernel (duration, DRAM bytes, throughputs,
occupancy, issue activity, registers, top stall reasons) and, with
--traffic, the per-launch DRAM bytes (read + write) of the forward and
backward pair kernels for bench.py's roofline.traffic.
ncu replays each kernel with cold caches and serialised launches: durations
are for comparison between kernels, not bench numbers.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem pipes % peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "registers"),
    ("smsp__inst_executed.sum", "warp instructions"),
    # pipe utilisation (the north_star's FP32 / SFU evidence): FMA pipe cycles,
    # FMA / XU (MUFU: ex2, rcp, sqrt) / FP64 / ALU / LSU instruction issue
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe cycles %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe inst %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe inst %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe inst %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe cycles %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe inst %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe inst %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared bank conflicts"),
    ("dram__bytes_read.sum.per_second", "DRAM read rate"),
]

ROLE = {"forward32c_kernel": "forward", "forward32_kernel": "forward_tiles",
        "backward32m_kernel": "backward",
        "backward32_kernel": "backward_span", "tail_kernel": "update",
        "tail_tma_kernel": "update_eager", "forward32w_kernel": "render_forward",
        "preprocess_kernel": "preprocess", "emit_kernel": "emit", "emit_warp_kernel": "emit"}


def to_bytes(v: str, unit: str) -> float:
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v.replace(",", "")) * scale.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--traffic", default=None)
    ap.add_argument("--config", type=int, default=3, help="BASELINE config the capture ran")
    args = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", args.report, "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    col = {n: i for i, n in enumerate(head)}
    stalls = [n for n in head if n.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not n.endswith("not_issued")]
    lines = [f"# ncu summary: `{args.report.split('/')[-1]}`", "",
             "Cold-cache, serialised replays (`--set full --clock-control none`): use the",
             "durations to compare kernels, not as bench numbers.", ""]
    traffic: dict = {}
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "").split("::")[-1]
        base = short.split("<")[0]
        lines.append(f"## `{short}`")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for m, label in METRICS:
            if m in col:
                lines.append(f"| {label} | {r[col[m]]} {units[col[m]]} |")
        samp = {n.replace("smsp__pcsamp_warps_issue_stalled_", ""):
                float(r[col[n]].replace(",", "") or 0) for n in stalls}
        tot = sum(samp.values()) or 1.0
        top = sorted(samp.items(), key=lambda x: -x[1])[:5]
        lines.append("| top stalls (% samples) | " +
                     ", ".join(f"{k} {100 * v / tot:.0f}" for k, v in top) + " |")
        lines.append("")
        role = ROLE.get(base)
        if role and "dram__bytes_read.sum" in col and role not in traffic:
            rd = to_bytes(r[col["dram__bytes_read.sum"]], units[col["dram__bytes_read.sum"]])
            wr = to_bytes(r[col["dram__bytes_write.sum"]], units[col["dram__bytes_write.sum"]])
            traffic[role] = rd + wr
            ia = "smsp__issue_active.avg.pct_of_peak_sustained_active"
            if ia in col:
                traffic[role + "_issue_active_pct"] = float(r[col[ia]].replace(",", ""))
    with open(args.out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    if args.traffic:
        traffic["source"] = args.report.split("/")[-1]
        traffic["config"] = args.config
        traffic["what"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch, "
                           "one ncu --set full capture (tools/kbench.py, config 3 LR)")
        with open(args.traffic, "w") as fh:
            json.dump(traffic, fh, indent=1)
    print(f"wrote {args.out}" + (f" and {args.traffic}" if args.traffic else ""))


if __name__ == "__main__":
    main()
