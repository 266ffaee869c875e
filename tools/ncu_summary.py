"""Summarise an ncu --set full report (one line of key metrics per kernel) and,
for the linearize kernel, write the DRAM bytes per point-factor used by
bench.py's roofline "traffic" field.  Usage:
  python tools/ncu_summary.py report.ncu-rep out.md [point_factors_of_linearize_launch]"""
import csv
import io
import json
import os
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main(rep, out, pf=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    lines = [f"# ncu --set full summary: {os.path.basename(rep)}", "",
             "| kernel | " + " | ".join(n for _, n in WANT) + " | top stalls (cycles/issue) |",
             "|" + "---|" * (len(WANT) + 2)]
    lin = None
    for r in data:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").split("::")[-1]
        vals = []
        for k, _ in WANT:
            if k in hdr:
                i = hdr.index(k)
                vals.append(f"{r[i]} {units[i]}".strip())
            else:
                vals.append("n/a")
        st = []
        for i, k in enumerate(hdr):
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
                try:
                    st.append((float(r[i]), k.replace("smsp__average_warps_issue_stalled_", "")
                               .replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        st = ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:4])
        lines.append(f"| {name} | " + " | ".join(vals) + f" | {st} |")
        if "k_linearize" in name and lin is None:
            lin = r
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if lin is not None and pf:
        def val(k):
            i = hdr.index(k)
            v = float(lin[i])
            u = units[i]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        b = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        inst = val("smsp__inst_executed.sum")
        def pct(k):
            try:
                return float(lin[hdr.index(k)])
            except (ValueError, IndexError):
                return None
        json.dump({"dram_bytes_per_point_factor": b / pf, "source": os.path.basename(rep),
                   "point_factors": pf, "dram_bytes": b,
                   "warp_instructions_per_point_factor": inst / pf,
                   "fma_pipe_pct": pct("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                   "alu_pipe_pct": pct("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                   "fp64_pipe_pct": pct("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                   "issue_active_pct": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                   "dram_pct_of_peak": pct("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                   "occupancy_pct": pct("sm__warps_active.avg.pct_of_peak_sustained_active"),
                   "duration_ms": float(lin[hdr.index("gpu__time_duration.sum")]) * {
                       "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "us": 1e-3,
                       "ns": 1e-6}.get(units[hdr.index("gpu__time_duration.sum")], float("nan"))},
                  open(os.path.join(os.path.dirname(out), "linearize_dram_bytes_per_pf.json"), "w"),
                  indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else None)
