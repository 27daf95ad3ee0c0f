"""One-screen summary of `ncu --set full` reports: time, instructions, issue, pipes,
DRAM bytes, registers, top stall reasons per issue.

  python tools/ncu_full_summary.py REPORT.ncu-rep [...]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time (us)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    unit = dict(zip(hdr, units))
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(f"== {d['Kernel Name'][:90]}")
        for k, label in KEYS:
            if k in d:
                print(f"   {label:20s} {d[k]} {unit.get(k, '')}")
        st = [(k, float(d[k] or 0)) for k in hdr
              if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")]
        st.sort(key=lambda x: -x[1])
        print("   stalls per issue   " + ", ".join(
            f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {v:.2f}"
            for k, v in st[:6]))


for p in sys.argv[1:]:
    print(f"### {p}")
    summarise(p)
