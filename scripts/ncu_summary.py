"""Summarise an ncu --set full report: one row per kernel launch with duration, DRAM bytes and
throughput, L2 throughput, tensor / XU pipe activity, issue activity. usage: ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
cols = [("Kernel Name", "kernel"), ("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "dram_rd"),
        ("dram__bytes_write.sum", "dram_wr"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor%"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("launch__registers_per_thread", "regs")]
ix = {h: i for i, h in enumerate(hdr)}
print("| " + " | ".join(c[1] for c in cols) + " |")
print("|" + "---|" * len(cols))
for d in data:
    out = []
    for name, short in cols:
        v = d[ix[name]] if name in ix else ""
        u = units[ix[name]] if name in ix else ""
        if short == "kernel":
            v = v.split("(")[0].replace("void ", "").replace("crv::", "")[:28]
        elif short == "us" and u == "ns":
            v = f"{float(v) / 1e3:.1f}"
        elif short == "us" and u == "msecond":
            v = f"{float(v) * 1e3:.1f}"
        elif short in ("dram_rd", "dram_wr"):
            scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
            v = f"{float(v) * scale:.1f} MB"
        elif v:
            try:
                v = f"{float(v):.1f}"
            except ValueError:
                pass
        out.append(v)
    print("| " + " | ".join(out) + " |")
