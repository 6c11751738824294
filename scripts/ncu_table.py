"""One row per captured launch of an ncu report: kernel, duration, DRAM bytes,
warp instructions, issue-slot and occupancy figures (ncu -i --page raw --csv)."""
import csv
import io
import subprocess
import sys

want = {"Kernel Name": "kernel", "gpu__time_duration.sum": "ms", "dram__bytes_read.sum": "dram read GB",
        "dram__bytes_write.sum": "dram write GB", "smsp__inst_executed.sum": "warp inst",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "warps active %",
        "sm__inst_issued.avg.pct_of_peak_sustained_active": "issue active %",
        "launch__registers_per_thread": "regs"}
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
idx = {k: hdr.index(k) for k in want if k in hdr}
scale = {"ms": {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0},
         "GB": {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}}
print(" | ".join(want[k] for k in idx))
for r in rows[2:]:
    out = []
    for k, i in idx.items():
        v, u = r[i], units[i]
        lab = want[k]
        if lab == "ms":
            v = f"{float(v.replace(',', '')) * scale['ms'].get(u, 1.0):.4f}"
        elif lab.endswith("GB"):
            v = f"{float(v.replace(',', '')) * scale['GB'].get(u, 1.0):.4f}"
        elif lab == "kernel":
            v = v.split("(")[0].replace("(anonymous namespace)::", "").replace("bmq::", "")
        out.append(v)
    print(" | ".join(out))
