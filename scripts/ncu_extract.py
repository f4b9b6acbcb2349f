"""Summarise one ncu --set full report (first matching launch) as JSON:
duration, DRAM bytes read/written, tensor-pipe and SM activity.
usage: python scripts/ncu_extract.py REPORT.ncu-rep [kernel-substring] > profiles/x.json"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
pick = None
for r in rows[2:]:
    if want in r[hdr.index("Kernel Name")]:
        pick = r
        break
get = lambda k: pick[hdr.index(k)] if k in hdr else None
num = lambda k: float(get(k).replace(",", "")) if get(k) not in (None, "", "n/a") else None
out = {
    "report": rep, "kernel": get("Kernel Name")[:160],
    "duration_us": num("gpu__time_duration.sum") / (1e3 if units[hdr.index("gpu__time_duration.sum")] == "ns" else 1.0),
    "dram_bytes_read": num("dram__bytes_read.sum"), "dram_bytes_write": num("dram__bytes_write.sum"),
    "dram_units": units[hdr.index("dram__bytes_read.sum")],
    "tensor_pipe_active_pct": num("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    "tensor_pipe_active_max_pct": num("sm__pipe_tensor_cycles_active.max.pct_of_peak_sustained_elapsed"),
    "sm_throughput_pct": num("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    "dram_throughput_pct": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    "registers": num("launch__registers_per_thread"), "grid": get("launch__grid_size"),
    "block": get("launch__block_size"),
}
# normalise DRAM to bytes (each column carries its own unit)
SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6}
for k, col in (("dram_bytes_read", "dram__bytes_read.sum"), ("dram_bytes_write", "dram__bytes_write.sum")):
    if out[k] is not None:
        out[k] = int(out[k] * SC.get(units[hdr.index(col)], 1))
del out["dram_units"]
print(json.dumps(out, indent=1))
