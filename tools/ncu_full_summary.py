"""Key metrics per kernel from an ncu --set full report:
python tools/ncu_full_summary.py report.ncu-rep > summary.txt"""
import csv, subprocess, sys

WANT = ["Duration", "Memory Throughput", "DRAM Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Warp Cycles Per Issued Instruction", "Registers Per Thread",
        "Achieved Occupancy", "Issue Slots Busy"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
import io
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
print("kernel | metric | value")
seen = set()
for r in rows[1:]:
    if len(r) <= vi or r[mi] not in WANT:
        continue
    k = r[ki].split("(")[0]
    key = (r[0], k, r[mi], r[ui])
    if key in seen:
        continue
    seen.add(key)
    print(f"{k} | {r[mi]} | {r[vi]} {r[ui]}")
