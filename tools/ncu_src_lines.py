"""Development: per-source-line warp-stall samples and instructions of ONE kernel from
`ncu -i rep --page source --csv --print-source cuda,sass --kernel-name ... --launch-count 1`
(file-qualified, unlike ncu_inst_lines.py)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fname, hdr = "?", None
samp, inst, thr, src = collections.Counter(), collections.Counter(), collections.Counter(), {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Name":
        fname = r[1].split("/")[-1]
        hdr = None
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].strip().isdigit():
        continue
    d = dict(zip(hdr, r))
    key = (fname, int(r[0]))
    try:
        samp[key] += int(d.get("Warp Stall Sampling (All Samples)") or 0)
        inst[key] += int(d.get("Instructions Executed") or 0)
        thr[key] += int(d.get("Thread Instructions Executed") or 0)
    except ValueError:
        continue
    src[key] = r[1].strip()[:96]
ts, ti = sum(samp.values()) or 1, sum(inst.values()) or 1
print(f"samples {ts}, warp inst {ti:.3e}, avg threads {sum(thr.values()) / ti:.1f}")
for key, v in samp.most_common(top):
    print(f"{100 * v / ts:5.1f}% samp {100 * inst[key] / ti:5.1f}% inst {thr[key] / max(inst[key], 1):4.1f}thr "
          f"{key[0]}:{key[1]:<5d} {src[key]}")
