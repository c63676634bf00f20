"""Warp-stall samples of one kernel in an ncu report, by reason and by source line (needs
-lineinfo and --import-source): python tools/ncu_stalls.py report.ncu-rep [N]"""
import csv, subprocess, sys
from collections import Counter, defaultdict
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr = "?", None
tot, by_reason, lines = 0, Counter(), defaultdict(Counter)
for rec in csv.reader(out.splitlines()):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].rsplit("/", 1)[-1]
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or not rec[0].isdigit():
        continue
    row = dict(zip(hdr, rec))
    for k, v in row.items():
        if k.startswith("stall_") and "Not Issued" not in k and v not in ("", "-"):
            c = int(float(v))
            if c:
                by_reason[k] += c
                lines[(fname, rec[0], rec[1].strip()[:90])][k] += c
                tot += c
print("total samples", tot)
for k, v in by_reason.most_common(12):
    print(f"  {k:28s} {v:7d} {100.0 * v / tot:5.1f}%")
print()
for key, cnt in sorted(lines.items(), key=lambda kv: -sum(kv[1].values()))[:n]:
    s = sum(cnt.values())
    top = ", ".join(f"{r[6:]}:{c}" for r, c in cnt.most_common(3))
    print(f"{s:6d} {100.0 * s / tot:5.1f}%  {key[0]}:{key[1]:<5} {top:45s} {key[2]}")
