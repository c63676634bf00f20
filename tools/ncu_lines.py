"""Top CUDA source lines by warp-stall samples of one kernel in an ncu report (needs -lineinfo):
python tools/ncu_lines.py report.ncu-rep [N]"""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, rows, tot = "?", [], 0
for rec in csv.reader(out.splitlines()):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].rsplit("/", 1)[-1]
        continue
    if rec[0] in ("Function Name", "Line No") or len(rec) < 5:
        continue
    if rec[0].isdigit() and rec[2] == "-":  # source line with aggregated metrics
        s = int(float(rec[4] or 0))
        tot += s
        rows.append((s, f"{fname}:{rec[0]}", rec[1].strip()[:100]))
rows.sort(reverse=True)
print("total samples", tot)
for s, ln, src in rows[:n]:
    print(f"{s:7d} {100.0 * s / max(tot, 1):5.1f}%  {ln:<22} {src}")
