"""Top SASS instructions by warp-stall samples from `ncu -i X --page source --csv`."""
import csv, sys
r = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hi = next(i for i, x in enumerate(r) if x and x[0] == "Address")
h = r[hi]; ix = {k: i for i, k in enumerate(h)}
c = ix["Warp Stall Sampling (All Samples)"]
sec = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # kernel section of a multi-kernel report
starts = [i for i, x in enumerate(r) if x and x[0] == "Address"]
hi = starts[sec]
end = starts[sec + 1] - 1 if sec + 1 < len(starts) else len(r)
rows = [x for x in r[hi + 1:end] if len(x) == len(h) and x[0] != "Address"]
tot = sum(float(x[c] or 0) for x in rows)
print("total samples", tot, "instructions", len(rows))
order = sorted(range(len(rows)), key=lambda i: -float(rows[i][c] or 0))
for i in order[:n]:
    x = rows[i]
    print(f"{float(x[c]):7.0f} {100*float(x[c])/tot:5.1f}% [{i:5d}] {x[ix['Address']]} {x[ix['Source']][:90]}")
