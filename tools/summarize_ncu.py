"""Summarise ncu outputs into profiles/ (run here, on the CPU box, after gpurun brought them back).

  python tools/summarize_ncu.py <launches.csv> <full.ncu-rep> <out_prefix>

Writes <out_prefix>_launches.md (per-kernel share of one step from the launch list) and
<out_prefix>_kernels.md (key counters of the --set full capture), plus
profiles/step_kernel_traffic.json that bench.py reads for roofline.traffic.
"""
import csv
import json
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[i]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    out = []
    for r in rows[i + 1:]:
        out.append((r[ki].split("(")[0].replace("eqx::", "").replace("void ", ""), float(r[vi].replace(",", ""))))
    return out


def main():
    lpath, rep, prefix = sys.argv[1:4]
    L = launches(lpath)
    # the last complete step: from the last flush memset onwards
    ours = [x for x in L if not x[0].startswith("at::")]  # drop the L2-flush memset
    per = defaultdict(list)
    for name, ns in ours:
        per[name].append(ns)
    step_names = list(dict.fromkeys(name for name, _ in ours))  # our kernels, launch order
    lines = ["# Launch list (ncu --metrics gpu__time_duration.sum --clock-control none)", "",
             "Serialised, cold-cache per-launch device times of one cold scheduling step (cfg2: 1M requests,",
             "64 clients).  Inside a real (graph-replayed) step score_kernel runs on a side stream beside the",
             "one-CTA selection loop, lift_kernel is the selection prologue, and drain_rank / window / selection",
             "are chained with programmatic launches, so the shares below are of the serial sum, not of the",
             "step's wall time (tools/graph_timeline.py measures that).", "",
             "| kernel | launches | median us | share of serial step |", "|---|---:|---:|---:|"]
    med = {k: sorted(v)[len(v) // 2] / 1000.0 for k, v in per.items()}
    tot = sum(med.get(k, 0.0) for k in step_names)
    for k in step_names:
        if k in med:
            lines.append(f"| {k} | {len(per[k])} | {med[k]:.1f} | {100 * med[k] / tot:.0f}% |")
    lines.append(f"| serial sum | | {tot:.1f} | 100% |")
    open(prefix + "_launches.md", "w").write("\n".join(lines) + "\n")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    idx = {m: h.index(m) for m, _ in METRICS if m in h}
    kn = h.index("Kernel Name")
    seen = {}
    for r in rows[2:]:
        name = r[kn].split("(")[0].replace("eqx::", "").replace("void ", "")
        if not name.startswith("at::"):
            seen.setdefault(name, r)
    out = ["# ncu --set full (clock-control none), one launch per kernel, cfg2 step", "",
           "| metric | " + " | ".join(seen) + " |", "|---|" + "---|" * len(seen)]
    for m, label in METRICS:
        if m not in idx:
            continue
        out.append(f"| {label} ({units[idx[m]]}) | " + " | ".join(seen[k][idx[m]] for k in seen) + " |")
    open(prefix + "_kernels.md", "w").write("\n".join(out) + "\n")
    if "score_kernel" in seen:
        r = seen["score_kernel"]

        def mb(m):
            v = float(r[idx[m]].replace(",", ""))
            u = units[idx[m]]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

        traffic = mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")
        json.dump({"kernel": "score_kernel", "dram_bytes_per_launch": traffic,
                   "note": "ncu --set full, cold cache; writes may still sit in L2 at kernel end"},
                  open("profiles/step_kernel_traffic.json", "w"), indent=1)
    print(open(prefix + "_launches.md").read())
    print(open(prefix + "_kernels.md").read())


if __name__ == "__main__":
    main()
