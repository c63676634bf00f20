"""Device timeline of one graph-replayed cold step (EQX_PROF build: EQX_LIB=.../libeqx_b200_prof.so).
Prints microseconds from the drain histogram's first CTA: drain_hist, drain_rank, selection
(windows filled / loop start / loop end) and the side-stream scoring kernel."""
import sys, os, ctypes as C, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2508_16646_b200 import _lib as L
q, led, perf, model, prof, desc = bench.load_inputs(sys.argv[1] if len(sys.argv) > 1 else "cfg2", 0)
sch, clients = bench.make_scheduler(q, led, perf, model, prof, 0)
dev = torch.device("cuda", 0)
cols = dict(client=torch.from_numpy(q["client"]).to(dev), arrival_s=torch.from_numpy(q["arrival"]).to(dev),
            input_tokens=torch.from_numpy(q["in_tokens"]).to(dev), tag=torch.from_numpy(bench.tag_ids(q)).to(dev))
sch.set_batch(0, 0); sch.checkpoint()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
rows = []
for i in range(12):
    sch.restore_async(); (flush.zero_() if not os.environ.get("NOFLUSH") else None); torch.cuda.synchronize()
    sch.drain_step_async(1.0, **cols); r = sch.collect(with_events=False)
    out = (C.c_double * 27)()
    L.load().eqx_phase_times(sch._ctx, out, 27)
    s0 = out[22]
    rows.append([out[17], out[19], out[20], out[23], out[24], s0, s0 + out[1], s0 + out[2], s0 + out[3], s0 + out[4],
                 s0 + out[5], s0 + out[8] * 1e-3, s0 + out[9] * 1e-3, s0 + out[10] * 1e-3, out[25], out[26]])
a = np.median(np.array(rows[2:]), axis=0)
names = ["hist_end", "rank_start", "rank_end", "window_start", "window_end", "select_start", "windows_filled",
         "loop_start", "loop_end", "score_start", "score_end", "sel_lift_done", "sel_ledger_in", "sel_wait_done", "select_done", "event_fill_done"]
print(" ".join(f"{n}={v:.1f}" for n, v in zip(names, a)))
