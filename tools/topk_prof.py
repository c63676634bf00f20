"""Per-phase cycle counters of the top-K selection rounds (instrumented build):
EQX_LIB=paper_2508_16646_b200/libeqx_b200_prof.so python tools/topk_prof.py cfg3"""
import sys, os, ctypes as C, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2508_16646_b200 import _lib as L
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
q, led, perf, model, prof, desc = bench.load_inputs(cfg, 0)
sch, clients = bench.make_scheduler(q, led, perf, model, prof, 0)
dev = torch.device("cuda", 0)
cols = dict(client=torch.from_numpy(q["client"]).to(dev), arrival_s=torch.from_numpy(q["arrival"]).to(dev),
            input_tokens=torch.from_numpy(q["in_tokens"]).to(dev), tag=torch.from_numpy(bench.tag_ids(q)).to(dev))
sch.set_batch(0, 0); sch.checkpoint()
for i in range(3):
    sch.restore_async(); torch.cuda.synchronize()
    sch.drain(**cols); sch.step_async(1.0); r = sch.collect(with_events=False)
    out = (C.c_double * 35)()
    L.load().eqx_phase_times(sch._ctx, out, 35)
    print(cfg, "admitted", r.n_admitted, "loop us", round(out[3] - out[2], 1) if out[3] else None,
          "rounds", out[7], "cycles heads/gather/chain/keys/select/rank/scan/seq", [int(x) for x in out[8:16]], "head loads, head radix, head passes, item passes, item selects, items, verify cycles, segments", [int(x) for x in out[27:35]])
