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
for i in range(5):
    sch.restore_async(); flush.zero_(); torch.cuda.synchronize()
    sch.drain(**cols); sch.step_async(1.0); r = sch.collect(with_events=False)
    out = (C.c_double * 22)()
    L.load().eqx_phase_times(sch._ctx, out, 22)
    print(r.n_admitted, [round(x, 2) for x in out[:6]], 'batches', out[6], 'seq', out[7], 'cyc gen/sort/verify/commit', list(out[8:12]), 'seq cyc arg/proc/tail/picks', list(out[12:16]), 'drain hist walk/epi rank start/walk/epi us', [round(x,2) for x in out[17:22]])
