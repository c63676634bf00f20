"""GPU-side timeline of the pipelined host path: copy-stream H2D vs main-stream step."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
q, led, perf, model, prof, desc = bench.load_inputs("cfg2", 0)
sch, clients = bench.make_scheduler(q, led, perf, model, prof, 0)
from paper_2508_16646_b200 import scheduler as S
hosts = [{k: S.pinned_copy(v) for k, v in
          dict(client=q["client"], arrival_s=q["arrival"], input_tokens=q["in_tokens"],
               tag=bench.tag_ids(q)).items()} for _ in range(2)]
sch.set_batch(0, 0); sch.checkpoint()
dev = torch.device("cuda", 0)
ms = torch.cuda.ExternalStream(sch.stream_ptr, device=dev)
cs = torch.cuda.ExternalStream(sch._lib.eqx_ctx_copy_stream(sch._ctx), device=dev)
E = lambda: torch.cuda.Event(enable_timing=True)
t0 = E(); t0.record(ms); torch.cuda.synchronize()
rows = []
sch.stage_async(**hosts[0])
for i in range(12):
    a0, a1, b0, b1 = E(), E(), E(), E()
    h0 = time.perf_counter()
    a0.record(cs)
    if i + 1 < 12: sch.stage_async(**hosts[(i + 1) % 2])
    a1.record(cs)
    sch.restore_async()
    b0.record(ms)
    sch.drain_step_async(1.0, **hosts[i % 2])
    b1.record(ms)
    h1 = time.perf_counter()
    r = sch.collect(with_events=True); sch.ledger()
    h2 = time.perf_counter()
    rows.append((a0, a1, b0, b1, (h1 - h0) * 1e3, (h2 - h1) * 1e3))
torch.cuda.synchronize()
for i, (a0, a1, b0, b1, hs, hw) in enumerate(rows):
    print(f"{i:2d} h2d[{t0.elapsed_time(a0):8.3f},{t0.elapsed_time(a1):8.3f}] step[{t0.elapsed_time(b0):8.3f},{t0.elapsed_time(b1):8.3f}] host submit {hs:.3f} wait {hw:.3f}")
