"""Per-call host wall times inside bench.py's pipelined e2e loop (cfg2, narrow + packed host
batches staged two ahead): python tools/e2e_calls.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2508_16646_b200 import scheduler as S
q, led, perf, model, prof, desc = bench.load_inputs("cfg2", 0)
sch, clients = bench.make_scheduler(q, led, perf, model, prof, 0)
sch.set_batch(0, 0); sch.checkpoint()
arr = S.pack_arrivals(q["arrival"])
hosts = [{k: S.pinned_copy(v) for k, v in dict(client=q["client"].astype(np.uint16), arrival_s=arr,
          input_tokens=q["in_tokens"].astype(np.uint16), tag=bench.tag_ids(q)).items()} for _ in range(3)]
names = ("stage", "restore", "drain_step", "collect", "ledger")
def loop(steps, acc=None):
    for i in range(min(2, steps)):
        sch.stage_async(**hosts[i])
    for i in range(steps):
        t = [time.perf_counter()]
        if i + 2 < steps:
            sch.stage_async(**hosts[(i + 2) % 3])
        t.append(time.perf_counter())
        sch.restore_async(); t.append(time.perf_counter())
        sch.drain_step_async(1.0, **hosts[i % 3]); t.append(time.perf_counter())
        sch.collect(with_events=True); t.append(time.perf_counter())
        (sch.step_ledger() if os.environ.get("STEP_LEDGER") else sch.ledger()); t.append(time.perf_counter())
        if acc is not None:
            for k, n in enumerate(names):
                acc[n] += t[k + 1] - t[k]
loop(20)
acc = {n: 0.0 for n in names}
N = 100
torch.cuda.synchronize(); t0 = time.perf_counter()
loop(N, acc)
torch.cuda.synchronize(); t1 = time.perf_counter()
print("step ms", round((t1 - t0) * 1e3 / N, 4), {k: round(v * 1e3 / N, 4) for k, v in acc.items()})
