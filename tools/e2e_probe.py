"""Probe of the host path: H2D bandwidth, per-call host costs, pipelined vs serial steps."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
q, led, perf, model, prof, desc = bench.load_inputs("cfg2", 0)
sch, clients = bench.make_scheduler(q, led, perf, model, prof, 0)
hosts = [{k: torch.from_numpy(v.copy()).pin_memory() for k, v in
          dict(client=q["client"], arrival_s=q["arrival"], input_tokens=q["in_tokens"],
               tag=bench.tag_ids(q)).items()} for _ in range(2)]
dev = {k: torch.empty_like(v, device="cuda") for k, v in hosts[0].items()}
sch.set_batch(0, 0); sch.checkpoint()
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for k in dev: dev[k].copy_(hosts[0][k], non_blocking=True)
    torch.cuda.synchronize(); print("h2d 17MB ms", (time.perf_counter() - t0) * 1e3)
def tm(f, n=20):
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) * 1e3 / n
print("restore", tm(lambda: sch.restore_async()))
print("drain(host)+sync", tm(lambda: (sch.drain(**hosts[0]), torch.cuda.synchronize())))
print("stage only", tm(lambda: (sch.stage_async(**hosts[0]), torch.cuda.synchronize())))
print("step(events)", tm(lambda: sch.step(1.0, with_events=True)))
print("step(no events)", tm(lambda: sch.step(1.0, with_events=False)))
print("ledger", tm(lambda: sch.ledger()))
def serial():
    sch.restore_async(); sch.drain(**hosts[0]); sch.step(1.0); sch.ledger()
print("serial step", tm(serial))
st = {"i": 0}
def piped():
    i = st["i"]; st["i"] += 1
    sch.stage_async(**hosts[(i + 1) % 2]); sch.restore_async(); sch.drain_step_async(1.0, **hosts[i % 2]); sch.collect(); sch.ledger()
sch.stage_async(**hosts[0])
print("pipelined step", tm(piped))
# per-call wall times inside the pipelined loop
acc = {k: 0.0 for k in ("stage", "restore", "drain", "step", "ledger")}
N = 20
for i in range(N):
    t = time.perf_counter(); sch.stage_async(**hosts[(i + 1) % 2]); t1 = time.perf_counter(); acc["stage"] += t1 - t
    sch.restore_async(); t2 = time.perf_counter(); acc["restore"] += t2 - t1
    sch.drain(**hosts[i % 2]); t3 = time.perf_counter(); acc["drain"] += t3 - t2
    sch.step(1.0); t4 = time.perf_counter(); acc["step"] += t4 - t3
    sch.ledger(); t5 = time.perf_counter(); acc["ledger"] += t5 - t4
print({k: round(v * 1e3 / N, 4) for k, v in acc.items()})
print("pinned?", hosts[0]["client"].is_pinned(), hosts[1]["arrival_s"].is_pinned())
