import sys, os
sys.path[:0] = ["/root/repo", "/root/repo/tests", "/root/repo/oracle"]
import numpy as np
import harness as H
from helpers import gpu_run
from test_gpu_parity import _random_case
for seed in (20,):
    rng = np.random.default_rng(1000 + seed)
    C = int(rng.choice([1, 5, 31, 64, 200, 777, 1500, 3000])); n = int(rng.integers(0, 60000))
    for CC in (C, 1000, 600, 300, 100):
        case = _random_case(seed, n, CC)
        want = H.run_step(case, "oracle")
        sch, res = gpu_run(case)
        ok = len(res.ids) == len(want["ev_id"]) and np.array_equal(res.ids, want["ev_id"])
        print(os.environ.get("EQX_SELECT_MODE"), CC, "ok" if ok else "BAD", res.ids[:10], want["ev_id"][:10])
