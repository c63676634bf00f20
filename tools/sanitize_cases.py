"""Small cases of every device path for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): python tools/sanitize_cases.py, under `compute-sanitizer --tool <t>`.  Each case is
checked against its oracle too, so a sanitizer run is also a parity run."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402

import harness as H  # noqa: E402
from helpers import case_from_golden, compare_step, gpu_run, load_golden  # noqa: E402
from test_gpu_parity import _graph_step, _random_case  # noqa: E402


def main():
    which = sys.argv[1:] or ["step", "graph", "sharded", "replay", "live", "feedback", "modes"]
    if "step" in which:  # eqx_drain + eqx_step: sort / hist drain, window, top-K selection, scoring
        for name in ("eqx_max_warm", "reject_stream_backfill", "tight_kv", "noisy"):
            meta, ins, outs = load_golden(name)
            case = case_from_golden(meta, ins)
            sch, res = gpu_run(case)
            compare_step(res, sch, outs, flagged_near_ties=res.noisy_near_ties, row_ids=case.id)
        for seed, C in ((1, 64), (2, 300), (3, 3000)):
            case = _random_case(300 + seed, 6000, C)
            sch, res = gpu_run(case)
            compare_step(res, sch, H.run_step(case, "oracle"))
        print("step ok", flush=True)
    if "graph" in which:  # the CUDA-graph step bench.py times (PDL chain, staged host columns)
        for seed, C in ((4, 64), (5, 700)):
            case = _random_case(400 + seed, 8000, C)
            case.finalize()
            sch, res = _graph_step(case, device_columns=bool(seed % 2), staged=not seed % 2)
            compare_step(res, sch, H.run_step(case, "oracle"))
        print("graph ok", flush=True)
    if "sharded" in which:  # shard export / ingest / unpack + selection over gathered heads
        from test_sharded import compare_sharded, sharded_sim
        case = _random_case(500, 6000, 130)
        res, led, sc, _ = sharded_sim(case, 3, window=2)
        compare_sharded(res, led, sc, H.run_step(case, "oracle"))
        print("sharded ok", flush=True)
    if "replay" in which and H.available("ref"):  # replay_kernel, small and large rosters, whole log
        from test_replay import check_log, poisson_trace, run_log
        for nc in (4, 20):
            traces = [poisson_trace(600 + nc + s, n_clients=nc, rate=150.0, duration=2.0) for s in range(2)]
            want, got = run_log(traces, [0.5, 0.8], duration=[6.0, 6.0], pred_kind=1)
            check_log(want, got)
        print("replay ok", flush=True)
    if "live" in which and H.available("ref"):
        from test_live import test_live_queue_multi_step_vs_reference
        test_live_queue_multi_step_vs_reference(0)
        print("live ok", flush=True)
    if "feedback" in which:
        from test_feedback import FB_NAMES, test_gpu_feedback_matches_golden
        test_gpu_feedback_matches_golden(FB_NAMES[0])
        print("feedback ok", flush=True)
    if "modes" in which:  # the scoring variants
        for k, v in (("EQX_SCORE", "tma"), ("EQX_NO_DIRECT", "1")):
            os.environ[k] = v
            for seed, C in ((6, 40), (7, 1500)):
                case = _random_case(700 + seed, 5000, C)
                sch, res = gpu_run(case)
                compare_step(res, sch, H.run_step(case, "oracle"))
            os.environ.pop(k)
        print("modes ok", flush=True)
    import gc
    gc.collect()  # contexts of finished cases are destroyed (their device buffers freed)
    import torch
    torch.cuda.empty_cache()

if __name__ == "__main__":
    main()
