"""The step's summary (events, batch, length fallbacks, noisy near-ties) reaches the host without a
copy kernel: the selection CTA writes it to the mapped host copy once the side-stream scoring
grid's packed counts are complete (score_counts / SelectArgs::h_st), and the
step's window kernel zeroes those counts.  These cases repeat steps on one context -- split
launches, the graph path, an empty queue (which keeps the copy kernel) in between -- and require
every step's summary to equal the oracle's / a fresh context's."""
import numpy as np
import pytest

import harness as H
from helpers import case_batch, case_clients, case_columns, case_kwargs, compare_step, gpu_run

pytestmark = pytest.mark.gpu


def _scheduler(case):
    from paper_2508_16646_b200 import scheduler as S
    sch = S.GpuScheduler(case_clients(case), running=case.running, **case_kwargs(case))
    sch.set_batch(*case_batch(case))
    sch.checkpoint()
    return sch


def _empty_cols():
    return dict(client=np.zeros(0, np.int32), arrival_s=np.zeros(0, np.float64),
                input_tokens=np.zeros(0, np.int32), tag=np.zeros(0, np.uint8))


@pytest.mark.parametrize("n", [3001, 250_000])
def test_repeated_steps_same_summary(n):
    from test_gpu_parity import _random_case
    case = _random_case(6100 + n % 97, n, 64, pred_kind=H.PRED_MOPE)
    want = H.run_step(case, "oracle")
    assert want["length_fallbacks"] > 0  # untagged rows route through the length fallback
    cols = case_columns(case)
    sch = _scheduler(case)
    for _ in range(3):  # split launches
        sch.restore_async()
        sch.drain(**cols)
        compare_step(sch.step(case.now), sch, want)
    for _ in range(3):  # one graph launch per step
        sch.restore_async()
        sch.drain_step_async(case.now, **cols)
        compare_step(sch.collect(), sch, want)
    sch.restore_async()  # an empty queue: nothing scored, the summary still arrives
    sch.drain(**_empty_cols())
    r0 = sch.step(case.now)
    assert r0.n_admitted == 0 and r0.length_fallbacks == 0 and r0.noisy_near_ties == 0
    sch.restore_async()
    sch.drain(**cols)
    compare_step(sch.step(case.now), sch, want)


def test_noisy_near_ties_per_step():
    """Near-tie counts come from the scoring grid's second packed word: every repeat of the step
    reports the count of a fresh context, not an accumulation."""
    from test_gpu_parity import _random_case
    case = _random_case(6200, 120_000, 31, pred_kind=H.PRED_NOISY)
    _, fresh = gpu_run(case)
    cols = case_columns(case)
    sch = _scheduler(case)
    for graph in (False, True, False, True):
        sch.restore_async()
        if graph:
            sch.drain_step_async(case.now, **cols)
            res = sch.collect()
        else:
            sch.drain(**cols)
            res = sch.step(case.now)
        assert res.noisy_near_ties == fresh.noisy_near_ties
        assert res.n_admitted == fresh.n_admitted and res.n_rejected == fresh.n_rejected
        np.testing.assert_array_equal(res.ids, fresh.ids)


def test_step_ledger_matches_device_ledger():
    """eqx_step_ledger: the ledger the step's selection CTA wrote to mapped host memory equals
    the device ledger read back by eqx_get_clients, on split and graph steps; once the device
    ledger changes (restore, drain) the published copy is refused."""
    from test_gpu_parity import _random_case
    from paper_2508_16646_b200.scheduler import ConfigError
    for C in (64, 1000):
        case = _random_case(6300 + C, 40_000, C, pred_kind=H.PRED_MOPE)
        sch = _scheduler(case)  # finalizes the case
        cols = case_columns(case)
        for graph in (False, True, False):
            sch.restore_async()
            if graph:
                sch.drain_step_async(case.now, **cols)
                sch.collect()
            else:
                sch.drain(**cols)
                sch.step(case.now)
            pub, dev = sch.step_ledger(), sch.ledger()
            for k in dev:
                np.testing.assert_array_equal(pub[k], dev[k], err_msg=k)
        sch.restore_async()
        with pytest.raises(ConfigError):
            sch.step_ledger()
