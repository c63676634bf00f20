"""CPU: the C-ABI library builds for sm_100a, loads, and exports every symbol eqx.h declares.
No compute calls are made here (no GPU in this container)."""
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2508_16646_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "eqx.h")).read()
    return sorted(set(re.findall(r"\b(eqx_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = L.load()
    decl = declared_symbols()
    assert decl == L.EXPORTED
    for name in decl:
        assert hasattr(lib, name), name
    assert lib.eqx_abi_version() == 3


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(8\d|9\d)", out)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2508_16646_b200 import scheduler as S
    prof = S.GpuProfile([S.ProfileEntry(32, 1.0, 0.5, 100.0)])
    with pytest.raises(S.EngineError):
        S.GpuScheduler([S.ClientState("a")], profile=prof, predictor="oracle")


def test_scalar_helpers_match_reference_known_answers():
    lib = L.load()
    assert lib.eqx_ufc_increment(1.0, 100, 400, 0.0, 0.0, 0.1, 4.0) == 1700.0
    assert lib.eqx_ufc_increment(1.0, 100, 400, 5.0, 5000.0, 0.1, 4.0) == 850.0
    assert lib.eqx_rfc_increment(1.0, 1000.0, 0.9) == 900.0


@pytest.mark.gpu
def test_pinned_host_arena():
    import torch
    from paper_2508_16646_b200 import scheduler as S
    a = S.pinned_empty((3, 1000), np.float64)
    a[...] = np.arange(3000).reshape(3, 1000)
    t = torch.from_numpy(a)
    d = t.to("cuda", non_blocking=True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(d.cpu().numpy(), a)
    b = S.pinned_copy(np.arange(5, dtype=np.int32))
    assert b.dtype == np.int32 and list(b) == [0, 1, 2, 3, 4]
    lib = S.L.load()
    assert lib.eqx_host_free(None) == 0
    assert lib.eqx_host_alloc(0) is None


@pytest.mark.gpu
def test_context_teardown_frees_device_memory():
    """eqx_ctx_destroy frees every device buffer a context grew (drain, step, live queue, replay
    and staging buffers): 30 create / use / destroy cycles leave the free device memory where it
    was (compute-sanitizer's leak report at exit lists only objects still alive then)."""
    import gc

    import torch
    from helpers import case_batch, case_clients, case_columns, case_kwargs
    from test_gpu_parity import _random_case
    from paper_2508_16646_b200 import scheduler as S
    case = _random_case(77, 20000, 300)
    case.finalize()
    cols = case_columns(case)

    def cycle():
        sch = S.GpuScheduler(case_clients(case), running=case.running, **case_kwargs(case))
        sch.set_batch(*case_batch(case))
        sch.stage_async(**{k: S.pinned_copy(v) for k, v in cols.items()})
        sch.drain(**cols)
        sch.step(case.now)
        sch.close()

    cycle()
    torch.cuda.synchronize()
    gc.collect()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(30):
        cycle()
    torch.cuda.synchronize()
    gc.collect()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 < 8 << 20, f"{(free0 - free1) >> 20} MiB not returned"
