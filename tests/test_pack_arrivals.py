"""CPU: the packed arrival column of eqx_pack_arrivals (include/eqx.h), decoded here by a numpy
restatement of its layout, reproduces every input bit pattern: dense arrivals (6-byte offsets),
arrivals near zero or sparse (raw blocks), and inputs no packed block may hold (negative, -0.0,
NaN, decreasing) -- those blocks are stored raw.  The device unpacking is checked against the
doubles in tests/test_gpu_parity.py::test_packed_arrival_host_columns."""
import numpy as np
import pytest

from paper_2508_16646_b200 import scheduler as S

ALL_ONES = np.uint64(2 ** 64 - 1)


def decode(data: np.ndarray, n: int) -> np.ndarray:
    nb = (n + 255) // 256
    assert int(data[:8].view(np.uint64)[0]) == len(data) or n == 0 and len(data) >= 16
    base = data[8:8 + 8 * nb].view(np.uint64)
    off = data[8 + 8 * nb:8 + 16 * nb].view(np.int64)
    out = np.empty(n, np.uint64)
    for b in range(nb):
        r0, r1 = 256 * b, min(n, 256 * b + 256)
        m, o = r1 - r0, int(off[b])
        assert o % 16 == 0
        if base[b] == ALL_ONES:
            out[r0:r1] = data[o:o + 8 * m].view(np.uint64)
        else:
            lo = data[o:o + 6 * m].reshape(m, 6).astype(np.uint64)
            d = np.zeros(m, np.uint64)
            for j in range(6):
                d |= lo[:, j] << np.uint64(8 * j)
            out[r0:r1] = base[b] + d
    return out


def cases():
    rng = np.random.default_rng(5)
    yield "empty", np.zeros(0)
    for n in (1, 7, 8, 255, 256, 257, 1000):
        yield f"uniform{n}", np.sort(rng.uniform(0, 60, n))
    yield "dense", 10.0 + np.cumsum(rng.exponential(1 / 16000, 100_003))
    yield "from_zero", np.cumsum(rng.exponential(1e-6, 50_000)) - 1e-6 * 0
    yield "bad", np.array([1.0, -1.0, -0.0, np.nan, 2.0, 1.0, np.inf, 0.0])
    yield "normal", rng.normal(size=3000)


@pytest.mark.parametrize("name,a", list(cases()), ids=[c[0] for c in cases()])
def test_roundtrip(name, a):
    p = S.pack_arrivals(a)
    assert p.n == len(a)
    np.testing.assert_array_equal(decode(p.data, len(a)), a.view(np.uint64))


def test_dense_arrivals_take_six_bytes():
    a = 10.0 + np.cumsum(np.random.default_rng(1).exponential(1 / 16000, 1_000_000))
    p = S.pack_arrivals(a)
    assert p.data.nbytes / len(a) < 6.1
