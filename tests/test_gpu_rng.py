"""The device Philox reproduces numpy's Philox(key=[seed, stream]) bit-for-bit
(R:52-61 SeededRng.uniform_ring), including offsets inside a block."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _np_ring(seed, stream, n, skip=0, ell=59):
    g = np.random.Generator(np.random.Philox(key=[seed, stream]))
    if skip:
        g.integers(0, 1 << ell, size=skip, dtype=np.uint64)
    return g.integers(0, 1 << ell, size=n, dtype=np.uint64)


@pytest.mark.parametrize("seed,stream,n,off", [(2024, 7, 5, 0), (1, 0, 1000, 3), (2**63 + 5, 2**40, 777, 9), (0, 0, 1, 1)])
def test_uniform_ring_matches_numpy(seed, stream, n, off):
    from paper_2403_11166_b200 import _dev, _lib
    from paper_2403_11166_b200.ring import RingParams, SeededRng

    key = np.random.Philox(key=[seed, stream]).state["state"]["key"]  # numpy's own key derivation
    out = _dev.empty_u64(n)
    _lib.call("pb_uniform_ring", _dev.ptr(out), n, int(key[0]), None, int(key[1]), off, 59, _dev.stream())
    assert np.array_equal(_dev.to_numpy_u64(out), _np_ring(seed, stream, n, off))
    # through the SeededRng mirror, interleaving device and host draws
    g = SeededRng(seed, stream)
    ref = np.random.Generator(np.random.Philox(key=[seed, stream]))
    P = RingParams()
    assert np.array_equal(_dev.to_numpy_u64(g.uniform_ring((off,), P)), ref.integers(0, 1 << 59, size=off, dtype=np.uint64))
    assert np.array_equal(g.ternary((7,)), ref.integers(-1, 2, size=7, dtype=np.int64))
    assert np.array_equal(_dev.to_numpy_u64(g.uniform_ring((n,), P)), ref.integers(0, 1 << 59, size=n, dtype=np.uint64))
    assert np.array_equal(g.cbd((5,)), ref.binomial(20, 0.5, 5).astype(np.int64) - ref.binomial(20, 0.5, 5).astype(np.int64))
    assert np.array_equal(_dev.to_numpy_u64(g.uniform_ring((3,), P)), ref.integers(0, 1 << 59, size=3, dtype=np.uint64))


def test_share_matches_numpy():
    from paper_2403_11166_b200 import _dev, _lib

    rng = np.random.default_rng(0)
    x = rng.integers(0, 1 << 59, size=333, dtype=np.uint64)
    mo, do = _dev.empty_u64(333), _dev.empty_u64(333)
    dx = _dev.u64_to_device(x)
    _lib.call("pb_share", _dev.ptr(dx), 333, 99, None, 3, 0, 59, _dev.ptr(mo), _dev.ptr(do), _dev.stream())
    r = _np_ring(99, 3, 333)
    assert np.array_equal(_dev.to_numpy_u64(mo), r)
    assert np.array_equal(_dev.to_numpy_u64(do), (x - r) & np.uint64((1 << 59) - 1))
