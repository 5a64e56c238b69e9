"""Every ring-GEMM backend on every shape class, directly against the
reference algorithms (K:206-218 matmul_wrap, K:260-278 conv2d_wrap with the
SPEC:284 pad / stride lowerings, oracle/convops.py), mod 2^59:

* PB_BACKEND_CUDA_CORE -- u64 IMAD tiles (pb_conv.cu, pb_ring.cu; convolutions
  with <= 16 output rows on the skinny column kernel);
* PB_BACKEND_TENSOR   -- tcgen05 kind::i8 on balanced base-256 digit planes
  with the eight partial products in TMEM (pb_tc.cu);
* PB_BACKEND_AUTO     -- what pb_ring_matmul / pb_ring_conv pick.

Shapes include the CIFAR CNN's local terms at batch 64 (>= 2^27 MACs, the
sizes the protocols run), tails in every dimension, the row/column swap of
the tensor path and contractions longer than one CTA's exact int32 range
(split-K with u64 atomics)."""

import numpy as np
import pytest

from oracle import convops as CO
from oracle import kernels as OK
from oracle import ring as OR

pytestmark = pytest.mark.gpu

RING = OR.RingParams()
M59 = np.uint64((1 << 59) - 1)
BACKENDS = (0, 1, 2)  # auto, CUDA core, tensor


def _dev(a):
    from paper_2403_11166_b200 import _dev as D

    return D.u64_to_device(np.ascontiguousarray(a))


def _np(t):
    from paper_2403_11166_b200 import _dev as D

    return D.to_numpy_u64(t).copy()


def _matmul(a, b, n, k, m, ta, tb, backend):
    from paper_2403_11166_b200 import _dev as D
    from paper_2403_11166_b200 import _lib

    out = D.empty_u64(n, m)
    _lib.call("pb_ring_matmul_ex", D.ptr(a), D.ptr(b), n, k, m, ta, tb, 59, D.ptr(out), backend, D.stream())
    return _np(out)


MM_SHAPES = [  # n, k, m
    (128, 784, 64),      # FC-784 local term
    (100, 777, 65),      # tails in all three dimensions
    (5, 300, 200),       # n < m: the tensor path swaps sides
    (1024, 1600, 512),   # 2^29.6 MACs (auto -> tensor)
    (64, 40000, 96),     # K beyond one CTA's exact int32 range: split-K + atomics
]


@pytest.mark.parametrize("shape", MM_SHAPES)
@pytest.mark.parametrize("backend", BACKENDS)
def test_ring_matmul_backends_equal_matmul_wrap(shape, backend):
    n, k, m = shape
    rng = np.random.default_rng(n * 7 + k)
    a = rng.integers(0, 1 << 59, size=(n, k), dtype=np.uint64)
    b = rng.integers(0, 1 << 59, size=(k, m), dtype=np.uint64)
    want = OK.matmul_wrap(a, b) & M59
    assert np.array_equal(_matmul(_dev(a), _dev(b), n, k, m, 0, 0, backend), want)
    if n * k * m <= (1 << 27):  # transposed storage of both operands
        got = _matmul(_dev(a.T.copy()), _dev(b.T.copy()), n, k, m, 1, 1, backend)
        assert np.array_equal(got, want)


def test_ring_matmul_tensor_edge_values():
    """Digits at the balanced-representation boundaries (0x7f / 0x80 bytes,
    all-ones 59-bit values) through the tensor path."""
    n, k, m = 130, 257, 70
    vals = np.array([0, 1, 0x7F, 0x80, 0x7F7F7F7F7F7F7F, 0x80808080808080, (1 << 59) - 1, 1 << 58,
                     0x0123456789ABCDE], dtype=np.uint64)
    rng = np.random.default_rng(9)
    a = vals[rng.integers(0, len(vals), size=(n, k))]
    b = vals[rng.integers(0, len(vals), size=(k, m))]
    want = OK.matmul_wrap(a, b) & M59
    assert np.array_equal(_matmul(_dev(a), _dev(b), n, k, m, 0, 0, 2), want)


CONV_SHAPES = [  # B, c_i, c_o, H, W, s, pad, stride
    (64, 3, 64, 32, 32, 5, 2, 1),    # CIFAR conv1 (B = 64): grad-W K = 65536
    (64, 64, 64, 16, 16, 5, 2, 1),   # CIFAR conv2: 1.68e9 MACs per operator
    (64, 64, 64, 8, 8, 3, 1, 1),     # CIFAR conv3
    (64, 64, 16, 8, 8, 1, 0, 1),     # CIFAR conv5 (1x1)
    (8, 1, 5, 28, 28, 5, 2, 2),      # MNIST conv (stride 2)
    (64, 5, 5, 14, 14, 5, 2, 1),     # MNIST conv2 at B = 64: the skinny kernel (<= 8 rows), split-K grad-W
    (5, 12, 11, 10, 10, 3, 1, 1),    # 9..16 rows (skinny kernel, 16-row accumulators), odd tails
    (3, 5, 7, 9, 9, 3, 1, 2),        # odd tails, stride 2 (square: K conv2d_wrap kernels are s x s)
]


@pytest.mark.parametrize("case", CONV_SHAPES)
@pytest.mark.parametrize("backend", BACKENDS)
def test_ring_conv_backends_equal_conv2d_wrap(case, backend):
    from paper_2403_11166_b200 import _dev as D
    from paper_2403_11166_b200 import _lib

    B, ci, co, H, W, s, p, st = case
    rng = np.random.default_rng(B + ci * 3 + co)
    x = rng.integers(0, 1 << 59, size=(B, ci, H, W), dtype=np.uint64)
    w = rng.integers(0, 1 << 59, size=(co, ci, s, s), dtype=np.uint64)
    y = CO.conv_fwd(x, w, p, st) & M59
    gy = rng.integers(0, 1 << 59, size=y.shape, dtype=np.uint64)
    gx = CO.conv_bwdx(gy, w, H, W, p, st) & M59
    gw = CO.conv_gradw(x, gy, s, p, st) & M59

    def run(kind, a, b, shape):
        out = D.empty_u64(*shape)
        _lib.call("pb_ring_conv_ex", kind, D.ptr(a), D.ptr(b), B, ci, co, H, W, s, p, st, 59, D.ptr(out), backend,
                  D.stream())
        return _np(out)

    assert np.array_equal(run(_lib.CONV_FWD, _dev(x), _dev(w), y.shape), y)
    assert np.array_equal(run(_lib.CONV_BWDX, _dev(gy), _dev(w), gx.shape), gx)
    assert np.array_equal(run(_lib.CONV_GRADW, _dev(x), _dev(gy), gw.shape), gw)


def test_backend_argument_is_checked():
    from paper_2403_11166_b200 import _dev as D
    from paper_2403_11166_b200 import _lib
    from paper_2403_11166_b200.errors import PencilError

    a = _dev(np.ones((4, 4), np.uint64))
    out = D.empty_u64(4, 4)
    with pytest.raises(PencilError):
        _lib.call("pb_ring_matmul_ex", D.ptr(a), D.ptr(a), 4, 4, 4, 0, 0, 59, D.ptr(out), 7, D.stream())
