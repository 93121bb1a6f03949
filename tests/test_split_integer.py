"""The split-integer (Ozaki) product behind the WNNM apply kernel
(csrc/wnnm.cu apply_oz_kernel), restated in numpy: base-256 balanced digits
from one fused multiply-add with the 1.5*2^52 + bias constant, int8 digit
products accumulated exactly per level k + l <= 5, adjacent levels joined in
int32, rounding into the 2^frac_bits fixed-point numerator. CPU-only checks
of the arithmetic the kernel relies on (exact reconstruction, int32 headroom,
error against the fp64 product); the kernel itself is checked against the
SVD oracle in tests/test_gpu_parity.py."""

import numpy as np
import pytest

MAGIC = 6755399441055744.0 + 141289400074368.0  # 1.5 * 2^52 + 0x808080808080
BITS = 46


def _exp(mx):
    """smallest E >= -60 with |v| < 2^E for every |v| <= mx (oz_exp)"""
    return max(int(np.frexp(mx)[1]), -60) if mx > 0 else -60


def _digits(v, e):
    """six signed base-256 digits, most significant first (oz_digits16)"""
    t = v * 2.0 ** (BITS - e) + MAGIC  # v * 2^k is exact; one rounding, as the DFMA
    b = t.view(np.uint64)
    by = [((b >> np.uint64(8 * k)) & np.uint64(0xFF)).astype(np.int64) - 128 for k in range(6)]
    return by[::-1]


def _apply(M, W, frac):
    em, ew = _exp(np.abs(M).max()), _exp(np.abs(W).max())
    dm, dw = _digits(M, em), _digits(W, ew)
    acc = [np.zeros((M.shape[0], W.shape[1]), np.int64) for _ in range(6)]
    for k in range(6):
        for l in range(6 - k):
            acc[k + l] += dm[k] @ dw[l]
    assert max(np.abs(a).max() for a in acc) < 2 ** 31  # s32 TMEM accumulators
    c = [acc[0] * 256 + acc[1], acc[2] * 256 + acc[3], acc[4] * 256 + acc[5]]
    assert max(np.abs(x).max() for x in c) < 2 ** 31  # int32 level pairs
    r = max(min(60 - 8 - em - ew - frac, 62), 0)  # R = 52 - e_m - e_w - frac_bits
    y = c[0] * 2 ** 32 + c[1] * 2 ** 16 + c[2]
    return ((y + (1 << (r - 1))) >> r) if r > 0 else y, em, ew


@pytest.mark.parametrize("amp,frac", [(1.0, 40), (255.0, 32), (1e-6, 40)])
def test_digits_reconstruct_exactly(amp, frac):
    rng = np.random.default_rng(0)
    v = (rng.random(4096) * 1.5 - 0.25) * amp
    v[:7] = [0.0, amp * 1.4999, -amp * 0.4999, 2.0 ** -70, -0.0, amp, -amp]
    e = _exp(np.abs(v).max())
    d = _digits(v, e)
    assert all(((x >= -128) & (x <= 127)).all() for x in d)
    u = sum(x * 256 ** (5 - k) for k, x in enumerate(d))
    assert np.array_equal(u, np.rint(v * 2.0 ** (BITS - e)).astype(np.int64))


@pytest.mark.parametrize("m,k,amp,frac", [(1536, 64, 1.0, 40), (512, 64, 1.0, 40),
                                          (128, 48, 1.0, 40), (64, 64, 255.0, 32),
                                          (100, 37, 1.0, 40)])
def test_split_product_matches_fp64(m, k, amp, frac):
    rng = np.random.default_rng(m + k)
    M = (rng.random((m, k)) * 1.5 - 0.25) * amp
    M[rng.random((m, k)) < 0.1] = 0.0
    q, _ = np.linalg.qr(rng.standard_normal((k, k)))
    W = (q * rng.random(k)) @ q.T  # V diag(r) V^T, r in [0, 1): |W| <= 1
    got, em, ew = _apply(M, W, frac)
    ref = M @ W * 2.0 ** frac
    # dropped levels <= 5 * 2^(e_m + e_w - 40) per entry (worst case); measured ~1e-12
    bound = 5 * 2.0 ** (em + ew - 40) * 2.0 ** frac + 1.0
    assert np.abs(got - ref).max() <= bound
    assert np.abs(got - ref).max() * 2.0 ** -frac <= 2e-12 * max(amp, 1.0)
