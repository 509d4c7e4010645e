"""Pins of the FP16(SVD(rho)) oracle (NEXT-1, oracle/svd.py) against what PAPER.md Eq. 1-5,
Table 5, SPEC.md's worked examples and linear algebra fix.  CPU only.  None of these re-calls
numpy.linalg.svd to produce an expected value: matrices are BUILT from known singular values
and orthonormal factors, so the singular values, the Eckart-Young error and the subspaces are
known in closed form."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def built(m, n, sig, seed):
    """A = Q1 diag(sig) Q2^T with Haar-ish orthonormal Q1 [m,k], Q2 [n,k] (QR of Gaussians)."""
    rng = np.random.default_rng(seed)
    k = len(sig)
    Q1, _ = np.linalg.qr(rng.standard_normal((m, k)))
    Q2, _ = np.linalg.qr(rng.standard_normal((n, k)))
    return Q1, np.asarray(sig, np.float64), Q2, (Q1 * np.asarray(sig)[None, :]) @ Q2.T


def test_eq4_ratio_and_payload_size():
    """PAPER.md:121-123 Eq. 4; SPEC.md:80 R(100, 50, 10) = 0.302; body = Eq. 4 / 2 (Eq. 5)."""
    with open(os.path.join(GOLD, "spec_examples.json")) as f:
        spec = json.load(f)
    assert O.svd_ratio(100, 50, 10) == pytest.approx(0.302, abs=1e-12)
    for m, n, r in [(100, 50, 10), (7, 5, 3), (8192, 768, 461), (33, 17, 1)]:
        A = np.random.default_rng(m).standard_normal((m, n)).astype(np.float32)
        pl = O.svd_compress(A, r)
        assert len(pl) == O.svd_payload_bytes(m, n, r) and len(pl) % 16 == 0
        assert O.svd_body_ratio(m, n, r) == pytest.approx(0.5 * O.svd_ratio(m, n, r), rel=1e-15)
    del spec


@pytest.mark.parametrize("rho,table5", [(0.9, 0.45), (0.8, 0.40), (0.7, 0.34), (0.6, 0.30), (0.5, 0.25),
                                        (0.4, 0.20), (0.3, 0.15), (0.2, 0.09)])
def test_table5_forward_column(rho, table5):
    """PAPER.md:431-439 forward ratios of FP16(SVD(rho)) on a tall H^E-shaped matrix (128 x 64
    tokens x 768): within +-0.05 (the paper's shape is unstated)."""
    m, n = 128 * 64, 768
    r = O.svd_rank(m, n, rho)
    assert abs(O.svd_body_ratio(m, n, r) - table5) <= 0.05


def test_rank_rule_R29():
    assert O.svd_rank(512, 48, 0.6) == 29                    # SPEC.md:150 (r = 29)
    assert O.svd_rank(8192, 768, 0.6) == 461
    assert O.svd_rank(10, 10, 0.01) == 1 and O.svd_rank(10, 4, 1.0) == 4


def test_spec_sigma_examples():
    """identity -> sigma [1, 1]; [[1,2],[2,4]] -> sigma [5, 0] (decoded fp16)."""
    _, _, _, _, s, _ = O.svd_decode_factors(O.svd_compress(np.eye(2, dtype=np.float32), 2))
    assert np.array_equal(s, [1.0, 1.0])
    pl = O.svd_compress(np.array([[1, 2], [2, 4]], np.float32), 2)
    _, _, _, U, s, V = O.svd_decode_factors(pl)
    assert s[0] == 5.0 and abs(s[1]) < 1e-6
    # rank-1: r = 1 reconstructs exactly up to binary16 rounding of the factors
    rec = O.svd_decompress(O.svd_compress(np.array([[1, 2], [2, 4]], np.float32), 1))
    assert np.max(np.abs(rec - np.array([[1, 2], [2, 4]]))) <= 5 * 2 * 2.0 ** -11 * 5


@pytest.mark.parametrize("m,n,r", [(64, 40, 10), (200, 30, 30), (50, 80, 20), (8192 // 8, 96, 58)])
def test_singular_values_subspaces_and_eckart_young(m, n, r):
    """Known sigma (well separated): decoded S_r = sigma[:r] to binary16 rounding; V_r spans the
    known top-r right subspace; the fp16-factor reconstruction error is the Eckart-Young tail
    sqrt(sum_{i>r} sigma_i^2) plus the factor rounding."""
    k = min(m, n)
    sig = 10.0 * 0.93 ** np.arange(k)
    Q1, sig, Q2, A = built(m, n, sig, m + n + r)
    A32 = A.astype(np.float32)
    pl = O.svd_compress(A32, r)
    _, _, _, U, s, V = O.svd_decode_factors(pl)
    assert np.all(np.abs(s - sig[:r]) <= sig[:r] * 2.0 ** -11 + 1e-5)
    # subspace: columns of V_r are (up to sign) the known Q2 columns
    for j in range(r):
        c = abs(float(V[:, j] @ Q2[:, j])) / np.linalg.norm(V[:, j])
        assert c > 1 - 1e-3
        c = abs(float(U[:, j] @ Q1[:, j])) / np.linalg.norm(U[:, j])
        assert c > 1 - 1e-3
    # R30 sign convention on the decoded U
    for j in range(r):
        i = int(np.argmax(np.abs(U[:, j])))
        assert U[i, j] > 0 or np.any((np.abs(U[:, j]) == abs(U[i, j])) & (U[:, j] > 0))
    rec = O.svd_decompress(pl).astype(np.float64)
    tail = math.sqrt(float(np.sum(sig[r:] ** 2)))
    err = np.linalg.norm(A32.astype(np.float64) - rec)
    fro = np.linalg.norm(A)
    assert tail - 1e-6 * fro <= err <= tail + 4 * 2.0 ** -11 * fro * math.sqrt(3)


def test_full_rank_and_rank2_roundtrip():
    """rho = 1 is lossless up to binary16 rounding; a rank-2 matrix with r = 2
    round-trips."""
    rng = np.random.default_rng(4)
    A = rng.standard_normal((40, 12)).astype(np.float32)
    rec = O.svd_decompress(O.svd_compress(A, 12))
    assert np.linalg.norm(rec - A) <= 4 * 2.0 ** -11 * np.linalg.norm(A) * math.sqrt(3)
    a, b = rng.standard_normal((2, 40)), rng.standard_normal((2, 12))
    A2 = (np.outer(a[0], b[0]) + np.outer(a[1], b[1])).astype(np.float32)
    rec = O.svd_decompress(O.svd_compress(A2, 2))
    assert np.linalg.norm(rec - A2) <= 4 * 2.0 ** -11 * np.linalg.norm(A2) * math.sqrt(3)


def test_zero_matrix_and_errors():
    rec = O.svd_decompress(O.svd_compress(np.zeros((9, 5), np.float32), 3))
    assert np.all(rec == 0)
    with pytest.raises(O.NebulaError) as e:
        O.svd_compress(np.full((4, 4), 1e5, np.float32), 1)      # sigma = 4e5 overflows binary16
    assert e.value.code == O.OVERFLOW
    bad = np.ones((3, 3), np.float32)
    bad[1, 1] = np.nan
    with pytest.raises(O.NebulaError):
        O.svd_compress(bad, 1)
