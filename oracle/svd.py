"""Oracle of the FP16(SVD(rho)) low-rank compressor.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain NumPy in float64; the SVD itself is
the library routine ``numpy.linalg.svd`` (a primitive serving as one step, as the tier rules
allow), everything around it follows the paper's equations in order:

    Eq. 1  A = U S V^T
    Eq. 2  U_r = U[:, 0:r], S_r = S[0:r, 0:r], V_r = V[:, 0:r]   (the
           garbled "U[m,0:r]" read as "all m rows, first r columns")
    Eq. 3  A' = U_r S_r V_r^T
    Eq. 4  R_svd = (m r + r + r n) / (m n)
    Eq. 5  X_compressed = C_FP16(C_SVD(X, r)): each factor to binary16

Readings (R29-R31):
    R29  r = clamp(floor(rho * min(m, n) + 0.5), 1, min(m, n)) — "r is the used ratio of the
         total singular values", "r = max(1, round(rho min(m,n)))"
         with R12's rounding.
    R30  sign convention: the largest-magnitude entry of every U column is
         positive (lowest index on ties); U and V columns flip together.  Thin factors only
         (SPEC.md:92).  A zero singular value leaves its U column unspecified (any unit vector
         completes the basis); the compressor emits 0 there and such columns are excluded
         from comparisons (they do not change A').
    R31  payload: 16-byte preamble {u32 method = 5, u32 m, u32 n, u32 r}, then binary16
         sections zero-padded to 16 bytes: U_r [m][r] row-major, S_r [r], V_r [n][r]
         row-major.  Value bytes / (4 m n) = Eq. 4 / 2 (Table 5's forward column,
         PAPER.md:431-439).  A binary16 overflow of any factor (|sigma| >= 65520) is an
         explicit failure, as for FP16 (R10).
"""
from __future__ import annotations

import math
import struct

import numpy as np

from .codec import NebulaError, OVERFLOW, NONFINITE, pad16

SVD_FP16 = 5

__all__ = ["SVD_FP16", "svd_rank", "svd_payload_bytes", "svd_body_ratio", "svd_factors", "svd_compress",
           "svd_decompress", "svd_decode_factors"]


def svd_rank(m: int, n: int, rho: float) -> int:
    """R29: r = clamp(floor(rho * min(m, n) + 0.5), 1, min(m, n)) in double."""
    k = min(m, n)
    r = math.floor(float(rho) * float(k) + 0.5)
    return max(1, min(k, r))


def svd_payload_bytes(m: int, n: int, r: int) -> int:
    """R31 layout: preamble + pad16(2 m r) + pad16(2 r) + pad16(2 n r)."""
    return 16 + pad16(2 * m * r) + pad16(2 * r) + pad16(2 * n * r)


def svd_body_ratio(m: int, n: int, r: int) -> float:
    """Value bytes over the dense fp32 baseline: 2 (m r + r + r n) / (4 m n) = R_svd / 2."""
    return 2.0 * (m * r + r + r * n) / (4.0 * m * n)


def svd_factors(A: np.ndarray, r: int):
    """Eq. 1-2 with R30's sign convention -> (U_r [m,r], s_r [r], V_r [n,r]) in float64."""
    A = np.asarray(A, dtype=np.float64)
    if A.size and not np.all(np.isfinite(A)):
        raise NebulaError(NONFINITE, "non-finite matrix entry")
    U, s, Vt = np.linalg.svd(A, full_matrices=False)      # Eq. 1 (thin), s descending
    U, s, V = U[:, :r].copy(), s[:r].copy(), Vt[:r, :].T.copy()   # Eq. 2
    for j in range(r):
        if s[j] == 0.0:
            U[:, j] = 0.0
            continue
        i = int(np.argmax(np.abs(U[:, j])))                # first index of the largest |U_ij|
        if U[i, j] < 0:
            U[:, j] = -U[:, j]
            V[:, j] = -V[:, j]
    return U, s, V


def _f16(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        h = np.asarray(x, dtype=np.float64).astype(np.float16)
    if h.size and np.any(np.isinf(h)):
        raise NebulaError(OVERFLOW, "an SVD factor overflows binary16 (|x| >= 65520)")
    return h


def svd_compress(A: np.ndarray, r: int) -> bytes:
    """Eq. 5: C_FP16(C_SVD(A, r)) -> R31 payload bytes."""
    A = np.asarray(A, dtype=np.float32)
    m, n = A.shape
    U, s, V = svd_factors(A, r)

    def sec(h):
        b = h.astype("<f2").tobytes()
        return b + bytes(pad16(len(b)) - len(b))
    return struct.pack("<IIII", SVD_FP16, m, n, r) + sec(_f16(U)) + sec(_f16(s)) + sec(_f16(V))


def svd_decode_factors(payload: bytes):
    """R31 payload -> (m, n, r, U_r, s_r, V_r) as float64 (binary16 values are exact)."""
    method, m, n, r = struct.unpack_from("<IIII", payload, 0)
    if method != SVD_FP16:
        raise ValueError(f"not an SVD payload (method {method})")
    o = 16
    U = np.frombuffer(payload, dtype="<f2", count=m * r, offset=o).astype(np.float64).reshape(m, r)
    o += pad16(2 * m * r)
    s = np.frombuffer(payload, dtype="<f2", count=r, offset=o).astype(np.float64)
    o += pad16(2 * r)
    V = np.frombuffer(payload, dtype="<f2", count=n * r, offset=o).astype(np.float64).reshape(n, r)
    return m, n, r, U, s, V


def svd_decompress(payload: bytes) -> np.ndarray:
    """Eq. 3: A' = U_r S_r V_r^T from the binary16 factors, in float64, rounded once to fp32."""
    m, n, r, U, s, V = svd_decode_factors(payload)
    return ((U * s[None, :]) @ V.T).astype(np.float32)
