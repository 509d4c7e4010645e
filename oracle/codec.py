"""Oracle of the compress -> exchange -> decompress-average -> residual step.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain NumPy, single thread,
explicit float32 at every operation.  Readings R1..R25 are DESIGN.md's list (they
are SURVEY.md §8(c) C1..C25, adopted unchanged unless DESIGN.md says otherwise).

Per cluster c, per bucket of n fp32 elements, step t (SURVEY.md §8(c) plain definition):

    method = IDENTITY if t < start_step else codec.method
    p      = fl(g + r)  (lossy methods with error feedback, R15)
    FP16 : h = RNE16(p), error iff any h is +-inf;  D = float(h)      PAPER.md:125-130 Eq.5
    INT8 : m = max|p|, s = fl(m/127) (s := 1 if m == 0 or s == 0)
           q = clamp(rint(fl(p/s)), -127, 127);  D = fl(q*s)
    FP8  : m = max|p|, s = fl(m/448) (s := 1 if m == 0 or s == 0)    PAPER.md:101 "8-bit floating point" (R27)
           c = RNE_E4M3_satfinite(fl(p/s));  D = fl(E4M3(c)*s)
    E5M2 : the same with OFP8 E5M2 (max 57344): s = fl(m/57344)      PAPER.md:101 (R33)
           c = RNE_E5M2_satfinite(fl(p/s));  D = fl(E5M2(c)*s)
    QSGD : INT8's s; x = fl(p/s); q = floor(x) + [u < x - floor(x)]  PAPER.md:63 (QSGD cited; R32)
           u = counter-based SplitMix64 uniform of (seed, step, cluster, bucket, shard, e)
    TOPK : k largest |p| by fp32 bit key, ties -> lower index,        PAPER.md:63, :99 (cited only; R11-R14)
           idx ascending; values f32 | RNE16 | int8 with the INT8 rule
    r_new = fl(p - D)                                                  R15 (error feedback)
    exchange: slot c <- cluster c's payload body
    out   = fl(tree_sum(D_0..D_{P-1}) / P)                             PAPER.md:76 "aggregated"; R16
"""
from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "IDENTITY", "FP16", "INT8", "TOPK", "VAL_F32", "VAL_F16", "VAL_I8",
    "NONFINITE", "OVERFLOW", "NebulaError", "Codec", "select_method", "topk_k",
    "pad16", "payload_bytes", "body_ratio", "fp16_encode", "int8_scale", "int8_quantize",
    "int8_dequantize", "topk_select", "topk_stats", "compress", "decode_payload",
    "tree_sum", "average", "CompressResult", "cluster_step", "oracle_step",
    "hierarchical_step", "svd_ratio", "FP16_OVERFLOW_ABS", "FP8",
    "fp8_e4m3_encode", "fp8_e4m3_decode", "fp8_scale", "FP8_E4M3_MAX",
    "QSGD", "splitmix64", "qsgd_uniforms", "qsgd_quantize",
    "FP8_E5M2", "FP8_E5M2_MAX", "fp8_e5m2_encode", "fp8_e5m2_decode",
]

F32 = np.float32
IDENTITY, FP16, INT8, TOPK, FP8 = 0, 1, 2, 3, 4
QSGD = 6                     # INT8 levels with stochastic rounding (R32); 5 = the SVD payload id
FP8_E5M2 = 7                 # OFP8 E5M2 reading of "8-bit floating point" (R33)
VAL_F32, VAL_F16, VAL_I8 = 0, 1, 2
VALUE_BYTES = {VAL_F32: 4, VAL_F16: 2, VAL_I8: 1}
NONFINITE, OVERFLOW = "NONFINITE", "OVERFLOW"

# R10: RNE to binary16 overflows to +-inf exactly when |p| >= 65520 (= 65504 + half an
# ulp of the top binade, 32/2); [65504, 65520) rounds down to 65504.  Used only in
# messages and pins — the oracle decides overflow from the conversion result itself.
FP16_OVERFLOW_ABS = 65520.0

# R27 (NEXT-4): OCP FP8 E4M3 ("E4M3FN"): 1 sign, 4 exponent bits (bias 7), 3 mantissa bits,
# no infinities, S.1111.111 = NaN, so the largest finite magnitude is 1.75 * 2^8 = 448.
FP8_E4M3_MAX = 448.0

# R33 (NEXT-4): OCP FP8 E5M2: 1 sign, 5 exponent bits (bias 15), 2 mantissa bits, IEEE-style
# infinities (S.11111.00) and NaNs, so the largest finite magnitude is 1.75 * 2^15 = 57344.
FP8_E5M2_MAX = 57344.0


class NebulaError(Exception):
    """Device-detected error of the C ABI (SPEC.md:129 fp16 overflow -> explicit
    failure; SPEC.md:358 non-finite gradient -> step rejected)."""

    def __init__(self, code: str, msg: str = ""):
        super().__init__(f"{code}: {msg}")
        self.code = code


@dataclass(frozen=True)
class Codec:
    """SPEC.md:111-122 CodecMethod/CodecSchedule, extended with TOPK (R11-R14) and
    error feedback (R15)."""
    method: int = INT8
    topk_values: int = VAL_F32
    topk_k: int = 0            # >0: exact k (capped at n); 0: derive from density (R12)
    topk_density: float = 0.01
    error_feedback: bool = True
    start_step: int = 0
    sr_seed: int = 0           # QSGD (R32): seed of the counter-based uniforms


def select_method(codec: Codec, step: int) -> int:
    """SPEC.md:164 'Identity when step < start_step; the schedule's directional method
    otherwise'; PAPER.md:453 'starting using communication compression from step'."""
    return IDENTITY if step < codec.start_step else codec.method


def topk_k(n: int, codec: Codec) -> int:
    """R12: k = clamp(floor(rho*n + 0.5), 1, n) evaluated in double, or the caller's k."""
    if n == 0:
        return 0
    if codec.topk_k > 0:
        return min(int(codec.topk_k), n)
    k = math.floor(float(codec.topk_density) * float(n) + 0.5)
    return max(1, min(n, k))


def pad16(nbytes: int) -> int:
    return (nbytes + 15) // 16 * 16


def payload_bytes(method: int, n: int, k: int = 0, value_type: int = VAL_F32) -> int:
    """R18 body layout: 16-byte preamble {u32 method, u32 count, f32 scale, u32 aux}
    followed by 16-byte-padded sections.  Dense: values[n].  TOPK: idx u32[k], val[k]."""
    if method == IDENTITY:
        return 16 + pad16(4 * n)
    if method == FP16:
        return 16 + pad16(2 * n)
    if method in (INT8, FP8, QSGD, FP8_E5M2):
        return 16 + pad16(n)
    if method == TOPK:
        return 16 + pad16(4 * k) + pad16(VALUE_BYTES[value_type] * k)
    raise ValueError(method)


def body_ratio(method: int, n: int, k: int = 0, value_type: int = VAL_F32) -> float:
    """R19 / Table 5 convention: transmitted value bytes,
    preamble and padding excluded, over the dense 32-bit baseline 4n."""
    if method == IDENTITY:
        b = 4 * n
    elif method == FP16:
        b = 2 * n
    elif method in (INT8, FP8, QSGD, FP8_E5M2):
        b = n
    else:
        b = (4 + VALUE_BYTES[value_type]) * k
    return b / (4.0 * n)


def svd_ratio(m: int, n: int, r: int) -> float:
    """PAPER.md:120-123 Eq. 4: R_svd = (m*r + r + r*n) / (m*n)  (NEXT-1; pinned now)."""
    return (m * r + r + r * n) / (m * n)


# --------------------------------------------------------------------------- codecs
def _check_finite(p: np.ndarray) -> None:
    if p.size and not np.all(np.isfinite(p)):
        raise NebulaError(NONFINITE, "non-finite gradient (+ residual) element")


def fp16_encode(p: np.ndarray) -> np.ndarray:
    """PAPER.md:130 Eq. 5 C_FP16 'converts the 32-bit floating point numbers to 16-bit';
    SPEC.md:127-129: RNE, subnormals kept, overflow is an explicit failure (R10)."""
    with np.errstate(over="ignore"):
        h = p.astype(np.float16)            # IEEE binary32 -> binary16, round-to-nearest-even
    if h.size and np.any(np.isinf(h)):
        bad = float(np.max(np.abs(p)))
        raise NebulaError(OVERFLOW, f"|p| = {bad} >= {FP16_OVERFLOW_ABS} overflows fp16")
    return h


def int8_scale(p: np.ndarray) -> np.float32:
    """SPEC.md:137 'scale = max|X|/127 (scale = 1 if X == 0)'; R3 per bucket, fp32;
    R4: also s := 1 when fl(m/127) underflows to 0."""
    m = np.max(np.abs(p)) if p.size else F32(0.0)
    m = F32(m)
    s = F32(m / F32(127.0))
    if m == F32(0.0) or s == F32(0.0):
        s = F32(1.0)
    return s


def int8_quantize(p: np.ndarray, s: np.float32) -> np.ndarray:
    """SPEC.md:137 'stored value = round(x/scale) clamped to [-127,127]'; R5 ties-to-even,
    R6 IEEE division (not a reciprocal multiply), R7 clamp."""
    q = np.rint(p / F32(s))                  # fl(p/s) in binary32, then round half to even
    return np.clip(q, -127, 127).astype(np.int8)


def int8_dequantize(q: np.ndarray, s: np.float32) -> np.ndarray:
    """R8: D = fl(q * s), one rounding (q is exact in binary32)."""
    return q.astype(F32) * F32(s)


def fp8_scale(p: np.ndarray, fmax: float = FP8_E4M3_MAX) -> np.float32:
    """R27 / R33: per-bucket symmetric scale mapping max|p| onto the largest finite FP8
    magnitude (448 for E4M3, 57344 for E5M2), s = fl(m / fmax); s := 1 if m == 0 or if
    fl(m / fmax) underflows to 0 (the INT8 rule R4 with fmax in place of 127)."""
    m = np.max(np.abs(p)) if p.size else F32(0.0)
    m = F32(m)
    s = F32(m / F32(fmax))
    if m == F32(0.0) or s == F32(0.0):
        s = F32(1.0)
    return s


def fp8_e4m3_encode(x: np.ndarray) -> np.ndarray:
    """R27: binary32 -> E4M3 code bytes, round to nearest, ties to even mantissa, saturating
    to +-448 (no infinities in E4M3); the sign is kept, also when the value rounds to zero.
    Written from the format's definition, in float64 (exact for binary32 inputs): the quantum
    of the binade holding |x| is 2^(max(e, -6) - 3) with e = floor(log2|x|) (-6 = the smallest
    normal exponent; below it the subnormal quantum 2^-9 applies)."""
    x = np.asarray(x, dtype=F32).ravel()
    if x.size and np.any(np.isnan(x)):
        raise NebulaError(NONFINITE, "NaN has no saturating E4M3 code")
    a = np.abs(x.astype(np.float64))
    sign = np.where(np.signbit(x), 0x80, 0).astype(np.int64)
    e = np.frexp(a)[1].astype(np.int64) - 1                 # a = f * 2^e, 1 <= f < 2 (a > 0)
    quantum = np.ldexp(1.0, np.maximum(e, -6) - 3)
    v = np.rint(a / quantum) * quantum                       # RNE on the exact quotient
    v = np.minimum(v, FP8_E4M3_MAX)                          # satfinite
    ev = np.frexp(v)[1].astype(np.int64) - 1
    normal = v >= 2.0 ** -6
    code_sub = (v / 2.0 ** -9).astype(np.int64)              # 0.mmm * 2^-6, mmm = v / 2^-9
    code_norm = ((ev + 7) << 3) | ((v / np.ldexp(1.0, ev - 3)).astype(np.int64) - 8)
    code = np.where(normal, code_norm, code_sub)
    code = np.where(a == 0.0, 0, code)
    return (sign | code).astype(np.uint8)


def fp8_e4m3_decode(c: np.ndarray) -> np.ndarray:
    """E4M3 code bytes -> binary32 (exact: every E4M3 value is a binary32 value)."""
    c = np.asarray(c, dtype=np.uint8).ravel().astype(np.int64)
    s = np.where(c & 0x80, -1.0, 1.0)
    ef, mf = (c >> 3) & 0xF, c & 0x7
    v = np.where(ef == 0, mf * 2.0 ** -9, (8 + mf) * np.ldexp(1.0, ef - 10))
    v = np.where((ef == 0xF) & (mf == 0x7), np.nan, v)
    return (s * v).astype(F32)


def fp8_e5m2_encode(x: np.ndarray) -> np.ndarray:
    """R33: binary32 -> E5M2 code bytes, round to nearest, ties to even mantissa, saturating to
    +-57344 (the satfinite conversion: magnitudes that would round to infinity give the largest
    finite code); the sign is kept, also when the value rounds to zero.  From the format's
    definition, in float64 (exact for binary32 inputs): the quantum of the binade holding |x| is
    2^(max(e, -14) - 2) (-14 = the smallest normal exponent; subnormal quantum 2^-16)."""
    x = np.asarray(x, dtype=F32).ravel()
    if x.size and np.any(np.isnan(x)):
        raise NebulaError(NONFINITE, "NaN has no saturating E5M2 code")
    a = np.abs(x.astype(np.float64))
    sign = np.where(np.signbit(x), 0x80, 0).astype(np.int64)
    with np.errstate(over="ignore", invalid="ignore"):
        e = np.frexp(np.minimum(a, 2.0 ** 20))[1].astype(np.int64) - 1
        quantum = np.ldexp(1.0, np.maximum(e, -14) - 2)
        v = np.rint(np.minimum(a, 2.0 ** 20) / quantum) * quantum     # RNE on the exact quotient
    v = np.minimum(v, FP8_E5M2_MAX)                                   # satfinite
    ev = np.frexp(v)[1].astype(np.int64) - 1
    normal = v >= 2.0 ** -14
    code_sub = (v / 2.0 ** -16).astype(np.int64)                      # 0.mm * 2^-14
    code_norm = ((ev + 15) << 2) | ((v / np.ldexp(1.0, ev - 2)).astype(np.int64) - 4)
    code = np.where(normal, code_norm, code_sub)
    code = np.where(a == 0.0, 0, code)
    return (sign | code).astype(np.uint8)


def fp8_e5m2_decode(c: np.ndarray) -> np.ndarray:
    """E5M2 code bytes -> binary32 (exact); exponent field 31 holds +-inf (mantissa 0) / NaN."""
    c = np.asarray(c, dtype=np.uint8).ravel().astype(np.int64)
    s = np.where(c & 0x80, -1.0, 1.0)
    ef, mf = (c >> 2) & 0x1F, c & 0x3
    v = np.where(ef == 0, mf * 2.0 ** -16, (4 + mf) * np.ldexp(1.0, ef - 17))
    v = np.where(ef == 0x1F, np.where(mf == 0, np.inf, np.nan), v)
    return (s * v).astype(F32)


def fp8_quantize(p: np.ndarray, s: np.float32) -> np.ndarray:
    """R27: c = RNE_E4M3_satfinite(fl(p / s)) — IEEE binary32 division first (as R6)."""
    return fp8_e4m3_encode((p / F32(s)).astype(F32))


def fp8_dequantize(c: np.ndarray, s: np.float32) -> np.ndarray:
    """R27: D = fl(E4M3(c) * s), one rounding."""
    return (fp8_e4m3_decode(c) * F32(s)).astype(F32)


# ------------------------------------------------------------------ QSGD (NEXT-4, R32)
_M64 = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15


def splitmix64(z):
    """SplitMix64 output function of state z (Steele, Lea & Flood 2014): one step of the
    generator whose state is z - gamma, i.e. mix(z + gamma).  Works on Python ints and on
    numpy uint64 arrays (wrapping arithmetic)."""
    if isinstance(z, np.ndarray):
        z = z.astype(np.uint64) + np.uint64(_GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))
    z = (int(z) + _GAMMA) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def qsgd_uniforms(n: int, seed: int, step: int, cluster: int, bucket: int, shard: int = 0) -> np.ndarray:
    """R32 counter-based uniforms in [0, 1) on the 2^-24 grid, two per 64-bit output:
    base = sm(seed ^ sm(step ^ sm(((cluster * 65536 + shard) << 32) | bucket))),
    h_j = sm(base + j * gamma)  (sm = splitmix64; j * gamma wraps mod 2^64),
    u_{2j} = (h_j >> 40) * 2^-24,  u_{2j+1} = ((h_j >> 16) & (2^24 - 1)) * 2^-24."""
    k = (((cluster * 65536 + shard) << 32) | bucket) & _M64
    base = splitmix64(seed ^ splitmix64(step ^ splitmix64(k)))
    e = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(base) + (e >> np.uint64(1)) * np.uint64(_GAMMA)
        h = splitmix64(z)
    bits = np.where((e & np.uint64(1)) == 0, h >> np.uint64(40), (h >> np.uint64(16)) & np.uint64(0xFFFFFF))
    return (bits.astype(np.float64) * 2.0 ** -24).astype(F32)


def qsgd_quantize(p: np.ndarray, s: np.float32, u: np.ndarray) -> np.ndarray:
    """R32 (QSGD, PAPER.md:63 cites it; l-inf normalisation with 127 levels): x = fl(p / s),
    f = floor(x), phi = x - f (exact), q = f + [u < phi], clamped to [-127, 127].
    E[q * s] = p up to the 2^-24 grid of u (unbiased stochastic rounding)."""
    x = (p / F32(s)).astype(F32)
    f = np.floor(x).astype(F32)
    phi = (x - f).astype(F32)
    q = f + (u < phi).astype(F32)
    return np.clip(q, -127, 127).astype(np.int8)


def _keys(p: np.ndarray) -> np.ndarray:
    """R11: selection key = fp32 bit pattern with the sign cleared (|p| order, -0 == +0)."""
    return p.view(np.uint32) & np.uint32(0x7FFFFFFF)


def topk_select(p: np.ndarray, k: int) -> np.ndarray:
    """R11: the k largest |p| (bit key); among equal keys the lower index wins; returned
    indices ascending.  Sort by (key descending, index ascending) and keep the first k."""
    n = p.size
    if k == 0:
        return np.zeros(0, dtype=np.uint32)
    keys = _keys(p).astype(np.int64)
    order = np.lexsort((np.arange(n, dtype=np.int64), -keys))
    return np.sort(order[:k]).astype(np.uint32)


def topk_stats(p: np.ndarray, k: int) -> dict:
    """R25 'ranks': the integer order statistics of the selection — threshold key T
    (key of the k-th selected element), count_above = #{key > T}, need_T = k - count_above
    (how many of the key == T elements, lowest indices first, are taken)."""
    if k == 0:
        return {"k": 0, "threshold": 0, "count_above": 0, "need": 0}
    keys = _keys(p).astype(np.int64)
    order = np.lexsort((np.arange(p.size, dtype=np.int64), -keys))
    T = int(keys[order[k - 1]])
    above = int(np.count_nonzero(keys > T))
    return {"k": k, "threshold": T, "count_above": above, "need": k - above}


# --------------------------------------------------------------------------- payloads
def _preamble(method: int, count: int, scale: float, aux: int) -> bytes:
    return struct.pack("<IIfI", method, count, scale, aux)


def _pad(b: bytes) -> bytes:
    return b + bytes(pad16(len(b)) - len(b))


@dataclass
class CompressResult:
    payload: bytes
    D: np.ndarray                 # decoded dense view of the payload, fp32[n]
    r_new: np.ndarray | None      # residual after the step (None without error feedback)
    method: int
    stats: dict = field(default_factory=dict)


def compress(p: np.ndarray, method: int, codec: Codec, scale=None, uniforms=None) -> tuple[bytes, np.ndarray, dict]:
    """Encode p with ``method`` -> (payload bytes, D = decode(payload), stats).
    ``scale`` overrides the INT8 / FP8 scale (NEXT-3: the exact cluster-wide scale of a
    hierarchical shard, R28); None = the scale of p itself.
    Raises NebulaError(NONFINITE) on NaN/Inf (SPEC.md:32 'all entries finite', :358) and
    NebulaError(OVERFLOW) when an fp16-encoded value overflows."""
    p = np.ascontiguousarray(p, dtype=F32)
    n = p.size
    _check_finite(p)
    if method == IDENTITY:
        return _preamble(IDENTITY, n, 1.0, 0) + _pad(p.tobytes()), p.copy(), {}
    if method == FP16:
        h = fp16_encode(p)
        return _preamble(FP16, n, 1.0, 0) + _pad(h.tobytes()), h.astype(F32), {}
    if method == INT8:
        s = int8_scale(p) if scale is None else F32(scale)
        q = int8_quantize(p, s)
        return (_preamble(INT8, n, float(s), 0) + _pad(q.tobytes()),
                int8_dequantize(q, s), {"scale": float(s)})
    if method == QSGD:
        s = int8_scale(p) if scale is None else F32(scale)
        if uniforms is None:
            raise ValueError("QSGD needs the step's uniforms (qsgd_uniforms)")
        q = qsgd_quantize(p, s, uniforms)
        return (_preamble(QSGD, n, float(s), 0) + _pad(q.tobytes()),
                int8_dequantize(q, s), {"scale": float(s)})
    if method == FP8:
        s = fp8_scale(p) if scale is None else F32(scale)
        c = fp8_quantize(p, s)
        return (_preamble(FP8, n, float(s), 0) + _pad(c.tobytes()),
                fp8_dequantize(c, s), {"scale": float(s)})
    if method == FP8_E5M2:
        # R33: s = fl(m / 57344); c = RNE_E5M2_satfinite(fl(p / s)); D = fl(E5M2(c) * s)
        s = fp8_scale(p, FP8_E5M2_MAX) if scale is None else F32(scale)
        c = fp8_e5m2_encode((p / F32(s)).astype(F32))
        return (_preamble(FP8_E5M2, n, float(s), 0) + _pad(c.tobytes()),
                (fp8_e5m2_decode(c) * F32(s)).astype(F32), {"scale": float(s)})
    if method == TOPK:
        k = topk_k(n, codec)
        idx = topk_select(p, k)
        v = p[idx.astype(np.int64)]
        D = np.zeros(n, dtype=F32)           # +0.0 where not selected (R16)
        scale = F32(1.0)
        if codec.topk_values == VAL_F32:
            vb, dv = v.tobytes(), v
        elif codec.topk_values == VAL_F16:
            h = fp16_encode(v)
            vb, dv = h.tobytes(), h.astype(F32)
        elif codec.topk_values == VAL_I8:
            scale = int8_scale(p)            # R13: max over the bucket (always selected)
            q = int8_quantize(v, scale)
            vb, dv = q.tobytes(), int8_dequantize(q, scale)
        else:
            raise ValueError(codec.topk_values)
        D[idx.astype(np.int64)] = dv
        payload = (_preamble(TOPK, k, float(scale), codec.topk_values)
                   + _pad(idx.astype("<u4").tobytes()) + _pad(vb))
        stats = topk_stats(p, k)
        stats["scale"] = float(scale)
        return payload, D, stats
    raise ValueError(method)


def decode_payload(payload: bytes, n: int) -> np.ndarray:
    """Inverse of the R18 layout -> dense fp32[n] (+0.0 where top-k did not select)."""
    method, count, scale, aux = struct.unpack_from("<IIfI", payload, 0)
    body = memoryview(payload)[16:]
    if method == IDENTITY:
        return np.frombuffer(body, dtype="<f4", count=n).astype(F32)
    if method == FP16:
        return np.frombuffer(body, dtype="<f2", count=n).astype(F32)
    if method == INT8:
        q = np.frombuffer(body, dtype=np.int8, count=n)
        return int8_dequantize(q, F32(scale))
    if method == FP8:
        return fp8_dequantize(np.frombuffer(body, dtype=np.uint8, count=n), F32(scale))
    if method == FP8_E5M2:
        return (fp8_e5m2_decode(np.frombuffer(body, dtype=np.uint8, count=n)) * F32(scale)).astype(F32)
    if method == QSGD:
        return int8_dequantize(np.frombuffer(body, dtype=np.int8, count=n), F32(scale))
    if method == TOPK:
        k = count
        idx = np.frombuffer(body, dtype="<u4", count=k).astype(np.int64)
        vals = body[pad16(4 * k):]
        if aux == VAL_F32:
            dv = np.frombuffer(vals, dtype="<f4", count=k).astype(F32)
        elif aux == VAL_F16:
            dv = np.frombuffer(vals, dtype="<f2", count=k).astype(F32)
        else:
            dv = int8_dequantize(np.frombuffer(vals, dtype=np.int8, count=k), F32(scale))
        D = np.zeros(n, dtype=F32)
        D[idx] = dv
        return D
    raise ValueError(method)


# --------------------------------------------------------------------------- average
def tree_sum(parts: list) -> np.ndarray:
    """R16: fixed pairwise tree over cluster ids: sum(lo,hi) = sum(lo,mid) + sum(mid,hi),
    mid = lo + ceil((hi-lo)/2); every '+' is one binary32 rounding."""
    def rec(lo, hi):
        if hi - lo == 1:
            return np.asarray(parts[lo], dtype=F32)
        mid = lo + (hi - lo + 1) // 2
        return (rec(lo, mid) + rec(mid, hi)).astype(F32)
    return rec(0, len(parts))


def average(payloads: list, n: int) -> np.ndarray:
    """PAPER.md:76 'the gradients are aggregated by the server' / north_star
    'decompressed and averaged': out = fl(tree_sum(decode(payload_c)) / P).  Every
    cluster's own term is decoded from its own payload (R16)."""
    P = len(payloads)
    acc = tree_sum([decode_payload(b, n) for b in payloads])
    return (acc / F32(P)).astype(F32)


# --------------------------------------------------------------------------- steps
def cluster_step(g: np.ndarray, r: np.ndarray | None, codec: Codec, step: int, scale=None,
                 ids: tuple = (0, 0, 0)) -> CompressResult:
    """One cluster's compress with error feedback (R15):
    lossy: p = fl(g + r); payload = C(p); r_new = fl(p - D(C(p))).
    IDENTITY (t < start_step): payload = g, residual untouched."""
    g = np.ascontiguousarray(g, dtype=F32)
    method = select_method(codec, step)
    if method == IDENTITY:
        payload, D, st = compress(g, IDENTITY, codec)
        return CompressResult(payload, D, None if r is None else r.copy(), IDENTITY, st)
    if codec.error_feedback:
        if r is None:
            r = np.zeros_like(g)
        p = (g + np.asarray(r, dtype=F32)).astype(F32)
    else:
        p = g
    u = qsgd_uniforms(p.size, codec.sr_seed, step, ids[0], ids[1], ids[2]) if method == QSGD else None
    payload, D, st = compress(p, method, codec, scale, u)
    r_new = (p - D).astype(F32) if codec.error_feedback else (None if r is None else r.copy())
    return CompressResult(payload, D, r_new, method, st)


def oracle_step(gs: list, rs: list, codec: Codec, step: int, scales=None, bucket: int = 0, shard: int = 0):
    """Whole step for P clusters: compress each cluster, exchange the
    payload bodies (slot c = cluster c), and have every cluster decompress-average all
    P slots.  scales[c] overrides cluster c's INT8/FP8 scale (R28).
    Returns (out, [r_new_c], [payload_c], [stats_c])."""
    if scales is None:
        scales = [None] * len(gs)
    res = [cluster_step(g, r, codec, step, s, (c, bucket, shard))
           for c, (g, r, s) in enumerate(zip(gs, rs, scales))]
    n = np.asarray(gs[0]).size
    out = average([x.payload for x in res], n)
    return out, [x.r_new for x in res], [x.payload for x in res], [x.stats for x in res]


def hierarchical_step(gs: list, rs: list, codec: Codec, step: int, exact_scale: bool = False, bucket: int = 0,
                      exact_topk: bool = False):
    """P clusters x G GPUs (R20, PAPER.md:95 / :288 intra-cluster parallelism + compressed
    inter-cluster hop).  gs[c][l] is GPU l of cluster c's full bucket (n % G == 0);
    rs[c][l] its residual shard.  The cluster gradient is the fp32 mean of its G GPUs
    (sum in GPU order, then / G; tests feed dyadic inputs so any order is exact);
    GPU l codes shard l; peers with the same l exchange; shards are all-gathered.
    exact_scale (NEXT-3, R28): the INT8 / FP8 scale of every shard is the scale of the whole
    cluster bucket p_c = concat_l(p_{c,l}) (max over all G shards) instead of the shard's own.
    exact_topk (NEXT-3, R34; TOPK only): the selection is the top-k of the WHOLE cluster bucket,
    k = k(rho, n) over p_c = concat_l(mean shards) + r_c, instead of k(rho, n/G) per shard: every
    GPU of cluster c holds the cluster's full residual rs[c][l] (identical for all l, n elements)
    and the cluster's one payload; the average is over the P clusters' full-bucket payloads.
    Returns (out, rs_new[c][l], payloads[c][l])."""
    P, G = len(gs), len(gs[0])
    n = np.asarray(gs[0][0]).size
    assert n % G == 0
    m = n // G
    outs, rs_new, pls = [], [[None] * G for _ in range(P)], [[None] * G for _ in range(P)]
    shards = [[None] * G for _ in range(P)]
    for l in range(G):
        for c in range(P):
            acc = np.asarray(gs[c][0][l * m:(l + 1) * m], dtype=F32)
            for j in range(1, G):
                acc = (acc + np.asarray(gs[c][j][l * m:(l + 1) * m], dtype=F32)).astype(F32)
            shards[c][l] = (acc / F32(G)).astype(F32)
    method = select_method(codec, step)
    if exact_topk and codec.method == TOPK:
        # R34: one selection over the whole cluster bucket (the G shards' means, in order)
        full = [np.concatenate([shards[c][l] for l in range(G)]).astype(F32) for c in range(P)]
        out, r_full, pl_full, _ = oracle_step(full, [rs[c][0] for c in range(P)], codec, step, None, bucket, 0)
        return (out, [[r_full[c] for _ in range(G)] for c in range(P)],
                [[pl_full[c] for _ in range(G)] for c in range(P)])
    scales = [None] * P
    if exact_scale and method in (INT8, FP8, QSGD, FP8_E5M2):
        for c in range(P):
            ps = [shards[c][l] if not codec.error_feedback else
                  (shards[c][l] + (np.zeros(m, F32) if rs[c][l] is None else np.asarray(rs[c][l], F32))).astype(F32)
                  for l in range(G)]
            p_c = np.concatenate(ps)
            scales[c] = (fp8_scale(p_c) if method == FP8 else
                         fp8_scale(p_c, FP8_E5M2_MAX) if method == FP8_E5M2 else int8_scale(p_c))
    for l in range(G):
        out_l, r_l, p_l, _ = oracle_step([shards[c][l] for c in range(P)], [rs[c][l] for c in range(P)], codec, step,
                                         scales, bucket, l)
        outs.append(out_l)
        for c in range(P):
            rs_new[c][l] = r_l[c]
            pls[c][l] = p_l[c]
    return np.concatenate(outs).astype(F32), rs_new, pls
