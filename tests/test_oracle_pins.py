"""Pins of the CPU oracle against what the paper, SPEC.md and mathematics fix.

CPU only (``-m "not gpu"``).  None of these re-types the oracle's formula: each checks a
printed value (Table 5, SPEC.md worked examples, hand-written IEEE encodings), a closed
form (error bounds, exact rational arithmetic), an invariant (residual identity, EF
telescoping), or brute force (all subsets for top-k).
"""
import itertools
import json
import math
import os
import struct
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
from gradgen import synthetic

GOLD = os.path.join(os.path.dirname(__file__), "golden")
F32 = np.float32


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------- P1: sizes / Table 5
def test_table5_ratio_column():
    t5 = gold("table5_ratios.json")
    for n in (1, 7, 4096, 1 << 20):
        assert O.body_ratio(O.FP16, n) == t5["fp16_ratio"]
        assert O.body_ratio(O.INT8, n) == t5["int8_ratio"]
        assert O.body_ratio(O.IDENTITY, n) == t5["identity_ratio"]
        assert 1.0 - O.body_ratio(O.INT8, n) == t5["int8_traffic_reduction"]


def test_spec_fp16_100x100_body_bytes():
    t5 = gold("table5_ratios.json")
    g = synthetic(100 * 100, 1, "uniform")
    payload, _, _ = O.compress(g, O.FP16, O.Codec(method=O.FP16))
    body = len(payload) - 16          # preamble excluded; 20000 is already 16-aligned
    assert body == t5["spec_fp16_100x100_body_bytes"]


@pytest.mark.parametrize("method", [O.IDENTITY, O.FP16, O.INT8])
@pytest.mark.parametrize("n", [0, 1, 3, 4, 5, 15, 16, 17, 1000, 4099])
def test_dense_payload_size_formula(method, n):
    g = synthetic(n, n, "normal")
    payload, _, _ = O.compress(g, method, O.Codec(method=method))
    per = {O.IDENTITY: 4, O.FP16: 2, O.INT8: 1}[method]
    assert len(payload) == 16 + math.ceil(per * n / 16) * 16 == O.payload_bytes(method, n)
    assert len(payload) % 16 == 0


@pytest.mark.parametrize("vt,vb", [(O.VAL_F32, 4), (O.VAL_F16, 2), (O.VAL_I8, 1)])
@pytest.mark.parametrize("n,rho", [(1, 0.5), (100, 0.01), (1000, 0.1), (4097, 0.25), (333, 1.0)])
def test_topk_payload_size_formula(vt, vb, n, rho):
    codec = O.Codec(method=O.TOPK, topk_values=vt, topk_density=rho)
    k = O.topk_k(n, codec)
    assert k == max(1, min(n, math.floor(rho * n + 0.5)))
    payload, _, st = O.compress(synthetic(n, 3, "normal"), O.TOPK, codec)
    assert len(payload) == 16 + math.ceil(4 * k / 16) * 16 + math.ceil(vb * k / 16) * 16
    assert st["k"] == k


def test_topk_k_config1():
    # config 1 (n = 2^20, rho = 1%) -> k = 10,486
    assert O.topk_k(1 << 20, O.Codec(method=O.TOPK, topk_density=0.01)) == 10486
    assert O.topk_k(10, O.Codec(method=O.TOPK, topk_k=50)) == 10
    assert O.topk_k(10, O.Codec(method=O.TOPK, topk_density=1e-9)) == 1
    assert O.topk_k(0, O.Codec(method=O.TOPK)) == 0


# ----------------------------------------------------------------- P2: SPEC examples
def test_spec_codec_examples():
    ex = gold("spec_examples.json")
    # fp16 0.5 exact
    _, D, _ = O.compress(np.array([ex["fp16_exact"]["x"]], F32), O.FP16, O.Codec(method=O.FP16))
    assert D[0] == ex["fp16_exact"]["decoded"]
    # fp16 1/3 within 2^-11 relative
    third = F32(1) / F32(3)
    _, D, _ = O.compress(np.array([third], F32), O.FP16, O.Codec(method=O.FP16))
    rel = abs(Fraction(float(D[0])) - Fraction(1, 3)) / Fraction(1, 3)
    assert rel <= Fraction(ex["fp16_third"]["max_rel_err"])
    # int8 zeros -> zeros, scale 1
    z = np.zeros(ex["int8_zero"]["n"], F32)
    payload, D, st = O.compress(z, O.INT8, O.Codec())
    assert np.all(D == 0) and st["scale"] == ex["int8_zero"]["scale"]
    # int8 [-1, 1] exact
    _, D, _ = O.compress(np.array(ex["int8_extrema"]["x"], F32), O.INT8, O.Codec())
    assert D.tolist() == ex["int8_extrema"]["decoded"]
    # int8 U[-1,1] 50x50 bound: s/2 with the R9 binary32 slack (1 + 2^-14)
    u = ex["int8_uniform_bound"]
    for seed in range(20):
        g = synthetic(u["m"] * u["n"], seed, "uniform")
        _, D, st = O.compress(g, O.INT8, O.Codec())
        s = st["scale"]
        assert s <= u["bound_scale_half"] * 2 * (1 + 2 ** -20)
        assert np.max(np.abs(g.astype(np.float64) - D)) <= s / 2 * (1 + 2 ** -14)


def test_spec_schedule_examples():
    ex = gold("spec_examples.json")
    for case in ex["schedule"]:
        c = O.Codec(method=O.INT8, start_step=case["start_step"])
        got = O.select_method(c, case["step"])
        assert got == (O.IDENTITY if case["method"] == "IDENTITY" else O.INT8)


def test_spec_svd_ratio_eq4():
    ex = gold("spec_examples.json")["svd_ratio"]
    assert O.svd_ratio(ex["m"], ex["n"], ex["r"]) == pytest.approx(ex["ratio"], abs=1e-15)
    # Eq. 4 by hand: (m r + r + r n) / (m n) as exact rationals, 200 random triples
    rng = np.random.default_rng(0)
    for _ in range(200):
        m, n = (int(x) for x in rng.integers(1, 5000, 2))
        r = int(rng.integers(1, min(m, n) + 1))
        assert O.svd_ratio(m, n, r) == float(Fraction(m * r + r + r * n, m * n))


# ----------------------------------------------------------------- P3: binary16 RNE
def test_fp16_textbook_encodings():
    tb = gold("ieee_binary16.json")
    for case in tb["cases"]:
        x = np.array([float(case["x"])], F32)
        payload, D, _ = O.compress(x, O.FP16, O.Codec(method=O.FP16))
        bits = struct.unpack_from("<H", payload, 16)[0]
        assert bits == int(case["bits"], 16), case
    with pytest.raises(O.NebulaError) as e:
        O.compress(np.array([float(tb["overflow"]["x"])], F32), O.FP16, O.Codec(method=O.FP16))
    assert e.value.code == O.OVERFLOW


def test_fp16_matches_struct_half_and_error_bound():
    # library cross-check (Python's struct 'e' is an independent binary16 RNE) + the
    # RNE error bound |x - h| <= 2^-11 |x| (normal range) / 2^-25 (subnormal range)
    g = np.concatenate([synthetic(100000, 7, "mixed-scale"), synthetic(100000, 8, "normal")])
    g = g[np.abs(g) < 65504].astype(F32)
    payload, D, _ = O.compress(g, O.FP16, O.Codec(method=O.FP16))
    ours = np.frombuffer(payload, dtype="<u2", offset=16, count=g.size)
    ref = np.array([struct.unpack("<H", struct.pack("<e", float(x)))[0] for x in g[:20000]], np.uint16)
    assert np.array_equal(ours[:20000], ref)
    err = np.abs(g.astype(np.float64) - D.astype(np.float64))
    bound = np.maximum(np.abs(g.astype(np.float64)) * 2.0 ** -11, 2.0 ** -25)
    assert np.all(err <= bound)


def test_fp16_overflow_boundary_R10():
    ok = np.array([65504.0, 65519.996, -65519.996], F32)
    _, D, _ = O.compress(ok, O.FP16, O.Codec(method=O.FP16))
    assert np.all(np.abs(D) == 65504.0)
    for bad in (65520.0, -65520.0, 1e30):
        with pytest.raises(O.NebulaError) as e:
            O.compress(np.array([1.0, bad], F32), O.FP16, O.Codec(method=O.FP16))
        assert e.value.code == O.OVERFLOW


# ----------------------------------------------------------------- INT8 closed forms
@pytest.mark.parametrize("kind", ["normal", "model-like", "uniform", "ties", "mixed-scale", "subnormal"])
def test_int8_exact_rational_properties(kind):
    g = synthetic(3000, 11, kind)
    payload, D, st = O.compress(g, O.INT8, O.Codec())
    s = F32(st["scale"])
    m = Fraction(float(np.max(np.abs(g))))
    # scale is m/127 correctly rounded to binary32 (or 1 when m == 0 / underflow, R4)
    if m != 0 and float(s) != 1.0:
        exact = m / 127
        sf = Fraction(float(s))
        nxt = Fraction(float(np.nextafter(s, F32(np.inf))))
        prv = Fraction(float(np.nextafter(s, F32(0))))
        assert abs(sf - exact) <= abs(nxt - exact) and abs(sf - exact) <= abs(prv - exact)
    q = np.frombuffer(payload, dtype=np.int8, offset=16, count=g.size).astype(np.int64)
    assert q.min() >= -127 and q.max() <= 127
    sF = Fraction(float(s))
    for i in range(0, g.size, 7):
        x = Fraction(float(g[i]))
        t = Fraction(float(F32(g[i]) / s))          # one binary32 division
        assert abs(t - x / sF) <= abs(x / sF) * Fraction(1, 2 ** 24)
        qi = int(q[i])
        # nearest integer to the rounded quotient, ties to even (R5)
        assert abs(t - qi) <= Fraction(1, 2) or abs(qi) == 127
        if abs(t - qi) == Fraction(1, 2):
            assert qi % 2 == 0
        # D = q*s correctly rounded (R8)
        d = Fraction(float(D[i]))
        prod = qi * sF
        assert abs(d - prod) <= abs(prod) * Fraction(1, 2 ** 24)


def test_int8_underflow_scale_R4():
    g = synthetic(64, 5, "tiny-max")
    assert 0 < np.max(np.abs(g)) < 127 * 2.0 ** -149
    _, D, st = O.compress(g, O.INT8, O.Codec())
    assert st["scale"] == 1.0 and np.all(D == 0)


def test_int8_golden_bytes_and_ties_to_even():
    for case in gold("payload_layout.json")["cases"]:
        g = np.array(case["g"], F32)
        if case["method"] == O.TOPK:
            codec = O.Codec(method=O.TOPK, topk_k=case["k"], topk_values=case["values"])
        else:
            codec = O.Codec(method=case["method"])
        payload, D, _ = O.compress(g, case["method"], codec)
        assert payload.hex() == case["hex"], case["name"]
        assert np.array_equal(O.decode_payload(payload, g.size), D)


# ----------------------------------------------------------------- P4: residual identity
@pytest.mark.parametrize("kind", ["normal", "model-like", "zipf-rows", "ties", "mixed-scale",
                                  "subnormal", "signed-zero", "uniform", "zeros"])
@pytest.mark.parametrize("method,vt", [(O.FP16, 0), (O.INT8, 0), (O.TOPK, O.VAL_F32),
                                       (O.TOPK, O.VAL_F16), (O.TOPK, O.VAL_I8)])
def test_residual_identity_exact(kind, method, vt):
    """north_star: g = decompress(compress(g)) + r, read with g := p = g + r_prev (R15).
    Holds bit-exactly in binary32 (Sterbenz) and exactly in the rationals."""
    g = synthetic(5000, 21, kind)
    if method in (O.FP16,) or vt == O.VAL_F16:
        g = np.clip(g, -60000, 60000).astype(F32)
    r0 = synthetic(5000, 22, "normal", sigma=1e-3) if kind != "zeros" else np.zeros(5000, F32)
    codec = O.Codec(method=method, topk_values=vt, topk_density=0.1)
    res = O.cluster_step(g, r0, codec, step=1)
    p = (g + r0).astype(F32)
    assert np.array_equal((res.D + res.r_new).astype(F32).view(np.uint32) & 0x7FFFFFFF,
                          p.view(np.uint32) & 0x7FFFFFFF)
    assert np.array_equal((res.D + res.r_new).astype(F32), p)
    idx = np.random.default_rng(0).integers(0, 5000, 300)
    for i in idx:  # exact in the rationals: p - D is representable (no rounding)
        assert Fraction(float(res.r_new[i])) == Fraction(float(p[i])) - Fraction(float(res.D[i]))


# ----------------------------------------------------------------- P5: EF telescoping
@pytest.mark.parametrize("method,vt", [(O.INT8, 0), (O.FP16, 0), (O.TOPK, O.VAL_F32), (O.TOPK, O.VAL_I8)])
def test_error_feedback_telescoping(method, vt):
    """sum_t D_t + r_T == sum_t g_t up to the roundings of the T additions p = g + r.
    A dropped residual (no EF carry) or a wrong sign fails by orders of magnitude."""
    n, T = 4000, 30
    codec = O.Codec(method=method, topk_values=vt, topk_density=0.05)
    r = np.zeros(n, F32)
    sumD = np.zeros(n, np.float64)
    sumg = np.zeros(n, np.float64)
    slack = np.zeros(n, np.float64)
    for t in range(T):
        g = synthetic(n, 100 + t, "model-like")
        p = (g + r).astype(F32)
        slack += np.abs(p.astype(np.float64)) * 2.0 ** -24
        res = O.cluster_step(g, r, codec, step=t)
        sumD += res.D
        sumg += g
        r = res.r_new
    err = np.abs(sumD + r - sumg)
    assert np.all(err <= slack + 1e-30)
    # and the residual is not trivially zero (the codec is lossy)
    assert np.max(np.abs(r)) > 0


# ----------------------------------------------------------------- P6: top-k
def _brute_topk(p, k):
    """max sum |p_i| over all k-subsets; among maximisers the lexicographically smallest
    ascending index tuple (R11 restated as an optimisation problem)."""
    mags = [Fraction(abs(float(x))) for x in p]
    best, best_set = None, None
    for S in itertools.combinations(range(len(p)), k):
        v = sum(mags[i] for i in S)
        if best is None or v > best or (v == best and S < best_set):
            best, best_set = v, S
    return list(best_set)


def test_topk_brute_force_tiny():
    rng = np.random.default_rng(5)
    vals = np.array([0.0, -0.0, 0.5, -0.5, 1.0, -1.0, 2.0, 1e-3, -2.0], F32)
    count = 0
    for trial in range(600):
        n = int(rng.integers(1, 11))
        p = vals[rng.integers(0, vals.size, n)] if trial % 2 else rng.standard_normal(n).astype(F32)
        for k in range(1, n + 1):
            got = O.topk_select(p, k).tolist()
            assert got == _brute_topk(p, k), (p, k)
            count += 1
    assert count > 1500


def test_topk_partition_cross_check_and_stats():
    # an independent selection: threshold from np.partition, ties by index
    for kind in ("model-like", "ties", "zipf-rows", "zeros", "signed-zero"):
        p = synthetic(200000, 9, kind)
        for k in (1, 17, 2000, 50000, 199999, 200000):
            idx = O.topk_select(p, k)
            keys = (p.view(np.uint32) & 0x7FFFFFFF).astype(np.int64)
            T = int(np.partition(keys, keys.size - k)[keys.size - k])
            above = np.flatnonzero(keys > T)
            ties = np.flatnonzero(keys == T)[: k - above.size]
            ref = np.sort(np.concatenate([above, ties]))
            assert np.array_equal(idx.astype(np.int64), ref)
            st = O.topk_stats(p, k)
            assert (st["threshold"], st["count_above"], st["need"]) == (T, above.size, k - above.size)
            assert np.all(np.diff(idx.astype(np.int64)) > 0)


@pytest.mark.parametrize("rho", [0.01, 0.1, 0.5])
def test_topk_contraction_and_lossless(rho):
    p = synthetic(20000, 4, "model-like")
    codec = O.Codec(method=O.TOPK, topk_density=rho, error_feedback=True)
    res = O.cluster_step(p, np.zeros_like(p), codec, 1)
    k = O.topk_k(p.size, codec)
    pn = np.sum(p.astype(np.float64) ** 2)
    rn = np.sum(res.r_new.astype(np.float64) ** 2)
    assert rn <= (1 - k / p.size) * pn * (1 + 1e-12)
    full = O.cluster_step(p, np.zeros_like(p), O.Codec(method=O.TOPK, topk_density=1.0), 1)
    assert np.array_equal(full.D, p) and np.all(full.r_new == 0)


# ----------------------------------------------------------------- P7: averaging
def test_average_special_cases():
    g = synthetic(3000, 1, "model-like")
    for method in (O.FP16, O.INT8, O.TOPK):
        codec = O.Codec(method=method, topk_density=0.1)
        res = O.cluster_step(g, None, codec, 0)
        assert np.array_equal(O.average([res.payload], g.size), res.D)          # P = 1
        for P in (2, 4, 8):                                                     # identical
            assert np.array_equal(O.average([res.payload] * P, g.size), res.D)


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 7, 8])
def test_average_vs_exact_mean_bound_R17(P):
    gs = [synthetic(5000, 40 + c, "model-like") for c in range(P)]
    codec = O.Codec(method=O.IDENTITY)
    out, _, pls, _ = O.oracle_step(gs, [None] * P, codec, 0)
    exact = np.sum(np.array(gs, np.float64), axis=0) / P
    depth = max(1, math.ceil(math.log2(P))) + 1
    bound = depth * 2.0 ** -24 * np.sum(np.abs(np.array(gs, np.float64)), axis=0) / P
    assert np.all(np.abs(out - exact) <= bound + 1e-45)
    # dyadic inputs: the tree mean is the exact mean (catches a wrong divisor / lost term)
    ints = [np.random.default_rng(c).integers(-2000, 2000, 777).astype(F32) * F32(2.0 ** -10) for c in range(P)]
    out2, _, _, _ = O.oracle_step(ints, [None] * P, codec, 0)
    ex2 = np.sum(np.array(ints, np.float64), axis=0) / P
    if P & (P - 1) == 0:
        assert np.array_equal(out2.astype(np.float64), ex2)
    else:
        assert np.all(np.abs(out2 - ex2) <= np.abs(ex2) * 2.0 ** -24)


def test_tree_order_R16():
    # the fixed tree is ((a+b)+(c+d)) for P = 4 and ((a+b)+c) for P = 3; a sequential
    # sum differs on this input, so a reordering would be caught
    a, b, c, d = F32(1.0), F32(2.0 ** -24), F32(2.0 ** -24), F32(-1.0)
    assert O.tree_sum([np.array([a]), np.array([b]), np.array([c]), np.array([d])])[0] == ((a + b) + (c + d))
    seq = ((a + b) + c) + d
    assert ((a + b) + (c + d)) != seq
    assert O.tree_sum([np.array([a]), np.array([b]), np.array([c])])[0] == (a + b) + c


def test_topk_average_signed_zero_R16():
    # a cluster that did not select i contributes +0.0; -0.0 + +0.0 = +0.0 (IEEE)
    p0 = np.array([-0.0, 5.0], F32)
    p1 = np.array([-0.0, 1.0], F32)
    codec = O.Codec(method=O.TOPK, topk_k=1, error_feedback=False)
    out, _, _, _ = O.oracle_step([p0, p1], [None, None], codec, 0)
    assert out[0] == 0 and not np.signbit(out[0]) and out[1] == 3.0


# ----------------------------------------------------------------- schedule + EF gate
def test_start_step_gate_leaves_residual():
    g = synthetic(1000, 3, "model-like")
    codec = O.Codec(method=O.INT8, start_step=5)
    r = np.zeros_like(g)
    res = O.cluster_step(g, r, codec, 4)
    assert res.method == O.IDENTITY and np.array_equal(res.D, g) and np.all(res.r_new == 0)
    res = O.cluster_step(g, r, codec, 5)
    assert res.method == O.INT8 and np.max(np.abs(res.r_new)) > 0


def test_nonfinite_rejected():
    for method in (O.IDENTITY, O.FP16, O.INT8, O.TOPK):
        for bad in (np.nan, np.inf, -np.inf):
            g = synthetic(100, 1, "normal")
            g[37] = bad
            with pytest.raises(O.NebulaError) as e:
                O.cluster_step(g, np.zeros_like(g), O.Codec(method=method), 0)
            assert e.value.code == O.NONFINITE


# ----------------------------------------------------------------- hierarchical (R20)
def test_hierarchical_identity_is_exact_global_mean():
    P, G, n = 2, 4, 4096
    rng = np.random.default_rng(3)
    gs = [[rng.integers(-1000, 1000, n).astype(F32) * F32(2.0 ** -12) for _ in range(G)] for _ in range(P)]
    rs = [[None] * G for _ in range(P)]
    out, _, _ = O.hierarchical_step(gs, rs, O.Codec(method=O.IDENTITY), 0)
    exact = np.sum(np.array(gs, np.float64).reshape(P * G, n), axis=0) / (P * G)
    assert np.array_equal(out.astype(np.float64), exact)


def test_hierarchical_G1_equals_flat():
    gs = [synthetic(3000, c, "model-like") for c in range(4)]
    codec = O.Codec(method=O.INT8)
    flat, rf, pf, _ = O.oracle_step(gs, [None] * 4, codec, 0)
    hier, rh, ph = O.hierarchical_step([[g] for g in gs], [[None] for _ in gs], codec, 0)
    assert np.array_equal(flat, hier)
    assert all(pf[c] == ph[c][0] for c in range(4))


# ----------------------------------------------------------------- FP8 E4M3 (NEXT-4, R27)
def test_fp8_textbook_encodings():
    g = gold("fp8_e4m3.json")
    for case in g["cases"]:
        x = np.array([float(case["x"])], F32)
        code = int(O.fp8_e4m3_encode(x)[0])
        assert code == int(case["code"], 16), case
    # every finite code decodes to the value its bit fields define; the 126 positive finite
    # codes are strictly increasing (a monotone, gap-free table)
    vals = O.fp8_e4m3_decode(np.arange(0, 127, dtype=np.uint8)).astype(np.float64)
    assert vals[0] == 0.0 and vals[-1] == 448.0 and np.all(np.diff(vals) > 0)
    assert np.isnan(O.fp8_e4m3_decode(np.array([0x7F, 0xFF], np.uint8))).all()


def test_fp8_matches_library_conversion():
    """Against an independent implementation: PyTorch's float8_e4m3fn cast (RNE, no
    saturation — so inputs stay inside the finite range, |x| < 464)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(5)
    x = (rng.standard_normal(400000) * np.exp(rng.uniform(-14, 7, 400000))).astype(F32)
    x = x[np.abs(x) < 464]
    ours = O.fp8_e4m3_encode(x)
    lib = torch.from_numpy(x).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    assert np.array_equal(ours, lib)
    # quotients on / next to every E4M3 rounding boundary (gradgen "fp8-ties")
    g = synthetic(50000, 8, "fp8-ties")
    xq = (g / O.fp8_scale(g)).astype(F32)
    xq = xq[np.abs(xq) < 464]
    assert np.array_equal(O.fp8_e4m3_encode(xq), torch.from_numpy(xq).to(torch.float8_e4m3fn).view(torch.uint8).numpy())
    # round trip: decode(encode(v)) == v for every representable v
    vals = O.fp8_e4m3_decode(np.arange(0, 256, dtype=np.uint8))
    fin = ~np.isnan(vals)
    assert np.array_equal(O.fp8_e4m3_decode(O.fp8_e4m3_encode(vals[fin])), vals[fin])


@pytest.mark.parametrize("kind", ["normal", "model-like", "uniform", "ties", "mixed-scale", "subnormal"])
def test_fp8_exact_rational_properties(kind):
    """R27 in the rationals: s = m/448 correctly rounded; c = nearest E4M3 value of the
    rounded quotient t = fl(p/s) (distance to every other finite E4M3 value no smaller,
    ties to an even mantissa); D = c*s correctly rounded."""
    g = synthetic(3000, 12, kind)
    payload, D, st = O.compress(g, O.FP8, O.Codec(method=O.FP8))
    s = F32(st["scale"])
    m = Fraction(float(np.max(np.abs(g))))
    if m != 0 and float(s) != 1.0:
        exact, sf = m / 448, Fraction(float(s))
        for nb in (np.nextafter(s, F32(np.inf)), np.nextafter(s, F32(0))):
            assert abs(sf - exact) <= abs(Fraction(float(nb)) - exact)
    table = [Fraction(float(v)) for v in O.fp8_e4m3_decode(np.arange(0, 127, dtype=np.uint8))]
    codes = np.frombuffer(payload, dtype=np.uint8, offset=16, count=g.size)
    sF = Fraction(float(s))
    for i in range(0, g.size, 11):
        t = Fraction(float(F32(g[i]) / s))
        c = int(codes[i])
        mag = c & 0x7F
        assert (c >> 7) == int(np.signbit(g[i]))
        dist = abs(abs(t) - table[mag])
        best = min(abs(abs(t) - v) for v in table)
        assert dist == best
        if sum(1 for v in table if abs(abs(t) - v) == best) > 1:
            assert mag % 2 == 0                                      # ties -> even mantissa
        d = Fraction(float(D[i]))
        prod = (-1 if c >> 7 else 1) * table[mag] * sF
        assert abs(d - prod) <= max(abs(prod) * Fraction(1, 2 ** 24), Fraction(1, 2 ** 150))  # binary32 subnormal ulp/2


def test_fp8_ratio_and_error_bound():
    """PAPER.md:101 '8-bit floating point ... reduces 75% communication traffic' (body n bytes
    -> 0.25) and the E4M3 relative error 2^-4 of the normal range (2^-10 * s absolute below)."""
    t5 = gold("table5_ratios.json")
    for n in (1, 17, 4096):
        assert 1.0 - O.body_ratio(O.FP8, n) == t5["int8_traffic_reduction"]
        assert O.payload_bytes(O.FP8, n) == 16 + math.ceil(n / 16) * 16
    g = synthetic(20000, 13, "model-like")
    _, D, st = O.compress(g, O.FP8, O.Codec(method=O.FP8))
    s = float(st["scale"])
    err = np.abs(g.astype(np.float64) - D.astype(np.float64))
    bound = np.maximum(np.abs(g.astype(np.float64)) * 2.0 ** -4, s * 2.0 ** -10) * (1 + 2.0 ** -10)
    assert np.all(err <= bound)


@pytest.mark.parametrize("kind", ["normal", "model-like", "zipf-rows", "ties", "subnormal", "signed-zero", "zeros"])
def test_fp8_residual_identity_exact(kind):
    g = synthetic(5000, 23, kind)
    r0 = synthetic(5000, 24, "normal", sigma=1e-3) if kind != "zeros" else np.zeros(5000, F32)
    res = O.cluster_step(g, r0, O.Codec(method=O.FP8), step=1)
    p = (g + r0).astype(F32)
    assert np.array_equal((res.D + res.r_new).astype(F32), p)
    for i in np.random.default_rng(1).integers(0, 5000, 300):
        assert Fraction(float(res.r_new[i])) == Fraction(float(p[i])) - Fraction(float(res.D[i]))


def test_fp8_zero_bucket_and_degenerate_scale():
    _, D, st = O.compress(np.zeros(33, F32), O.FP8, O.Codec(method=O.FP8))
    assert st["scale"] == 1.0 and np.all(D == 0)
    g = synthetic(64, 5, "tiny-max")
    _, D, st = O.compress(g, O.FP8, O.Codec(method=O.FP8))
    assert st["scale"] == 1.0


# ----------------------------------------------------------------- exact cluster scale (NEXT-3, R28)
@pytest.mark.parametrize("method", [O.INT8, O.FP8])
def test_hierarchical_exact_scale(method):
    """With exact_scale every shard of a cluster carries the scale of the WHOLE cluster bucket:
    equal to the flat (G = 1) compress of the concatenated cluster gradient, shard by shard.
    Dyadic inputs make the intra-cluster mean exact in any order."""
    P, G, n = 2, 4, 4096
    rng = np.random.default_rng(9)
    gs = [[(rng.integers(-1000, 1000, n) * (4.0 ** rng.integers(-3, 3, n))).astype(F32) * F32(2.0 ** -12)
           for _ in range(G)] for _ in range(P)]
    codec = O.Codec(method=method)
    out, rs, pls = O.hierarchical_step(gs, [[None] * G for _ in range(P)], codec, 0, exact_scale=True)
    means = [np.sum(np.array(gs[c], np.float64), axis=0) / G for c in range(P)]
    flat_out, flat_r, flat_pl, _ = O.oracle_step([x.astype(F32) for x in means], [None] * P, codec, 0)
    assert np.array_equal(out, flat_out)
    m = n // G
    for c in range(P):
        sc = {struct.unpack_from("<f", pls[c][l], 8)[0] for l in range(G)}
        assert len(sc) == 1 and sc.pop() == struct.unpack_from("<f", flat_pl[c], 8)[0]
        assert np.array_equal(np.concatenate(rs[c]), flat_r[c])
        for l in range(G):
            assert pls[c][l][16:16 + m] == flat_pl[c][16 + l * m:16 + (l + 1) * m]
    # without exact_scale the shards' scales differ (the per-shard reading R20)
    _, _, pls2 = O.hierarchical_step(gs, [[None] * G for _ in range(P)], codec, 0)
    assert len({struct.unpack_from("<f", pls2[0][l], 8)[0] for l in range(G)}) > 1


# ----------------------------------------------------------------- QSGD stochastic rounding (NEXT-4, R32)
def test_splitmix64_reference_output():
    g = gold("splitmix64.json")
    assert O.splitmix64(0) == int(g["seed0_first_output"], 16)
    # the vectorised (numpy uint64) and scalar forms agree
    zs = np.array([0, 1, 2 ** 63, 2 ** 64 - 1, 12345678901234567], dtype=np.uint64)
    assert [int(v) for v in O.splitmix64(zs)] == [O.splitmix64(int(z)) for z in zs]


def test_qsgd_uniforms_are_uniform_and_distinct():
    u = O.qsgd_uniforms(200000, 7, 3, 1, 2).astype(np.float64)
    assert u.min() >= 0 and u.max() < 1 and np.all(u * 2 ** 24 == np.floor(u * 2 ** 24))
    hist, _ = np.histogram(u, bins=64, range=(0, 1))
    chi2 = float(np.sum((hist - u.size / 64) ** 2 / (u.size / 64)))
    assert chi2 < 120                                    # 63 dof: p ~ 1e-5
    for other in [(8, 3, 1, 2), (7, 4, 1, 2), (7, 3, 0, 2), (7, 3, 1, 3)]:
        assert not np.array_equal(u[:64], O.qsgd_uniforms(64, *other).astype(np.float64))
    # the two halves of one 64-bit output (even / odd elements) are uncorrelated
    ev, od = u[0::2] - 0.5, u[1::2] - 0.5
    assert abs(float(np.mean(ev * od))) < 6 * (1 / 12) / math.sqrt(ev.size)
    # the even-element stream is the SplitMix64 stream itself (top 24 bits of each output)
    k = ((1 * 65536 + 0) << 32) | 2
    base = O.splitmix64(7 ^ O.splitmix64(3 ^ O.splitmix64(k)))
    for j in range(4):
        h = O.splitmix64((base + j * 0x9E3779B97F4A7C15) % 2 ** 64)
        assert u[2 * j] == (h >> 40) * 2.0 ** -24 and u[2 * j + 1] == ((h >> 16) & 0xFFFFFF) * 2.0 ** -24


def test_qsgd_rounds_to_neighbours_and_is_unbiased():
    """q in {floor(x), floor(x) + 1}; integer quotients are kept; the mean of the decoded value
    over many seeds converges to p (E[D] = p up to the 2^-24 grid of u)."""
    g = synthetic(4000, 31, "normal")
    s = O.int8_scale(g)
    x = (g / s).astype(F32)
    acc = np.zeros(g.size, np.float64)
    T = 400
    for seed in range(T):
        pl, D, _ = O.compress(g, O.QSGD, O.Codec(method=O.QSGD), uniforms=O.qsgd_uniforms(g.size, seed, 0, 0, 0))
        q = np.frombuffer(pl, np.int8, count=g.size, offset=16).astype(np.float64)
        assert np.all((q == np.floor(x)) | (q == np.floor(x) + 1))
        acc += D
    mean = acc / T
    # Var[D] <= s^2 / 4 per seed -> standard error s / (2 sqrt(T)); 6 sigma over 4000 elements
    assert np.all(np.abs(mean - g) <= 6 * float(s) / (2 * math.sqrt(T)))
    assert abs(float(np.mean(mean - g))) <= 6 * float(s) / (2 * math.sqrt(T * g.size))
    xi = np.array([0.0, 1.0, -3.0, 127.0], F32) * s
    pl, D, _ = O.compress(xi.astype(F32), O.QSGD, O.Codec(method=O.QSGD), uniforms=O.qsgd_uniforms(4, 1, 0, 0, 0))
    assert np.array_equal(np.frombuffer(pl, np.int8, count=4, offset=16), [0, 1, -3, 127])


def test_qsgd_payload_layout_and_ratio():
    g = synthetic(1001, 5, "model-like")
    pl, D, st = O.compress(g, O.QSGD, O.Codec(method=O.QSGD), uniforms=O.qsgd_uniforms(1001, 0, 0, 0, 0))
    assert len(pl) == O.payload_bytes(O.QSGD, 1001) == 16 + O.pad16(1001)
    assert struct.unpack_from("<IIfI", pl, 0) == (O.QSGD, 1001, st["scale"], 0)
    assert np.array_equal(O.decode_payload(pl, 1001), D)
    assert O.body_ratio(O.QSGD, 1001) == 0.25
    # one quantum: |p - D| < s
    assert np.all(np.abs(g.astype(np.float64) - D) < float(st["scale"]) * (1 + 2.0 ** -20))


# ----------------------------------------------------------------- FP8 E5M2 (NEXT-4, R33)
def test_e5m2_textbook_encodings():
    g = gold("fp8_e5m2.json")
    for case in g["cases"]:
        x = np.array([float(case["x"])], F32)
        code = int(O.fp8_e5m2_encode(x)[0])
        assert code == int(case["code"], 16), case
    # the 123 positive finite codes decode to strictly increasing values ending at 57344;
    # exponent field 31 holds infinity (mantissa 0) and NaNs
    vals = O.fp8_e5m2_decode(np.arange(0, 124, dtype=np.uint8)).astype(np.float64)
    assert vals[0] == 0.0 and vals[-1] == 57344.0 and np.all(np.diff(vals) > 0)
    assert np.isinf(O.fp8_e5m2_decode(np.array([0x7C, 0xFC], np.uint8))).all()
    assert np.isnan(O.fp8_e5m2_decode(np.array([0x7D, 0x7E, 0x7F, 0xFF], np.uint8))).all()


def test_e5m2_matches_library_conversion():
    """Against an independent implementation: PyTorch's float8_e5m2 cast (RNE; it overflows to
    infinity instead of saturating, so inputs stay below the 61440 rounding boundary)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(6)
    x = (rng.standard_normal(400000) * np.exp(rng.uniform(-20, 11, 400000))).astype(F32)
    x = x[np.abs(x) < 61440]
    assert np.array_equal(O.fp8_e5m2_encode(x), torch.from_numpy(x).to(torch.float8_e5m2).view(torch.uint8).numpy())
    # every midpoint between neighbouring E5M2 magnitudes, and its binary32 neighbours
    vals = O.fp8_e5m2_decode(np.arange(0, 124, dtype=np.uint8)).astype(np.float64)
    mids = ((vals[:-1] + vals[1:]) / 2).astype(F32)
    for m in (mids, np.nextafter(mids, F32(np.inf)), np.nextafter(mids, F32(0))):
        xm = np.concatenate([m, -m]).astype(F32)
        assert np.array_equal(O.fp8_e5m2_encode(xm), torch.from_numpy(xm).to(torch.float8_e5m2).view(torch.uint8).numpy())
    fin = np.arange(0, 256, dtype=np.uint8)
    v = O.fp8_e5m2_decode(fin)
    ok = np.isfinite(v)
    assert np.array_equal(O.fp8_e5m2_decode(O.fp8_e5m2_encode(v[ok])), v[ok])


@pytest.mark.parametrize("kind", ["normal", "model-like", "uniform", "ties", "mixed-scale", "subnormal"])
def test_e5m2_exact_rational_properties(kind):
    """R33 in the rationals: s = m/57344 correctly rounded; c = nearest E5M2 value of t = fl(p/s)
    (ties to an even mantissa); D = c*s correctly rounded."""
    g = synthetic(3000, 14, kind)
    payload, D, st = O.compress(g, O.FP8_E5M2, O.Codec(method=O.FP8_E5M2))
    s = F32(st["scale"])
    m = Fraction(float(np.max(np.abs(g))))
    if m != 0 and float(s) != 1.0:
        exact, sf = m / 57344, Fraction(float(s))
        for nb in (np.nextafter(s, F32(np.inf)), np.nextafter(s, F32(0))):
            assert abs(sf - exact) <= abs(Fraction(float(nb)) - exact)
    table = [Fraction(float(v)) for v in O.fp8_e5m2_decode(np.arange(0, 124, dtype=np.uint8))]
    codes = np.frombuffer(payload, dtype=np.uint8, offset=16, count=g.size)
    sF = Fraction(float(s))
    for i in range(0, g.size, 11):
        t = Fraction(float(F32(g[i]) / s))
        c = int(codes[i])
        mag = c & 0x7F
        assert (c >> 7) == int(np.signbit(g[i]))
        best = min(abs(abs(t) - v) for v in table)
        assert abs(abs(t) - table[mag]) == best
        if sum(1 for v in table if abs(abs(t) - v) == best) > 1:
            assert mag % 2 == 0
        d = Fraction(float(D[i]))
        prod = (-1 if c >> 7 else 1) * table[mag] * sF
        assert abs(d - prod) <= max(abs(prod) * Fraction(1, 2 ** 24), Fraction(1, 2 ** 150))


def test_e5m2_ratio_error_bound_and_residual_identity():
    """PAPER.md:101 (body n bytes -> ratio 0.25, a 75 % reduction); E5M2's relative error 2^-3
    in the normal range (2^-17 * s absolute below); p == D + r_new bit for bit."""
    t5 = gold("table5_ratios.json")
    for n in (1, 17, 4096):
        assert 1.0 - O.body_ratio(O.FP8_E5M2, n) == t5["int8_traffic_reduction"]
        assert O.payload_bytes(O.FP8_E5M2, n) == 16 + math.ceil(n / 16) * 16
    g = synthetic(20000, 15, "model-like")
    _, D, st = O.compress(g, O.FP8_E5M2, O.Codec(method=O.FP8_E5M2))
    s = float(st["scale"])
    err = np.abs(g.astype(np.float64) - D.astype(np.float64))
    assert np.all(err <= np.maximum(np.abs(g.astype(np.float64)) * 2.0 ** -3, s * 2.0 ** -17) * (1 + 2.0 ** -10))
    for kind in ("normal", "zipf-rows", "subnormal", "signed-zero", "zeros"):
        g = synthetic(5000, 25, kind)
        r0 = synthetic(5000, 26, "normal", sigma=1e-3) if kind != "zeros" else np.zeros(5000, F32)
        res = O.cluster_step(g, r0, O.Codec(method=O.FP8_E5M2), step=1)
        assert np.array_equal((res.D + res.r_new).astype(F32), (g + r0).astype(F32))
    _, D, st = O.compress(np.zeros(33, F32), O.FP8_E5M2, O.Codec(method=O.FP8_E5M2))
    assert st["scale"] == 1.0 and np.all(D == 0)


# ----------------------------------------------------------------- exact cluster-wide top-k (NEXT-3, R34)
def _brute_topk(p, k):
    """Brute force (independent of topk_select's lexsort): repeatedly take the largest |p| key,
    lowest index first among equal keys, k times."""
    keys = (p.view(np.uint32) & 0x7FFFFFFF).astype(np.int64)
    taken = np.zeros(p.size, bool)
    sel = []
    for _ in range(k):
        best = -1
        for i in range(p.size):
            if not taken[i] and (best < 0 or keys[i] > keys[best]):
                best = i
        taken[best] = True
        sel.append(best)
    return sorted(sel)


@pytest.mark.parametrize("vt", [O.VAL_F32, O.VAL_I8])
def test_hierarchical_exact_topk_is_global_selection(vt):
    """R34: the selection is the top-k of the concatenated cluster bucket (brute force over the
    concatenation), not k/G per shard; one shard holding every large value makes the two
    readings differ."""
    P, G, m = 2, 4, 24
    rng = np.random.default_rng(17)
    gs = [[(rng.integers(-50, 50, G * m) * 2.0 ** -6).astype(F32) for _ in range(G)] for _ in range(P)]
    for c in range(P):      # shard 1 of every GPU's bucket carries the large values
        for l in range(G):
            gs[c][l][m:2 * m] *= F32(64.0)
    codec = O.Codec(method=O.TOPK, topk_values=vt, topk_density=0.125)
    out, rs, pls = O.hierarchical_step(gs, [[None] * G for _ in range(P)], codec, 0, exact_topk=True)
    k = O.topk_k(G * m, codec)
    assert k == 12
    for c in range(P):
        p_c = (np.sum(np.array(gs[c], np.float64), axis=0) / G).astype(F32)   # dyadic: exact mean
        idx = np.frombuffer(pls[c][0], dtype="<u4", count=k, offset=16)
        assert list(idx) == _brute_topk(p_c, k)
        assert all(pls[c][l] == pls[c][0] for l in range(G))
        assert np.all(idx >= m) and np.all(idx < 2 * m)          # all from shard 1
        D = O.decode_payload(pls[c][0], G * m)
        assert np.array_equal((D + rs[c][0]).astype(F32), p_c)  # residual identity on the full bucket
    # per-shard reading (R20) selects k/G = 3 per shard instead
    _, _, pls2 = O.hierarchical_step(gs, [[None] * G for _ in range(P)], codec, 0)
    assert struct.unpack_from("<I", pls2[0][0], 4)[0] == O.topk_k(m, codec) == 3
