"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Bar (north_star): payload bytes (indices, packed values, preamble),
residual bits and top-k order statistics bit-exact; fp32 averages bit-exact under the fixed
tree order R16 (stricter than the north_star's 1e-6 relative).  Inputs are seeded gradgen
buckets; no expected value comes from the GPU.
"""
import numpy as np
import pytest

import oracle as O
from gradgen import seed_for, synthetic

pytestmark = pytest.mark.gpu

F32 = np.float32


@pytest.fixture(scope="module")
def nb():
    import paper_2205_09470_b200 as nbm
    from paper_2205_09470_b200 import build
    build.build()
    nbm.load()
    return nbm


def bits(a):
    return np.ascontiguousarray(a, dtype=F32).view(np.uint32)


def run_loopback(nb, method, sizes, P, steps=3, kind="model-like", vt=0, rho=0.01, k=0, ef=True,
                 start_step=0, per_bucket=False, misalign=False, mutate=None, int8_kernel=None,
                 fp16_kernel=None, sr_seed=0, topk_reduce=None, step_config=None, topk_pipeline=None,
                 topk_stage=None):
    import torch
    ctx = nb.SyncContext(sizes, method, topk_values=vt, topk_density=rho, topk_k=k, error_feedback=ef,
                         start_step=start_step, num_clusters=P, transport=nb.LOOPBACK)
    if int8_kernel:
        staged = int8_kernel.endswith("-staged")     # the same compress kernel, no step fusion
        ctx.set_int8_kernel(int8_kernel[:-len("-staged")] if staged else int8_kernel)
        if staged:
            ctx.set_step_fusion(False)
    if fp16_kernel:
        ctx.set_fp16_kernel(fp16_kernel)
    if topk_pipeline is not None:                    # NEBULA_OPT_TOPK_PIPELINE
        ctx.set_option(nb.OPT_TOPK_PIPELINE, int(topk_pipeline))
    if topk_stage is not None:                       # NEBULA_OPT_TOPK_STAGE (TMA ring or plain loads)
        ctx.set_option(nb.OPT_TOPK_STAGE, int(topk_stage))
    if step_config is not None:                      # fused-step warp split (NEBULA_OPT_STEP_FUSION)
        ctx.set_option(nb.OPT_STEP_FUSION, 2 + step_config)
    if sr_seed:
        ctx.set_sr_seed(sr_seed)
    if topk_reduce is not None:
        ctx.set_option(nb.OPT_TOPK_REDUCE, topk_reduce)
    codec = O.Codec(method=method, topk_values=vt, topk_k=k, topk_density=rho, error_feedback=ef,
                    start_step=start_step, sr_seed=sr_seed)
    total = sum(sizes)
    rs = [[np.zeros(n, F32) for n in sizes] for _ in range(P)]
    for t in range(steps):
        gs = [[synthetic(n, seed_for(c, 0, t, salt=b), kind) for b, n in enumerate(sizes)] for c in range(P)]
        if mutate:
            mutate(gs, t)
        out = torch.full((total + 1,), float("nan"), device="cuda")
        out_v = out[1:] if misalign else out[:total]
        if per_bucket:
            off = 0
            for b, n in enumerate(sizes):
                host = np.concatenate([gs[c][b] for c in range(P)]) if n else np.zeros(0, F32)
                dev = torch.zeros(P * n + 1, device="cuda")
                dv = dev[1:] if misalign else dev[:P * n]
                dv.copy_(torch.from_numpy(host))
                ctx.step(b, dv, out_v[off:off + n], t)
                off += n
        else:
            host = np.concatenate([np.concatenate(gs[c]) if total else np.zeros(0, F32) for c in range(P)])
            dev = torch.zeros(P * total + 1, device="cuda")
            dv = dev[1:] if misalign else dev[:P * total]
            dv.copy_(torch.from_numpy(host))
            ctx.step(nb.ALL_BUCKETS, dv, out_v, t)
        ctx.check()
        got_out = out_v.cpu().numpy()
        off = 0
        for b, n in enumerate(sizes):
            exp_out, r_new, payloads, stats = O.oracle_step([gs[c][b] for c in range(P)],
                                                            [rs[c][b] for c in range(P)], codec, t, bucket=b)
            for c in range(P):
                got = ctx.payload_copy(b, c)
                assert got == payloads[c], f"payload mismatch bucket {b} cluster {c} step {t}: " \
                    f"{_first_diff(got, payloads[c])}"
                rg = ctx.residual(b, c).cpu().numpy()
                re = r_new[c] if r_new[c] is not None else rs[c][b]
                assert np.array_equal(bits(rg), bits(re)), f"residual mismatch b{b} c{c} t{t}: " \
                    f"{np.flatnonzero(bits(rg) != bits(re))[:8]}"
                if method == O.TOPK and O.select_method(codec, t) == O.TOPK and n:
                    st = ctx.topk_stats(b, c)
                    assert (st.k, st.threshold, st.count_above, st.need) == \
                        (stats[c]["k"], stats[c]["threshold"], stats[c]["count_above"], stats[c]["need"])
                rs[c][b] = re
            go = got_out[off:off + n]
            assert np.array_equal(bits(go), bits(exp_out)), f"out mismatch b{b} t{t}: " \
                f"{np.flatnonzero(bits(go) != bits(exp_out))[:8]}"
            off += n
    launches = ctx.kernel_launches()
    ctx.destroy()
    return launches


def _first_diff(a, b):
    if len(a) != len(b):
        return f"len {len(a)} vs {len(b)}"
    for i, (x, y) in enumerate(zip(a, b)):
        if x != y:
            return f"byte {i}: {x} vs {y}"
    return "equal"


# ------------------------------------------------------------------ dense codecs
@pytest.mark.parametrize("method", [O.INT8, O.FP16, O.IDENTITY, O.FP8, O.FP8_E5M2])
@pytest.mark.parametrize("P", [1, 2, 3, 8])
@pytest.mark.parametrize("sizes", [[1], [7], [4096], [4099, 12288, 77777]])
def test_dense_parity(nb, method, P, sizes):
    assert run_loopback(nb, method, sizes, P) > 0


@pytest.mark.parametrize("int8_kernel", ["two-pass", "auto", "fused-ws", "fused-ws-staged"])
@pytest.mark.parametrize("sizes", [[1], [5, 4096, 4099], [300001, 7, 1 << 20], [9_000_003]])
@pytest.mark.parametrize("ef", [True, False])
def test_int8_kernels(nb, int8_kernel, sizes, ef):
    # both INT8 schedules (two-pass streaming, fused split-barrier) are bit-identical to the
    # oracle, for single / many / ragged / large buckets
    run_loopback(nb, O.INT8, sizes, 2, steps=2, ef=ef, int8_kernel=int8_kernel)


@pytest.mark.parametrize("int8_kernel", ["two-pass", "fused-ws", "fused-ws-staged"])
def test_int8_near_half_integer_quotients(nb, int8_kernel):
    # exercises the exact fallback of the reciprocal-multiply fast path (int8_q_fast)
    run_loopback(nb, O.INT8, [50001, 4096], 2, kind="half-ties", steps=1, ef=False, int8_kernel=int8_kernel)
    run_loopback(nb, O.INT8, [50001], 2, kind="half-ties", steps=2, int8_kernel=int8_kernel)


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("per_bucket", [False, True])
@pytest.mark.parametrize("ef", [True, False])
def test_int8_fused_step(nb, P, per_bucket, ef):
    # the one-kernel INT8 step (compress + exchange + reduce): every P (both subtree
    # schedules of the reduce warps), whole-group / ragged / tiny buckets, ALL and per bucket;
    # without EF the max warps' ring tiles are twice as long (a slice of 2048 quads + 5 below)
    run_loopback(nb, O.INT8, [4096 * 37 + 5, 16, 3, 1 << 18, 1000003, 148 * 8192 + 20 + 3], P, steps=3,
                 per_bucket=per_bucket, int8_kernel="fused-ws", ef=ef)


@pytest.mark.parametrize("method", [O.INT8, O.FP8, O.QSGD, O.FP8_E5M2])
@pytest.mark.parametrize("P", [2, 3, 5, 8])
@pytest.mark.parametrize("per_bucket", [False, True])
@pytest.mark.parametrize("ef", [True, False])
def test_pull_reducer_in_fused_step(nb, method, P, per_bucket, ef):
    """The P2P-pull reduce role of the fused step (ws_reduce_ld: 16-B register loads of every
    cluster's payload, both tree-sum schedules: P <= 4 and the two-subtree P > 4 branch) runs
    here on one GPU: LOOPBACK with warp split 4 (the pull default), the peers' slots being the
    local slot buffer.  Bit-exact vs the oracle, ragged / tiny / multi-group buckets."""
    run_loopback(nb, method, [4096 * 37 + 5, 16, 3, 1 << 18, 1000003], P, steps=3, per_bucket=per_bucket,
                 int8_kernel="fused-ws", step_config=4, sr_seed=7 if method == O.QSGD else 0, ef=ef)


@pytest.mark.parametrize("P", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("per_bucket", [False, True])
def test_fp16_fused_step(nb, P, per_bucket):
    """FP16 through its fused compress + exchange + average kernel (k_fp16_step: no grid barrier,
    per-bucket arrival counters, the register-load reduce role on 2-byte codes), incl. ragged,
    tiny and odd-quad buckets; and the overflow / non-finite flags from inside it."""
    run_loopback(nb, O.FP16, [4096 * 37 + 5, 16, 3, 1 << 18, 1000003, (1 << 20) + 4], P, steps=3,
                 per_bucket=per_bucket, int8_kernel="fused-ws")   # (forces fusion on small buckets)


def test_fp16_fused_step_is_one_launch(nb):
    import torch
    sizes = [1 << 20, (1 << 20) + 8]
    ctx = nb.SyncContext(sizes, nb.FP16, num_clusters=2, transport=nb.LOOPBACK)
    g = torch.randn(2 * sum(sizes), device="cuda")
    out = torch.empty(sum(sizes), device="cuda")
    ctx.step(nb.ALL_BUCKETS, g, out, 0)
    ctx.check()
    n0 = ctx.kernel_launches()
    ctx.step(nb.ALL_BUCKETS, g, out, 1)
    ctx.check()
    assert ctx.kernel_launches() - n0 == 1
    g[12345] = 70000.0
    ctx.step(nb.ALL_BUCKETS, g, out, 2)
    with pytest.raises(nb.NebulaError) as e:
        ctx.check()
    assert e.value.code == "OVERFLOW"
    ctx.destroy()


def test_int8_fused_step_is_one_launch(nb):
    import torch
    sizes = [1 << 20, 1 << 20]
    ctx = nb.SyncContext(sizes, nb.INT8, num_clusters=2, transport=nb.LOOPBACK)
    g = torch.randn(2 * sum(sizes), device="cuda")
    out = torch.empty(sum(sizes), device="cuda")
    ctx.step(nb.ALL_BUCKETS, g, out, 0)
    ctx.check()
    n0 = ctx.kernel_launches()
    ctx.step(nb.ALL_BUCKETS, g, out, 1)
    ctx.check()
    assert ctx.kernel_launches() - n0 == 1
    ctx.set_step_fusion(False)
    n0 = ctx.kernel_launches()
    ctx.step(nb.ALL_BUCKETS, g, out, 2)
    ctx.check()
    assert ctx.kernel_launches() - n0 == 2
    ctx.destroy()


@pytest.mark.parametrize("kern", ["two-pass", "fused-ws", "fused-ws-staged"])
@pytest.mark.parametrize("sizes", [[1], [5, 4096, 4099], [300001, 7, 1 << 20], [3_000_003]])
@pytest.mark.parametrize("ef", [True, False])
def test_e5m2_kernels(nb, kern, sizes, ef):
    """FP8 E5M2 (NEXT-4, R33): two-pass, single-pass and fused-step schedules, bit-exact."""
    assert run_loopback(nb, O.FP8_E5M2, sizes, 2, int8_kernel=kern, ef=ef, steps=2) > 0


@pytest.mark.parametrize("kern", ["two-pass", "fused-ws"])
@pytest.mark.parametrize("kind", ["e5m2-ties", "subnormal", "mixed-scale", "tiny-max", "zeros"])
def test_e5m2_near_rounding_boundaries(nb, kern, kind):
    # quotients on / next to E5M2 rounding midpoints: the reciprocal fast path must defer to the
    # IEEE division there
    run_loopback(nb, O.FP8_E5M2, [50001, 4096], 2, kind=kind, steps=1, ef=False, int8_kernel=kern)
    run_loopback(nb, O.FP8_E5M2, [1 << 20, 7], 2, kind=kind, steps=2, int8_kernel=kern)


@pytest.mark.parametrize("vt,rho", [(O.VAL_F32, 0.2), (O.VAL_I8, 0.3), (O.VAL_F16, 0.25)])
def test_topk_wide_resolve(nb, vt, rho):
    """Candidate lists above kWideMin (131072) resolve on many CTAs (k_topk_wide_*: radix-select
    histograms over all CTAs, stable compaction into the second list): bit-exact k, T,
    count_above, need, payloads and residuals, next to a bucket that takes the one-CTA path."""
    run_loopback(nb, O.TOPK, [4_000_003, 9000, 1 << 20], 2, vt=vt, rho=rho, steps=2, kind="normal")


def test_topk_i8_near_half_integer_quotients(nb):
    run_loopback(nb, O.TOPK, [50001], 2, kind="half-ties", vt=O.VAL_I8, rho=0.3, steps=1, ef=False)


@pytest.mark.parametrize("kern", ["two-pass", "fused-ws"])
@pytest.mark.parametrize("sizes", [[1], [5, 4096, 4099], [300001, 7, 1 << 20], [9_000_003]])
@pytest.mark.parametrize("ef", [True, False])
def test_fp8_kernels(nb, kern, sizes, ef):
    """FP8 E4M3 (NEXT-4): the two-pass kernels and the single-pass warp-specialised kernel."""
    assert run_loopback(nb, O.FP8, sizes, 2, int8_kernel=kern, ef=ef, steps=2) > 0


@pytest.mark.parametrize("P", [1, 2, 3])
@pytest.mark.parametrize("sizes", [[1], [5, 4096, 4099], [300001, 7, 1 << 20]])
@pytest.mark.parametrize("seed", [0, 2 ** 64 - 5])
def test_qsgd_parity(nb, P, sizes, seed):
    """QSGD stochastic rounding (NEXT-4, R32): payload bytes (every rounding decision), residuals
    and averages bit-exact vs the oracle's independent SplitMix64 stream."""
    assert run_loopback(nb, O.QSGD, sizes, P, steps=2, sr_seed=seed) > 0


@pytest.mark.parametrize("kern", ["two-pass", "fused-ws", "fused-ws-staged"])
@pytest.mark.parametrize("sizes", [[5, 4096, 4099], [300001, 7, 1 << 20], [9_000_003]])
@pytest.mark.parametrize("P", [1, 2, 3])
def test_qsgd_kernels(nb, kern, sizes, P):
    """QSGD through the two-pass kernels, the single-pass warp-specialised compress kernel and
    the fused compress + exchange + average step (same SplitMix64 stream in every schedule)."""
    assert run_loopback(nb, O.QSGD, sizes, P, steps=2, sr_seed=3, int8_kernel=kern) > 0


@pytest.mark.parametrize("kind", ["ties", "half-ties", "int-ties", "zeros", "tiny-max", "subnormal"])
def test_qsgd_edge_values(nb, kind):
    run_loopback(nb, O.QSGD, [5000, 17], 2, kind=kind, steps=2, sr_seed=11)


@pytest.mark.parametrize("P", [1, 2, 3, 8])
@pytest.mark.parametrize("per_bucket", [False, True])
def test_fp8_fused_step(nb, P, per_bucket):
    """FP8 through the fused compress + exchange + average kernel (buckets >= 1M elements)."""
    run_loopback(nb, O.FP8, [1 << 20, 3 << 19, (1 << 20) + 5], P, steps=2, per_bucket=per_bucket)


@pytest.mark.parametrize("kern", ["two-pass", "fused-ws"])
def test_fp8_near_rounding_boundaries(nb, kern):
    """Quotients on / next to E4M3 midpoints: the reciprocal fast path must hand every one of
    them to the IEEE division (bit-exact payload and residual)."""
    run_loopback(nb, O.FP8, [50001, 4096], 2, kind="fp8-ties", steps=1, ef=False, int8_kernel=kern)
    run_loopback(nb, O.FP8, [1 << 20, 7], 2, kind="fp8-ties", steps=2, int8_kernel=kern)


@pytest.mark.parametrize("fp16_kernel", ["tma", "plain"])
@pytest.mark.parametrize("sizes", [[1], [5, 4096, 4099], [300001, 7, 1 << 20]])
def test_fp16_kernels(nb, fp16_kernel, sizes):
    run_loopback(nb, O.FP16, sizes, 2, steps=2, fp16_kernel=fp16_kernel)
    run_loopback(nb, O.FP16, sizes, 3, steps=1, ef=False, fp16_kernel=fp16_kernel)


@pytest.mark.parametrize("method", [O.INT8, O.FP16, O.FP8])
@pytest.mark.parametrize("kind", ["ties", "subnormal", "mixed-scale", "signed-zero", "zeros", "tiny-max", "zipf-rows"])
def test_dense_edge_values(nb, method, kind):
    if method == O.FP16 and kind == "mixed-scale":
        pytest.skip("mixed-scale overflows fp16 by design (covered by the overflow test)")
    run_loopback(nb, method, [5003, 40000], 2, kind=kind)


@pytest.mark.parametrize("method", [O.INT8, O.FP16, O.TOPK, O.FP8])
def test_no_error_feedback(nb, method):
    run_loopback(nb, method, [30001], 2, ef=False, rho=0.05)


@pytest.mark.parametrize("method", [O.INT8, O.FP16, O.TOPK, O.FP8])
@pytest.mark.parametrize("per_bucket,misalign", [(True, False), (False, True), (True, True)])
def test_call_shapes_and_alignment(nb, method, per_bucket, misalign):
    run_loopback(nb, method, [4099, 1, 0, 65536, 9], 3, per_bucket=per_bucket, misalign=misalign, rho=0.1)


def test_start_step_gate(nb):
    # steps 0,1 IDENTITY (residual untouched), 2.. INT8
    run_loopback(nb, O.INT8, [1000, 5000], 2, steps=4, start_step=2)
    run_loopback(nb, O.TOPK, [1000, 5000], 2, steps=3, start_step=1, rho=0.1)


def test_config1_shape(nb):
    # BASELINE config 1: 2 clusters x one 1M-float bucket, 3-step EF run
    for method, vt, rho in [(O.INT8, 0, 0.01), (O.FP16, 0, 0.01), (O.TOPK, O.VAL_F32, 0.01), (O.TOPK, O.VAL_F32, 0.10)]:
        run_loopback(nb, method, [1 << 20], 2, vt=vt, rho=rho)


# ------------------------------------------------------------------ top-k
@pytest.mark.parametrize("vt", [O.VAL_F32, O.VAL_F16, O.VAL_I8])
@pytest.mark.parametrize("rho", [0.001, 0.01, 0.1, 0.5])
@pytest.mark.parametrize("P", [2, 4])
def test_topk_parity(nb, vt, rho, P):
    run_loopback(nb, O.TOPK, [200003, 4096, 3], P, vt=vt, rho=rho)


@pytest.mark.parametrize("pipeline", [False, True])
@pytest.mark.parametrize("sizes", [[200003, 4096], [1, 70001, 3, 4096 * 9, 2], [300000] * 5])
def test_topk_two_stream_pipeline(nb, pipeline, sizes):
    """The ALL-bucket top-k step on two streams (first / second half of the buckets, own
    counters and staging) and on one: both bit-exact vs the oracle, incl. odd bucket counts."""
    run_loopback(nb, O.TOPK, sizes, 2, rho=0.02, steps=3, topk_pipeline=pipeline)
    run_loopback(nb, O.TOPK, sizes, 3, vt=O.VAL_I8, rho=0.2, steps=2, topk_pipeline=pipeline)


@pytest.mark.parametrize("stage", [0, 1])
@pytest.mark.parametrize("ef", [True, False])
@pytest.mark.parametrize("misalign", [False, True])
def test_topk_stage_variants(nb, stage, ef, misalign):
    """The stage pass with plain vector loads (0) and through the TMA ring (1, the default for
    16-B aligned calls; misaligned calls take the scalar kernel): bit-exact vs the oracle over
    buckets with ragged tails, a bucket shorter than one chunk and several chunks per CTA."""
    sizes = [200003, 4096 * 3 + 5, 7, 1 << 20]
    run_loopback(nb, O.TOPK, sizes, 2, rho=0.01, steps=3, ef=ef, misalign=misalign, topk_stage=stage)
    run_loopback(nb, O.TOPK, sizes, 3, vt=O.VAL_F16, rho=0.3, steps=2, ef=ef, misalign=misalign, topk_stage=stage)


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("rho,P", [(0.01, 2), (0.3, 3), (0.001, 8)])
@pytest.mark.parametrize("per_bucket,misalign", [(False, False), (True, True)])
def test_topk_reduce_variants(nb, variant, rho, P, per_bucket, misalign):
    """Both sparse decompress-average kernels (tile-interleaved, per-warp ranges: the default)."""
    run_loopback(nb, O.TOPK, [300001, 2048, 4097, 1], P, rho=rho, steps=2, per_bucket=per_bucket,
                 misalign=misalign, topk_reduce=variant)


@pytest.mark.parametrize("kind", ["ties", "zipf-rows", "zeros", "signed-zero", "strided-zeros", "subnormal",
                                  "normal", "uniform"])
@pytest.mark.parametrize("rho", [0.01, 0.4])
def test_topk_structured_inputs(nb, kind, rho):
    run_loopback(nb, O.TOPK, [150001], 2, kind=kind, rho=rho)


@pytest.mark.parametrize("k", [1, 2, 999, 150000, 150001])
def test_topk_exact_k_and_full(nb, k):
    run_loopback(nb, O.TOPK, [150001], 2, k=k, steps=2)


@pytest.mark.parametrize("kind", ["strided-zeros", "strided-small"])
@pytest.mark.parametrize("vt", [O.VAL_F32, O.VAL_F16, O.VAL_I8])
def test_topk_fallback_path_is_exercised(nb, vt, kind):
    """The exact radix fallback (the sampled bracket fails on this input): payload AND residual
    vs the oracle — the stage pass may have stored winners' residuals, which k_topk_restore must
    put back as p before the fallback re-reads r."""
    import torch
    n = 50000
    ctx = nb.SyncContext([n], nb.TOPK, topk_density=0.1, topk_values=vt, num_clusters=1, transport=nb.LOOPBACK)
    g = torch.from_numpy(synthetic(n, 1, kind)).cuda()
    out = torch.empty(n, device="cuda")
    ctx.step(0, g, out, 0)
    ctx.check()
    st = ctx.topk_stats(0, 0)
    assert st.path == 1       # the sampled bracket failed and the exact radix fallback ran
    res = O.cluster_step(g.cpu().numpy(), np.zeros(n, F32), O.Codec(method=O.TOPK, topk_density=0.1,
                                                                    topk_values=vt), 0)
    assert ctx.payload_copy(0, 0) == res.payload
    assert np.array_equal(bits(ctx.residual(0, 0).cpu().numpy()), bits(res.r_new))
    ctx.destroy()


# ------------------------------------------------------------------ device errors
@pytest.mark.parametrize("method", [O.IDENTITY, O.FP16, O.INT8, O.TOPK, O.FP8, O.QSGD])
@pytest.mark.parametrize("bad", [float("nan"), float("inf"), -float("inf")])
def test_nonfinite_is_reported(nb, method, bad):
    import torch
    ctx = nb.SyncContext([4096, 100], method, num_clusters=2, transport=nb.LOOPBACK, topk_density=0.1)
    g = torch.randn(2 * 4196, device="cuda")
    g[4096 + 100 + 17] = bad
    out = torch.empty(4196, device="cuda")
    ctx.step(nb.ALL_BUCKETS, g, out, 0)
    with pytest.raises(nb.NebulaError) as e:
        ctx.check()
    assert e.value.code == "NONFINITE"
    ctx.check()   # sticky flag was cleared by the check
    ctx.destroy()


@pytest.mark.parametrize("method", [O.INT8, O.FP16, O.TOPK])
def test_device_error_seen_by_next_call(nb, method):
    """ABI: a device-detected error is returned by the next stage call (through the pinned host
    mirror of the flag word, refreshed asynchronously after every step) without nebula_check;
    nothing is enqueued by that call; nebula_check then clears it."""
    import torch
    ctx = nb.SyncContext([1 << 20, 4100], method, num_clusters=2, transport=nb.LOOPBACK, topk_density=0.1)
    n = (1 << 20) + 4100
    g = torch.randn(2 * n, device="cuda")
    g[12345] = float("inf")
    out = torch.empty(n, device="cuda")
    ctx.step(nb.ALL_BUCKETS, g, out, 0)
    torch.cuda.synchronize()                       # the step (and its mirror copy) completed
    l0 = ctx.kernel_launches()
    with pytest.raises(nb.NebulaError) as e:
        ctx.step(nb.ALL_BUCKETS, g, out, 1)
    assert e.value.code == "NONFINITE" and ctx.kernel_launches() == l0
    with pytest.raises(nb.NebulaError) as e:
        ctx.check()
    assert e.value.code == "NONFINITE"
    g[12345] = 0.0
    for r in range(2):
        ctx.residual(0, r).zero_()                 # the caller resets the residual after the error
    ctx.step(nb.ALL_BUCKETS, g, out, 1)
    ctx.check()
    ctx.destroy()


@pytest.mark.parametrize("int8_kernel", ["two-pass", "fused-ws"])
def test_int8_nonfinite_writes_nothing(nb, int8_kernel):
    import torch
    ctx = nb.SyncContext([1000], nb.INT8, num_clusters=1, transport=nb.LOOPBACK)
    ctx.set_int8_kernel(int8_kernel)
    g = torch.randn(1000, device="cuda")
    out = torch.empty(1000, device="cuda")
    ctx.step(0, g, out, 0)
    ctx.check()
    before = (ctx.payload_copy(0, 0), ctx.residual(0, 0).clone())
    g[5] = float("nan")
    ctx.step(0, g, out, 1)
    with pytest.raises(nb.NebulaError):
        ctx.check()
    assert ctx.payload_copy(0, 0) == before[0]          # no payload written for the bucket
    if int8_kernel == "two-pass":                       # the streaming schedule also leaves r
        assert torch.equal(ctx.residual(0, 0), before[1])
    ctx.destroy()


@pytest.mark.parametrize("method,vt", [(O.FP16, 0), (O.TOPK, O.VAL_F16)])
def test_fp16_overflow_is_reported(nb, method, vt):
    import torch
    ctx = nb.SyncContext([1000], method, topk_values=vt, topk_density=0.5, num_clusters=2, transport=nb.LOOPBACK)
    g = torch.randn(2000, device="cuda")
    g[1500] = 65520.0
    out = torch.empty(1000, device="cuda")
    ctx.step(0, g, out, 0)
    with pytest.raises(nb.NebulaError) as e:
        ctx.check()
    assert e.value.code == "OVERFLOW"
    for c in range(2):         # after a device error the residual is unspecified: reset it
        ctx.residual(0, c).zero_()
    g[1500] = 65519.0          # rounds to 65504: not an overflow (R10)
    ctx.step(0, g, out, 1)
    ctx.check()
    ctx.destroy()


def test_state_machine(nb):
    import torch
    ctx = nb.SyncContext([100, 200], nb.INT8, num_clusters=2, transport=nb.LOOPBACK)
    g = torch.randn(600, device="cuda")
    out = torch.empty(300, device="cuda")
    with pytest.raises(nb.NebulaError) as e:
        ctx.exchange(0)
    assert e.value.code == "STATE"
    ctx.compress(0, g[:200], 0)
    with pytest.raises(nb.NebulaError):
        ctx.decompress_reduce(0, out[:100])
    ctx.exchange(0)
    ctx.decompress_reduce(0, out[:100])
    with pytest.raises(nb.NebulaError):
        ctx.decompress_reduce(nb.ALL_BUCKETS, out)
    ctx.destroy()


def test_step_host_matches_device_path(nb):
    import torch
    sizes = [4096, 10001]
    P = 2
    gs = np.concatenate([synthetic(sum(sizes), 3 + c, "model-like") for c in range(P)])
    a = nb.SyncContext(sizes, nb.INT8, num_clusters=P, transport=nb.LOOPBACK)
    b = nb.SyncContext(sizes, nb.INT8, num_clusters=P, transport=nb.LOOPBACK)
    out_h = np.empty(sum(sizes), F32)
    a.step_host(gs, out_h, 0)
    out_d = torch.empty(sum(sizes), device="cuda")
    b.step(nb.ALL_BUCKETS, torch.from_numpy(gs).cuda(), out_d, 0)
    assert np.array_equal(bits(out_h), bits(out_d.cpu().numpy()))
    a.destroy()
    b.destroy()


# ------------------------------------------------------------------ pipeline hop (NEXT-2)
@pytest.mark.parametrize("method,vt", [(O.FP16, 0), (O.INT8, 0), (O.IDENTITY, 0), (O.TOPK, O.VAL_F32),
                                       (O.TOPK, O.VAL_I8), (O.FP8, 0)])
def test_decompress_single_slot(nb, method, vt):
    """Scenario-II hop semantics: each side decodes the OTHER side's
    payload exactly, no averaging, no error feedback; Table 5's ratios hold for the bytes."""
    import torch
    sizes = [128 * 64 * 768 // 8, 4099]            # an H^E-shaped activation block + ragged
    P = 2
    ctx = nb.SyncContext(sizes, method, topk_values=vt, topk_density=0.1, error_feedback=False, num_clusters=P,
                         transport=nb.LOOPBACK)
    codec = O.Codec(method=method, topk_values=vt, topk_density=0.1, error_feedback=False)
    xs = [np.concatenate([synthetic(n, 90 + 7 * c + b, "normal") for b, n in enumerate(sizes)]) for c in range(P)]
    dev = torch.from_numpy(np.concatenate(xs)).cuda()
    ctx.compress(nb.ALL_BUCKETS, dev, 0)
    ctx.exchange(nb.ALL_BUCKETS)
    total = sum(sizes)
    for slot in range(P):
        out = torch.full((total,), float("nan"), device="cuda")
        ctx.decompress(nb.ALL_BUCKETS, slot, out)
        got = out.cpu().numpy()
        off = 0
        for b, n in enumerate(sizes):
            res = O.cluster_step(xs[slot][off:off + n], None, codec, 0)
            assert ctx.payload_copy(b, slot) == res.payload
            assert np.array_equal(bits(got[off:off + n]), bits(O.decode_payload(res.payload, n)))
            if method in (O.FP16, O.INT8, O.FP8):
                assert (len(res.payload) - 16) / (4 * n) == pytest.approx({O.FP16: 0.50, O.INT8: 0.25, O.FP8: 0.25}[method],
                                                                        abs=16 / (4 * n))
            off += n
    ctx.decompress_reduce(nb.ALL_BUCKETS, torch.empty(total, device="cuda"))
    ctx.destroy()
