"""Every cross-GPU code path on ONE GPU: the SELF transport (include/nebula_sync.h) gives each
(cluster, GPU) its own context inside this process, and the contexts reach each other's
buffers directly — so the P2P push stores (push_u32 / push_u64 into the peers' slot
buffers), the pull reducer reading the peers' own slots, the system-scope release/acquire
arrival-flag protocol (k_exchange_flags), the double-buffered slot parity, and the G > 1
intra-cluster hop (push reduce-scatter + fixed-order reduce, flags, all-gather pull, the exact
cluster scale mailbox) all run exactly as they do across processes over NVLink.

Bar: every member's output, own payload and residual bit-identical to the oracle
(oracle_step for P x 1, hierarchical_step for P x G) on NON-dyadic model-like gradients, and
all members' outputs bit-identical.  PAPER.md:76 (aggregation), :95 / :288 (data parallelism
across clusters, intra vs inter split); SPEC.md:242 / :547 (transport equivalence).
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


def _sync(grid):
    for row in grid:
        for ctx in row:
            ctx.stream.synchronize()


def run_self(nb, method, P, G, sizes, *, steps=2, vt=0, rho=0.05, exchange="auto", per_bucket=False,
             exact=False, int8_kernel="two-pass", kind="model-like", sr_seed=0, ef=True, exact_topk=False,
             intra=None):
    import torch
    grid = nb.self_group(sizes, num_clusters=P, gpus_per_cluster=G, device=0, method=method, topk_values=vt,
                         topk_density=rho, error_feedback=ef, exact_topk=exact_topk)
    for row in grid:
        for ctx in row:
            if method in (O.INT8, O.FP8, O.QSGD, O.FP8_E5M2):
                ctx.set_int8_kernel(int8_kernel)
            if P > 1:
                ctx.set_exchange(exchange)
            if exact:
                ctx.set_exact_scale(True)
            if sr_seed:
                ctx.set_sr_seed(sr_seed)
            if intra:
                ctx.set_intra(intra)
    codec = O.Codec(method=method, topk_values=vt, topk_density=rho, sr_seed=sr_seed, error_feedback=ef)
    total = sum(sizes)
    m = [s if exact_topk else s // G for s in sizes]   # coded elements per GPU (R34: the whole bucket)
    rs = [[[np.zeros(mb, F32) for mb in m] for _ in range(G)] for _ in range(P)]
    modes = {grid[0][0].exchange_mode()}
    for t in range(steps):
        def grad(c, l, b):
            return synthetic(sizes[b], seed_for(c, l, t, salt=b), kind)
        gdev = [[torch.from_numpy(np.concatenate([grad(c, l, b) for b in range(len(sizes))])).cuda()
                 for l in range(G)] for c in range(P)]
        outs = [[torch.full((total,), float("nan"), device="cuda") for _ in range(G)] for _ in range(P)]
        torch.cuda.synchronize()
        calls = [(b, off, n) for b, (off, n) in enumerate(zip(np.cumsum([0] + sizes[:-1]), sizes))] \
            if per_bucket else [(nb.ALL_BUCKETS, 0, total)]
        for b, off, n in calls:
            # each stage is enqueued for every member before anyone waits (a member's exchange
            # waits for its peers' compress; its intra-cluster hop for its peers' pushes)
            for c in range(P):
                for l in range(G):
                    grid[c][l].compress(b, gdev[c][l][off:off + n], t)
            _sync(grid)
            for c in range(P):
                for l in range(G):
                    grid[c][l].exchange(b)
            for c in range(P):
                for l in range(G):
                    grid[c][l].decompress_reduce(b, outs[c][l][off:off + n])
            _sync(grid)
        for row in grid:
            for ctx in row:
                ctx.check()
        ref = outs[0][0].cpu().numpy()
        for c in range(P):
            for l in range(G):
                assert np.array_equal(outs[c][l].cpu().numpy().view(np.uint32), ref.view(np.uint32)), \
                    f"members disagree: ({c},{l}) vs (0,0) step {t}"
        off = 0
        for b, n in enumerate(sizes):
            if G == 1:
                exp, r_new, payloads, _ = O.oracle_step([grad(c, 0, b) for c in range(P)],
                                                        [rs[c][0][b] for c in range(P)], codec, t, bucket=b)
                pls = [[p] for p in payloads]
                r_new = [[r] for r in r_new]
            else:
                exp, r_new, pls = O.hierarchical_step([[grad(c, l, b) for l in range(G)] for c in range(P)],
                                                      [[rs[c][l][b] for l in range(G)] for c in range(P)], codec, t,
                                                      exact_scale=exact, bucket=b, exact_topk=exact_topk)
            assert np.array_equal(ref[off:off + n].view(np.uint32), exp.view(np.uint32)), \
                f"out mismatch bucket {b} step {t}: {np.flatnonzero(ref[off:off + n].view(np.uint32) != exp.view(np.uint32))[:8]}"
            for c in range(P):
                for l in range(G):
                    ctx = grid[c][l]
                    assert ctx.payload_copy(b, c) == pls[c][l], f"payload mismatch ({c},{l}) b{b} t{t}"
                    if G == 1:   # after the exchange every slot holds that cluster's payload
                        for c2 in range(P):
                            assert ctx.payload_copy(b, c2) == pls[c2][0], f"slot {c2} at member {c} b{b}"
                    if r_new[c][l] is not None:
                        rg = ctx.residual(b, c).cpu().numpy()
                        assert np.array_equal(rg.view(np.uint32), r_new[c][l].view(np.uint32)), \
                            f"residual mismatch ({c},{l}) b{b} t{t}"
                        rs[c][l][b] = r_new[c][l]
            off += n
    launches = sum(ctx.kernel_launches() for row in grid for ctx in row)
    _sync(grid)
    for row in grid:
        for ctx in row:
            ctx.destroy()
    return modes, launches


SIZES = [4096, 12288, 300004, 8, 77777 * 4]


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("exchange", ["push", "pull"])
@pytest.mark.parametrize("per_bucket", [False, True])
def test_self_p2p_exchange_int8(nb, P, exchange, per_bucket):
    """P clusters x 1 GPU: the compress kernels push every payload word into the peers' slots
    (push) or the reducer loads the peers' own slots (pull); arrival flags in between."""
    modes, _ = run_self(nb, O.INT8, P, 1, SIZES, exchange=exchange, per_bucket=per_bucket, steps=3)
    assert modes == {"p2p-" + exchange}


@pytest.mark.parametrize("method,vt", [(O.FP16, 0), (O.IDENTITY, 0), (O.FP8, 0), (O.QSGD, 0), (O.FP8_E5M2, 0),
                                       (O.TOPK, O.VAL_F32), (O.TOPK, O.VAL_F16), (O.TOPK, O.VAL_I8)])
@pytest.mark.parametrize("exchange", ["push", "pull"])
def test_self_p2p_exchange_codecs(nb, method, vt, exchange):
    run_self(nb, method, 3, 1, SIZES, vt=vt, exchange=exchange, sr_seed=5 if method == O.QSGD else 0)


@pytest.mark.parametrize("P,G", [(1, 2), (2, 2), (1, 4), (2, 4), (1, 8)])
@pytest.mark.parametrize("per_bucket", [False, True])
def test_self_hierarchical_exact_any_input(nb, P, G, per_bucket):
    """G > 1: the cluster mean is the fixed-order P2P reduce-scatter (push + flags + sum in
    local-rank order / G), so it is bit-identical to the oracle on non-dyadic inputs."""
    run_self(nb, O.INT8, P, G, [s * G for s in [4096, 12288, 300004, 8]], per_bucket=per_bucket)


@pytest.mark.parametrize("method,vt", [(O.FP16, 0), (O.TOPK, O.VAL_F32), (O.TOPK, O.VAL_I8), (O.FP8, 0),
                                       (O.QSGD, 0), (O.IDENTITY, 0)])
def test_self_hierarchical_codecs(nb, method, vt):
    run_self(nb, method, 2, 2, [s * 2 for s in [4096, 300004, 8]], vt=vt, exchange="pull",
             sr_seed=9 if method == O.QSGD else 0)


@pytest.mark.parametrize("method", [O.INT8, O.FP8, O.QSGD, O.FP8_E5M2])
@pytest.mark.parametrize("P,G", [(2, 2), (1, 4)])
def test_self_exact_cluster_scale(nb, method, P, G):
    """NEXT-3 (R28): every shard quantises with the scale of the whole cluster bucket; the G
    shards' max words meet in the P2P mailbox kernel."""
    run_self(nb, method, P, G, [s * G for s in [4096, 300004, 8]], exact=True, sr_seed=3 if method == O.QSGD else 0)


@pytest.mark.parametrize("vt", [O.VAL_F32, O.VAL_F16, O.VAL_I8])
@pytest.mark.parametrize("P,G", [(2, 2), (1, 4), (2, 4)])
@pytest.mark.parametrize("per_bucket", [False, True])
def test_self_exact_cluster_topk(nb, vt, P, G, per_bucket):
    """NEXT-3 (R34): with NEBULA_CODEC_EXACT_TOPK every GPU selects the top-k of the WHOLE
    cluster bucket (fixed-order P2P mean, all-gathered), so payloads, the cluster's full
    residual and the average equal the oracle's global selection bit for bit."""
    run_self(nb, O.TOPK, P, G, [s * G for s in [4096, 300004, 8, 12288]], vt=vt, rho=0.02, per_bucket=per_bucket,
             exact_topk=True, steps=3)


def test_self_state_rules(nb):
    import torch
    grid = nb.self_group([1024, 1024], num_clusters=2, device=0, method=nb.INT8)
    g = torch.randn(2048, device="cuda")
    out = torch.empty(2048, device="cuda")
    a, b = grid[0][0], grid[1][0]
    with pytest.raises(nb.NebulaError) as e:
        a.set_exchange("nccl")
    assert e.value.code == "UNSUPPORTED"
    a.compress(0, g[:1024], 0)
    with pytest.raises(nb.NebulaError) as e:   # compress twice without exchange / reduce
        a.compress(0, g[:1024], 1)
    assert e.value.code == "STATE"
    b.compress(0, g[:1024], 0)
    _sync(grid)
    a.exchange(0)
    b.exchange(0)
    a.decompress_reduce(0, out[:1024])
    b.decompress_reduce(0, out[:1024])
    _sync(grid)
    with pytest.raises(nb.NebulaError) as e:   # ALL over buckets at different step counts
        a.compress(nb.ALL_BUCKETS, g, 1)
    assert e.value.code == "STATE"
    for ctx in (a, b):
        ctx.check()
        ctx.destroy()


def test_self_group_must_be_complete(nb):
    import torch
    gid = nb.self_group_id()
    a = nb.SyncContext([1024], nb.INT8, num_clusters=2, cluster_id=0, transport=nb.SELF, device=0, unique_id=gid)
    with pytest.raises(nb.NebulaError) as e:
        a.compress(0, torch.zeros(1024, device="cuda"), 0)
    assert e.value.code == "STATE"
    with pytest.raises(nb.NebulaError):       # the same (cluster, GPU) twice in one group
        nb.SyncContext([1024], nb.INT8, num_clusters=2, cluster_id=0, transport=nb.SELF, device=0, unique_id=gid)
    a.destroy()
