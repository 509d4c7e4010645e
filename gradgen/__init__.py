"""gradgen — seeded synthetic gradient generator.

This module is the ONE piece shared by the CPU oracle tests, the GPU parity tests and
``bench.py``.  It holds no compression arithmetic at all (no casting, no scaling, no
selection, no averaging): it only produces fp32 gradient buffers with the shapes,
sparsity structure and value spread of the paper's workloads, so that both sides of a
parity test consume the same bytes.

Recipe (restated in DESIGN.md "Input recipe"; SURVEY.md §8(d) "Value distributions"):

* seed = 20220519 + 7919*cluster + 104729*local_rank + 15485863*step  (numpy PCG64)
* dense weights / biases / LayerNorm tensors: N(0, sigma_t^2) with
  sigma_t = 10**U(-4, -2) drawn per tensor — the spread that makes a per-bucket INT8
  scale push small-sigma tensors into the error-feedback residual;
* word-embedding gradients [V, d]: only rows of tokens present in the step's token
  budget are nonzero.  Tokens are drawn Zipf(1.1) over the vocabulary (rank r has
  probability proportional to r**-1.1), ranks are mapped to row ids by a fixed seeded
  permutation; every other row is exactly 0.0.  Token budgets follow the paper's batch
  recipes: ERNIE-M 2048 x 512 over 64 devices -> 32 x 512 = 16,384 tokens per GPU
  (§4.1 settings); ABNet / MT 128 x 64 = 8,192 tokens (§4.2);
* outliers: a 1e-4 fraction of elements (seeded positions) multiplied by 100.

Model shapes (parameter counts are the BASELINE.json configs):

* ``ernie-m-base``  : vocab 250,002, d 768, 12 layers, FFN 3072, 514 positions, pooler
                      -> 278,042,880 elements in 198 tensors;
* ``ernie-m-large`` : vocab 250,002, d 1024, 24 layers, FFN 4096 -> 559,889,408 / 390;
* ``ernie-m-large-adapters`` : the ABNet adapter subset ("adapter",
  bottleneck 512 from PAPER.md:350): 24 x (LN 2*1024 + 1024x512 + 512 + 512x1024 + 1024)
  -> 25,251,840 elements in 144 tensors (the parameter-efficient trainable subset,
  PAPER.md:80 "only the parameters of the add-in networks are to be transferred");
* ``transformer-big``: d 1024, FFN 4096, 6+6 layers, tied vocab 32,768
                      -> 209,915,904 elements in 257 tensors.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "SEED_BASE", "seed_for", "model_tensors", "model_numel", "MODELS",
    "model_gradient", "synthetic", "fixed_buckets", "EDGE_KINDS",
]

SEED_BASE = 20220519


def seed_for(cluster: int = 0, local_rank: int = 0, step: int = 0, salt: int = 0) -> int:
    """Per-(cluster, GPU, step) seed of SURVEY.md §8(d)."""
    return SEED_BASE + 7919 * cluster + 104729 * local_rank + 15485863 * step + 1000003 * salt


# --------------------------------------------------------------------------- shapes
def _encoder_layer(p, d, ffn):
    t = []
    for m in ("q", "k", "v", "o"):
        t += [(f"{p}.attn.{m}.weight", (d, d), "dense"), (f"{p}.attn.{m}.bias", (d,), "dense")]
    t += [(f"{p}.ln1.weight", (d,), "dense"), (f"{p}.ln1.bias", (d,), "dense")]
    t += [(f"{p}.ffn1.weight", (d, ffn), "dense"), (f"{p}.ffn1.bias", (ffn,), "dense")]
    t += [(f"{p}.ffn2.weight", (ffn, d), "dense"), (f"{p}.ffn2.bias", (d,), "dense")]
    t += [(f"{p}.ln2.weight", (d,), "dense"), (f"{p}.ln2.bias", (d,), "dense")]
    return t


def _ernie_m(vocab, d, layers, ffn, pos=514):
    t = [("emb.word", (vocab, d), "embedding"), ("emb.pos", (pos, d), "dense"),
         ("emb.ln.weight", (d,), "dense"), ("emb.ln.bias", (d,), "dense")]
    for i in range(layers):
        t += _encoder_layer(f"enc.{i}", d, ffn)
    t += [("pooler.weight", (d, d), "dense"), ("pooler.bias", (d,), "dense")]
    return t


def _adapters(layers=24, d=1024, bottleneck=512):
    t = []
    for i in range(layers):
        p = f"adapter.{i}"
        t += [(f"{p}.ln.weight", (d,), "dense"), (f"{p}.ln.bias", (d,), "dense"),
              (f"{p}.down.weight", (d, bottleneck), "dense"), (f"{p}.down.bias", (bottleneck,), "dense"),
              (f"{p}.up.weight", (bottleneck, d), "dense"), (f"{p}.up.bias", (d,), "dense")]
    return t


def _transformer_big(vocab=32768, d=1024, ffn=4096, enc=6, dec=6):
    t = [("emb.shared", (vocab, d), "embedding")]
    for i in range(enc):
        t += _encoder_layer(f"enc.{i}", d, ffn)
    for i in range(dec):
        p = f"dec.{i}"
        for blk in ("self", "cross"):
            for m in ("q", "k", "v", "o"):
                t += [(f"{p}.{blk}.{m}.weight", (d, d), "dense"), (f"{p}.{blk}.{m}.bias", (d,), "dense")]
        t += [(f"{p}.ln1.weight", (d,), "dense"), (f"{p}.ln1.bias", (d,), "dense"),
              (f"{p}.ln2.weight", (d,), "dense"), (f"{p}.ln2.bias", (d,), "dense"),
              (f"{p}.ffn1.weight", (d, ffn), "dense"), (f"{p}.ffn1.bias", (ffn,), "dense"),
              (f"{p}.ffn2.weight", (ffn, d), "dense"), (f"{p}.ffn2.bias", (d,), "dense"),
              (f"{p}.ln3.weight", (d,), "dense"), (f"{p}.ln3.bias", (d,), "dense")]
    t += [("enc.ln.weight", (d,), "dense"), ("enc.ln.bias", (d,), "dense"),
          ("dec.ln.weight", (d,), "dense"), ("dec.ln.bias", (d,), "dense")]
    return t


MODELS = {
    "ernie-m-base": (lambda: _ernie_m(250002, 768, 12, 3072), 16384),
    "ernie-m-large": (lambda: _ernie_m(250002, 1024, 24, 4096), 16384),
    "ernie-m-large-adapters": (lambda: _adapters(), 0),
    "transformer-big": (lambda: _transformer_big(), 8192),
}


def model_tensors(name: str):
    """[(tensor name, shape, kind)] in state-dict order (the flat-buffer order)."""
    return MODELS[name][0]()


def model_numel(name: str) -> int:
    return int(sum(int(np.prod(s)) for _, s, _ in model_tensors(name)))


# --------------------------------------------------------------------------- values
def _zipf_rows(rng, vocab, tokens, a=1.1):
    ranks = np.arange(1, vocab + 1, dtype=np.float64)
    cdf = np.cumsum(ranks ** -a)
    cdf /= cdf[-1]
    draws = np.searchsorted(cdf, rng.random(tokens))
    perm = np.random.default_rng(SEED_BASE).permutation(vocab)  # fixed rank -> row id map
    return np.unique(perm[np.minimum(draws, vocab - 1)])


def model_gradient(name: str, cluster: int = 0, local_rank: int = 0, step: int = 0,
                   outlier_frac: float = 1e-4, out: np.ndarray | None = None) -> np.ndarray:
    """Flat fp32 gradient of model ``name`` for one (cluster, GPU, step)."""
    tensors = model_tensors(name)
    tokens = MODELS[name][1]
    n = sum(int(np.prod(s)) for _, s, _ in tensors)
    rng = np.random.default_rng(seed_for(cluster, local_rank, step))
    g = np.empty(n, dtype=np.float32) if out is None else out
    assert g.dtype == np.float32 and g.size == n
    off = 0
    for _, shape, kind in tensors:
        size = int(np.prod(shape))
        sigma = np.float32(10.0 ** rng.uniform(-4.0, -2.0))
        view = g[off:off + size]
        if kind == "embedding" and tokens > 0:
            rows, d = shape
            view[:] = 0.0
            live = _zipf_rows(rng, rows, tokens)
            mat = view.reshape(rows, d)
            mat[live] = rng.standard_normal((live.size, d), dtype=np.float32) * sigma
        else:
            rng.standard_normal(size, dtype=np.float32, out=view)
            view *= sigma
        off += size
    if outlier_frac > 0:
        m = int(n * outlier_frac)
        pos = rng.integers(0, n, size=m)
        g[pos] *= np.float32(100.0)
    return g


EDGE_KINDS = ("normal", "model-like", "zipf-rows", "ties", "zeros", "subnormal",
              "mixed-scale", "signed-zero", "uniform", "tiny-max", "strided-zeros", "strided-small", "half-ties", "fp8-ties", "e5m2-ties", "int-ties")


def synthetic(n: int, seed: int, kind: str = "normal", sigma: float = 1.0) -> np.ndarray:
    """Flat fp32 test bucket of ``n`` elements with a given value structure.

    kinds: normal N(0, sigma^2); model-like (per-4096-chunk sigma 10**U(-4,-2) plus 1e-4
    outliers x100); zipf-rows (rows of 64 elements, ~7% nonzero, Zipf(1.1) picked);
    ties (values drawn from 7 distinct magnitudes with random signs — many exact ties);
    zeros (all +0.0); subnormal (values around 1e-40); mixed-scale (N(0,1) scaled by
    10**U(-30, 3) per element); signed-zero (half +0.0, half -0.0, a few nonzeros);
    uniform U(-1, 1); tiny-max (max |g| ~ 1e-44, below 127 * 2**-149); strided-zeros (every
    16th element 0, the rest N(0,1)); strided-small (every 16th element N(0, 1e-6), the rest
    N(0,1)).
    """
    rng = np.random.default_rng(seed)
    if n == 0:
        return np.zeros(0, dtype=np.float32)
    if kind == "normal":
        return (rng.standard_normal(n, dtype=np.float32) * np.float32(sigma)).astype(np.float32)
    if kind == "model-like":
        g = rng.standard_normal(n, dtype=np.float32)
        nchunk = (n + 4095) // 4096
        sig = (10.0 ** rng.uniform(-4, -2, size=nchunk)).astype(np.float32)
        g *= np.repeat(sig, 4096)[:n]
        m = max(1, int(n * 1e-4))
        g[rng.integers(0, n, size=m)] *= np.float32(100.0)
        return g
    if kind == "zipf-rows":
        d = 64
        rows = (n + d - 1) // d
        g = np.zeros(rows * d, dtype=np.float32)
        live = _zipf_rows(rng, rows, max(1, rows // 10))
        mat = g.reshape(rows, d)
        mat[live] = rng.standard_normal((live.size, d), dtype=np.float32) * np.float32(1e-3)
        return g[:n].copy()
    if kind == "ties":
        mags = np.array([0.0, 0.25, 0.5, 1.0, 1.5, 3.0, 1e-3], dtype=np.float32)
        g = mags[rng.integers(0, mags.size, size=n)]
        return (g * np.where(rng.random(n) < 0.5, -1, 1).astype(np.float32)).astype(np.float32)
    if kind == "zeros":
        return np.zeros(n, dtype=np.float32)
    if kind == "subnormal":
        return (rng.standard_normal(n).astype(np.float32) * np.float32(1e-40)).astype(np.float32)
    if kind == "mixed-scale":
        return (rng.standard_normal(n) * 10.0 ** rng.uniform(-30, 3, size=n)).astype(np.float32)
    if kind == "signed-zero":
        g = np.where(rng.random(n) < 0.5, np.float32(-0.0), np.float32(0.0)).astype(np.float32)
        m = max(1, n // 100)
        g[rng.integers(0, n, size=m)] = rng.standard_normal(m).astype(np.float32)
        return g
    if kind == "uniform":
        return rng.uniform(-1.0, 1.0, size=n).astype(np.float32)
    if kind == "tiny-max":
        return (rng.uniform(-1.0, 1.0, size=n) * 1e-44).astype(np.float32)
    if kind == "fp8-ties":
        # max |g| = 1 and every other value within a few ulps of (midpoint between two
        # neighbouring E4M3 magnitudes) / 448: with a max-abs/448 scale the quotients sit on or
        # next to E4M3 rounding boundaries (adversarial for any shortcut around the IEEE division)
        grid = [mm * 2.0 ** -9 for mm in range(8)] + \
               [(8 + mm) * 2.0 ** (ee - 10) for ee in range(1, 16) for mm in range(8)]
        grid = np.array(grid[:-1] + [480.0])            # 448 is the last finite; 480 marks the 464 boundary
        mids = (grid[:-1] + grid[1:]) / 2.0
        g = (mids[rng.integers(0, mids.size, size=n)] / 448.0).astype(np.float32)
        g *= np.where(rng.random(n) < 0.5, -1.0, 1.0).astype(np.float32)
        steps = rng.integers(-3, 4, size=n)
        for d in (-3, -2, -1, 1, 2, 3):
            sel = steps == d
            toward = np.float32(np.inf) if d > 0 else np.float32(-np.inf)
            for _ in range(abs(d)):
                g[sel] = np.nextafter(g[sel], toward)
        g = np.clip(g, -1.0, 1.0).astype(np.float32)
        g[0] = np.float32(1.0)
        return g
    if kind == "e5m2-ties":
        # max |g| = 1 and every other value within a few ulps of (midpoint between two
        # neighbouring E5M2 magnitudes) / 57344 (the E5M2 analogue of "fp8-ties")
        grid = [mm * 2.0 ** -16 for mm in range(4)] + \
               [(4 + mm) * 2.0 ** (ee - 17) for ee in range(1, 31) for mm in range(4)]
        grid = np.array(grid + [65536.0])              # 57344 is the last finite; 65536 marks 61440
        mids = (grid[:-1] + grid[1:]) / 2.0
        g = (mids[rng.integers(0, mids.size, size=n)] / 57344.0).astype(np.float32)
        g *= np.where(rng.random(n) < 0.5, -1.0, 1.0).astype(np.float32)
        steps = rng.integers(-3, 4, size=n)
        for d in (-3, -2, -1, 1, 2, 3):
            sel = steps == d
            toward = np.float32(np.inf) if d > 0 else np.float32(-np.inf)
            for _ in range(abs(d)):
                g[sel] = np.nextafter(g[sel], toward)
        g = np.clip(g, -1.0, 1.0).astype(np.float32)
        g[0] = np.float32(1.0)
        return g
    if kind == "int-ties":
        # max |g| = 1 and every other value within a few ulps of k/127: quotients on or next to
        # integers (where a floor / fractional-part shortcut is most fragile)
        k = rng.integers(-127, 128, size=n).astype(np.float64)
        g = (k / 127.0).astype(np.float32)
        steps = rng.integers(-3, 4, size=n)
        for d in (-3, -2, -1, 1, 2, 3):
            sel = steps == d
            toward = np.float32(np.inf) if d > 0 else np.float32(-np.inf)
            for _ in range(abs(d)):
                g[sel] = np.nextafter(g[sel], toward)
        g = np.clip(g, -1.0, 1.0).astype(np.float32)
        g[0] = np.float32(1.0)
        return g
    if kind == "half-ties":
        # max |g| = 1 and every other value within a few ulps of (k + 1/2)/127: with a
        # max-abs/127 scale the quotients sit on or next to half-integers (adversarial for any
        # shortcut around an IEEE division followed by round-half-even)
        k = rng.integers(-127, 127, size=n).astype(np.float64)
        g = ((k + 0.5) / 127.0).astype(np.float32)
        steps = rng.integers(-3, 4, size=n)
        for d in (-3, -2, -1, 1, 2, 3):
            sel = steps == d
            toward = np.float32(np.inf) if d > 0 else np.float32(-np.inf)
            for _ in range(abs(d)):
                g[sel] = np.nextafter(g[sel], toward)
        g[0] = np.float32(1.0)
        return g
    if kind == "strided-small":
        # like strided-zeros, but the sampled elements are small and NONZERO: a regular sampler
        # sees a bracket far below the true k-th key (every other element is a "winner")
        g = rng.standard_normal(n, dtype=np.float32)
        g[::16] = (rng.standard_normal((n + 15) // 16, dtype=np.float32) * np.float32(1e-3)).astype(np.float32)
        return g
    if kind == "strided-zeros":
        # every element whose index is a multiple of 16 is 0.0, the rest N(0, 1): a regular
        # sampler with a power-of-two stride >= 16 sees only zeros (adversarial structure)
        g = rng.standard_normal(n, dtype=np.float32)
        g[::16] = 0.0
        return g
    raise ValueError(f"unknown kind {kind!r}")


def fixed_buckets(total: int, bucket_bytes: int, elem_bytes: int = 4, multiple: int = 4):
    """Split a flat buffer of ``total`` elements into fixed-size buckets of
    ``bucket_bytes`` (the last one ragged), each a multiple of ``multiple`` elements
    except possibly the last.  This is a contiguous-gradient-buffer bucketing (ZeRO-
    style), not per-tensor; see DESIGN.md "Bucketing"."""
    per = max(multiple, (bucket_bytes // elem_bytes) // multiple * multiple)
    sizes = [per] * (total // per)
    if total % per:
        sizes.append(total % per)
    return sizes
