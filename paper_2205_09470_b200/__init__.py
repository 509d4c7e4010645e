"""paper_2205_09470_b200 — B200-native compressed gradient sync (Nebula-I hot path).

Thin ctypes binding over ``libnebula_sync.so`` (C ABI: ``include/nebula_sync.h``).  It only
marshals arguments: every step of the path runs in the library's sm_100a kernels and NCCL.
There is no CPU or PyTorch fallback — if the library is missing, importing the binding's
``load()`` raises.  PyTorch is used only for device memory (tensors whose ``data_ptr`` is
passed through), streams and ``torch.distributed`` (to broadcast the NCCL unique id).

Names follow the C ABI: ``SyncContext.compress`` == ``nebula_compress`` etc.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

__all__ = [
    "IDENTITY", "FP16", "INT8", "TOPK", "FP8", "QSGD", "FP8_E5M2", "VAL_F32", "VAL_F16", "VAL_I8", "NCCL", "LOOPBACK", "SELF",
    "ALL_BUCKETS", "NebulaError", "load", "lib_path", "get_unique_id", "SyncContext", "TopkInfo",
    "status_string", "abi_version", "HEADER", "SvdCodec", "SVD_FP16",
]

HERE = os.path.dirname(os.path.abspath(__file__))
HEADER = os.path.join(os.path.dirname(HERE), "include", "nebula_sync.h")

IDENTITY, FP16, INT8, TOPK, FP8 = 0, 1, 2, 3, 4
QSGD = 6
FP8_E5M2 = 7
VAL_F32, VAL_F16, VAL_I8 = 0, 1, 2
NCCL, LOOPBACK, SELF = 0, 1, 2
SVD_FP16 = 5   # payload method id of the FP16(SVD(rho)) compressor (R31)
ALL_BUCKETS = -1
OPT_INT8_KERNEL = 1
OPT_EXCHANGE = 2
OPT_FP16_KERNEL = 3
OPT_STEP_FUSION = 4
OPT_EXACT_SCALE = 5
OPT_SR_SEED = 6
OPT_TOPK_REDUCE = 7
OPT_INTRA = 8
OPT_PIPELINE = OPT_TOPK_PIPELINE = 9
OPT_TOPK_STAGE = 10
CODEC_EXACT_TOPK = 1   # NEBULA_CODEC_EXACT_TOPK (NEXT-3, R34)
EXCHANGE_MODES = {0: "loopback", 1: "nccl-allgather", 2: "p2p-push", 3: "p2p-pull"}
UNIQUE_ID_BYTES = 128

STATUS = {0: "OK", 1: "INVALID_ARG", 2: "STATE", 3: "OOM", 4: "CUDA", 5: "NCCL",
          6: "NONFINITE", 7: "OVERFLOW", 8: "UNSUPPORTED"}


class NebulaError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status
        self.code = STATUS.get(status, str(status))


class _Codec(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int32), ("topk_values", ctypes.c_int32), ("topk_k", ctypes.c_uint64),
                ("topk_density", ctypes.c_double), ("error_feedback", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("start_step", ctypes.c_uint64)]


class _Topology(ctypes.Structure):
    _fields_ = [("num_clusters", ctypes.c_int32), ("cluster_id", ctypes.c_int32),
                ("gpus_per_cluster", ctypes.c_int32), ("local_rank", ctypes.c_int32),
                ("transport", ctypes.c_int32), ("device", ctypes.c_int32), ("nccl_unique_id", ctypes.c_void_p)]


class _TopkInfo(ctypes.Structure):
    _fields_ = [("k", ctypes.c_uint64), ("threshold", ctypes.c_uint32), ("reserved", ctypes.c_uint32),
                ("count_above", ctypes.c_uint64), ("need", ctypes.c_uint64), ("candidates", ctypes.c_uint64),
                ("path", ctypes.c_uint32), ("reserved2", ctypes.c_uint32)]


class _PhaseTime(ctypes.Structure):
    _fields_ = [("phase", ctypes.c_uint32), ("count", ctypes.c_uint32), ("ms", ctypes.c_double)]


@dataclass
class TopkInfo:
    k: int
    threshold: int
    count_above: int
    need: int
    candidates: int
    path: int


_lib = None


def lib_path() -> str:
    return os.path.join(HERE, "libnebula_sync.so")


def load() -> ctypes.CDLL:
    """Load the in-tree CUDA library; raise loudly if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -m paper_2205_09470_b200.build` "
                          "(the product path has no CPU fallback)")
    L = ctypes.CDLL(path)
    P, U64, I32, VP = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p
    sig = {
        "nebula_abi_version": (I32, []),
        "nebula_status_string": (ctypes.c_char_p, [I32]),
        "nebula_get_unique_id": (I32, [VP]),
        "nebula_sync_init": (I32, [ctypes.POINTER(P), ctypes.POINTER(_Topology), ctypes.POINTER(_Codec),
                                   ctypes.POINTER(U64), I32, VP]),
        "nebula_set_stream": (I32, [P, VP]),
        "nebula_compress": (I32, [P, I32, VP, U64]),
        "nebula_exchange": (I32, [P, I32]),
        "nebula_decompress_reduce": (I32, [P, I32, VP]),
        "nebula_step": (I32, [P, I32, VP, VP, U64]),
        "nebula_decompress": (I32, [P, I32, I32, VP]),
        "nebula_step_host": (I32, [P, VP, VP, U64]),
        "nebula_check": (I32, [P]),
        "nebula_payload_bytes": (I32, [P, I32, ctypes.POINTER(U64)]),
        "nebula_payload_copy": (I32, [P, I32, I32, VP, U64]),
        "nebula_residual_ptr": (I32, [P, I32, I32, ctypes.POINTER(ctypes.c_void_p)]),
        "nebula_topk_stats": (I32, [P, I32, I32, ctypes.POINTER(_TopkInfo)]),
        "nebula_kernel_launches": (U64, [P]),
        "nebula_timing_enable": (I32, [P, I32]),
        "nebula_set_option": (I32, [P, I32, ctypes.c_int64]),
        "nebula_exchange_mode": (I32, [P]),
        "nebula_intra_mode": (I32, [P]),
        "nebula_timing_read": (I32, [P, ctypes.POINTER(_PhaseTime), I32, ctypes.POINTER(I32)]),
        "nebula_phase_name": (ctypes.c_char_p, [ctypes.c_uint32]),
        "nebula_sync_destroy": (I32, [P]),
        "nebula_svd_init": (I32, [ctypes.POINTER(P), ctypes.c_int64, ctypes.c_int64, I32, I32, VP]),
        "nebula_svd_init_density": (I32, [ctypes.POINTER(P), ctypes.c_int64, ctypes.c_int64, ctypes.c_double, I32, VP]),
        "nebula_svd_rank": (I32, [ctypes.c_int64, ctypes.c_int64, ctypes.c_double]),
        "nebula_svd_set_stream": (I32, [P, VP]),
        "nebula_svd_payload_bytes": (I32, [P, ctypes.POINTER(U64)]),
        "nebula_svd_compress": (I32, [P, VP, VP]),
        "nebula_svd_decompress": (I32, [P, VP, VP]),
        "nebula_svd_check": (I32, [P]),
        "nebula_svd_kernel_launches": (U64, [P]),
        "nebula_svd_set_eigensolver": (I32, [P, I32]),
        "nebula_svd_destroy": (I32, [P]),
        "nebula_svd_last_error": (ctypes.c_char_p, [P]),
        "nebula_last_error": (ctypes.c_char_p, [P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    _lib = L
    return L


def abi_version() -> int:
    return load().nebula_abi_version()


def status_string(s: int) -> str:
    return load().nebula_status_string(s).decode()


def _err(ctx_ptr) -> str:
    m = load().nebula_last_error(ctx_ptr)
    return m.decode() if m else ""


def get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(UNIQUE_ID_BYTES)
    s = load().nebula_get_unique_id(buf)
    if s:
        raise NebulaError(s, _err(None))
    return buf.raw


def _ptr(x) -> int:
    """Device/host pointer of a torch tensor, or an int address (passed through unchecked)."""
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    return x.data_ptr()


def _dev_f32(x, device: int, min_numel: int, what: str) -> int:
    """Pointer of a caller buffer after the checks the C ABI cannot make: fp32, contiguous, on
    the context's device, at least `min_numel` elements (the library reads / writes exactly
    that many; a smaller buffer would be an out-of-bounds device access).  Ints pass through."""
    if x is None or isinstance(x, int):
        return _ptr(x)
    import torch
    if x.dtype != torch.float32:
        raise ValueError(f"{what}: expected torch.float32, got {x.dtype}")
    if not x.is_contiguous():
        raise ValueError(f"{what}: must be contiguous")
    if x.device.type != "cuda" or x.device.index != device:
        raise ValueError(f"{what}: must live on cuda:{device}, got {x.device}")
    if x.numel() < min_numel:
        raise ValueError(f"{what}: {x.numel()} elements, the call needs {min_numel}")
    return x.data_ptr()


def _stream_handle(stream, device):
    if stream is None:
        import torch
        if not torch.cuda.is_available():
            return 0      # validation-only use on a CPU box: init fails before any CUDA call
        return torch.cuda.current_stream(device).cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class SyncContext:
    """One ``nebula_ctx``.  Arguments mirror ``nebula_topology`` / ``nebula_codec``."""

    def __init__(self, bucket_numel, method=INT8, *, topk_values=VAL_F32, topk_k=0, topk_density=0.01,
                 error_feedback=True, start_step=0, exact_topk=False, num_clusters=2, cluster_id=0, gpus_per_cluster=1,
                 local_rank=0, transport=LOOPBACK, device=0, unique_id: bytes | None = None, stream=None):
        L = load()
        self._L = L
        self.bucket_numel = [int(n) for n in bucket_numel]
        self.num_clusters, self.cluster_id = num_clusters, cluster_id
        self.gpus_per_cluster, self.local_rank = gpus_per_cluster, local_rank
        self.transport, self.device = transport, device
        self.exact_topk = bool(exact_topk)
        self.codec = _Codec(method, topk_values, int(topk_k), float(topk_density), int(bool(error_feedback)),
                            CODEC_EXACT_TOPK if exact_topk else 0, int(start_step))
        self._uid = ctypes.create_string_buffer(unique_id, UNIQUE_ID_BYTES) if unique_id is not None else None
        topo = _Topology(num_clusters, cluster_id, gpus_per_cluster, local_rank, transport, device,
                         ctypes.cast(self._uid, ctypes.c_void_p) if self._uid is not None else None)
        arr = (ctypes.c_uint64 * len(self.bucket_numel))(*self.bucket_numel)
        h = ctypes.c_void_p()
        st = _stream_handle(stream, device)
        s = L.nebula_sync_init(ctypes.byref(h), ctypes.byref(topo), ctypes.byref(self.codec), arr,
                               len(self.bucket_numel), st)
        if s:
            raise NebulaError(s, _err(None))
        self._h = h

    # ------------------------------------------------------------------ helpers
    def _ck(self, s):
        if s:
            raise NebulaError(s, _err(self._h))

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream):
        self._ck(self._L.nebula_set_stream(self._h, _stream_handle(stream, self.device)))

    # ------------------------------------------------------------------ stages
    def _elems(self, bucket) -> int:
        return sum(self.bucket_numel) if bucket == ALL_BUCKETS else self.bucket_numel[bucket]

    def _grad(self, bucket, grad) -> int:
        stacked = self.num_clusters if self.transport == LOOPBACK else 1   # LOOPBACK: [P][elems]
        return _dev_f32(grad, self.device, stacked * self._elems(bucket), "grad")

    def _out(self, bucket, out) -> int:
        return _dev_f32(out, self.device, self._elems(bucket), "out")

    def compress(self, bucket, grad, step):
        self._ck(self._L.nebula_compress(self._h, bucket, self._grad(bucket, grad), step))

    def exchange(self, bucket):
        self._ck(self._L.nebula_exchange(self._h, bucket))

    def decompress_reduce(self, bucket, out):
        self._ck(self._L.nebula_decompress_reduce(self._h, bucket, self._out(bucket, out)))

    def decompress(self, bucket, slot, out):
        """Decode one cluster's payload (no averaging): the pipeline-hop use (NEXT-2)."""
        self._ck(self._L.nebula_decompress(self._h, bucket, slot, self._out(bucket, out)))

    def step(self, bucket, grad, out, step):
        self._ck(self._L.nebula_step(self._h, bucket, self._grad(bucket, grad), self._out(bucket, out), step))

    def step_host(self, host_grad, host_out, step):
        """host_grad / host_out: CPU tensors (pinned for full bandwidth) or numpy arrays."""
        g = host_grad.ctypes.data if hasattr(host_grad, "ctypes") else host_grad.data_ptr()
        o = host_out.ctypes.data if hasattr(host_out, "ctypes") else host_out.data_ptr()
        self._ck(self._L.nebula_step_host(self._h, g, o, step))

    def check(self):
        """Synchronise; raise NebulaError(NONFINITE/OVERFLOW) if the device flagged one."""
        self._ck(self._L.nebula_check(self._h))

    def check_status(self) -> int:
        return self._L.nebula_check(self._h)

    def payload_bytes(self, bucket) -> int:
        v = ctypes.c_uint64()
        self._ck(self._L.nebula_payload_bytes(self._h, bucket, ctypes.byref(v)))
        return v.value

    def payload_copy(self, bucket, slot) -> bytes:
        n = self.payload_bytes(bucket)
        buf = ctypes.create_string_buffer(max(n, 1))
        self._ck(self._L.nebula_payload_copy(self._h, bucket, slot, buf, n))
        return buf.raw[:n]

    def residual_ptr(self, bucket, cluster) -> int:
        p = ctypes.c_void_p()
        self._ck(self._L.nebula_residual_ptr(self._h, bucket, cluster, ctypes.byref(p)))
        return p.value or 0

    def residual(self, bucket, cluster):
        """A torch view (no copy) of the library-owned residual (checkpoint / restore it)."""
        import torch
        exact = self.exact_topk and self.codec.method == TOPK
        n = self.bucket_numel[bucket] // (1 if exact else self.gpus_per_cluster)
        ptr = self.residual_ptr(bucket, cluster)

        class _CAI:
            __cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3}
        return torch.as_tensor(_CAI(), device=f"cuda:{self.device}")

    def topk_stats(self, bucket, cluster) -> TopkInfo:
        info = _TopkInfo()
        self._ck(self._L.nebula_topk_stats(self._h, bucket, cluster, ctypes.byref(info)))
        return TopkInfo(info.k, info.threshold, info.count_above, info.need, info.candidates, info.path)

    def kernel_launches(self) -> int:
        return self._L.nebula_kernel_launches(self._h)

    def set_option(self, option: int, value: int):
        self._ck(self._L.nebula_set_option(self._h, option, value))

    def set_int8_kernel(self, which: str):
        """'auto' | 'two-pass' | 'single-pass' (= 'onchip' = 'fused-ws': the warp-specialised
        TMA kernel) (NEBULA_OPT_INT8_KERNEL; INT8, FP8 and QSGD)."""
        self.set_option(OPT_INT8_KERNEL, {"auto": 0, "two-pass": 1, "single-pass": 2, "onchip": 2,
                                          "fused-ws": 2}[which])

    def set_fp16_kernel(self, which: str):
        """'tma' (default) | 'plain' (NEBULA_OPT_FP16_KERNEL)."""
        self.set_option(OPT_FP16_KERNEL, {"tma": 0, "plain": 1}[which])

    def set_step_fusion(self, on: bool):
        """True (default): step() runs INT8 compress + exchange + reduce as one kernel where
        eligible; False: three stage launches (NEBULA_OPT_STEP_FUSION)."""
        self.set_option(OPT_STEP_FUSION, 0 if on else 1)

    def set_exact_scale(self, on: bool):
        """Hierarchical (G > 1) INT8/FP8: True = the scale of the whole cluster bucket (one
        4-byte-per-bucket intra-cluster all-reduce of the maxima, NEBULA_OPT_EXACT_SCALE);
        False (default) = per-shard scales."""
        self.set_option(OPT_EXACT_SCALE, int(bool(on)))

    def set_sr_seed(self, seed: int):
        """Seed of the QSGD stochastic-rounding uniforms (NEBULA_OPT_SR_SEED)."""
        self.set_option(OPT_SR_SEED, int(seed) - (1 << 64) if int(seed) >= (1 << 63) else int(seed))

    def set_intra(self, which: str):
        """G > 1: 'p2p' (default: fixed-order reduce-scatter / all-gather over NVLink peer
        memory) | 'nccl' (NEBULA_OPT_INTRA)."""
        self.set_option(OPT_INTRA, {"p2p": 0, "auto": 0, "nccl": 1}[which])

    def set_exchange(self, which: str):
        """'auto' | 'nccl' | 'push' | 'pull' (NEBULA_OPT_EXCHANGE; between steps only)."""
        self.set_option(OPT_EXCHANGE, {"auto": 0, "nccl": 1, "push": 2, "pull": 3, "p2p": 3}[which])

    def exchange_mode(self) -> str:
        return EXCHANGE_MODES[self._L.nebula_exchange_mode(self._h)]

    def intra_mode(self) -> str:
        return {0: "none", 1: "nccl", 2: "p2p"}[self._L.nebula_intra_mode(self._h)]

    def timing_enable(self, on: bool = True):
        self._ck(self._L.nebula_timing_enable(self._h, int(bool(on))))

    def timing_read(self) -> dict:
        """{phase name: (launches, summed ms)} since the last read (synchronises)."""
        buf = (_PhaseTime * 64)()
        n = ctypes.c_int32()
        self._ck(self._L.nebula_timing_read(self._h, buf, 64, ctypes.byref(n)))
        return {self._L.nebula_phase_name(buf[i].phase).decode(): (buf[i].count, buf[i].ms) for i in range(n.value)}

    def destroy(self):
        if getattr(self, "_h", None):
            self._L.nebula_sync_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def broadcast_unique_id(src: int = 0, group=None) -> bytes:
    """Rank `src` creates the NCCL unique id (nebula_get_unique_id); torch.distributed
    broadcasts the 128 bytes to every rank (plumbing only; works on gloo or nccl)."""
    import torch.distributed as dist
    uid = [get_unique_id() if dist.get_rank() == src else None]
    dist.broadcast_object_list(uid, src=src, group=group)
    return uid[0]


def self_group_id() -> bytes:
    """A fresh 128-byte group id for SELF-transport contexts (any bytes shared by the group)."""
    return os.urandom(UNIQUE_ID_BYTES)


def self_group(bucket_numel, *, num_clusters, gpus_per_cluster=1, device=0, streams=None, **codec):
    """All P x G contexts of one SELF-transport group on `device` (one process; every P2P path
    of the NCCL transport runs on one GPU).  Returns [[ctx of (cluster c, local rank l)]];
    streams[c][l] (torch streams) default to fresh ones — members need their own streams."""
    import torch
    gid = self_group_id()
    P, G = num_clusters, gpus_per_cluster
    out = []
    for c in range(P):
        row = []
        for l in range(G):
            st = streams[c][l] if streams is not None else torch.cuda.Stream(device=device)
            row.append(SyncContext(bucket_numel, num_clusters=P, cluster_id=c, gpus_per_cluster=G, local_rank=l,
                                   transport=SELF, device=device, unique_id=gid, stream=st, **codec))
            row[-1].stream = st
        out.append(row)
    return out


def topology_for_rank(rank: int, world: int, gpus_per_cluster: int = 1):
    """(num_clusters, cluster_id, local_rank) of a rank: cluster r // G, local rank r % G
    (G = 1 -> topology A, G > 1 -> topology B)."""
    G = gpus_per_cluster
    if G < 1 or world % G:
        raise ValueError("world size must be a positive multiple of gpus_per_cluster")
    return world // G, rank // G, rank % G


def init_process_group_context(bucket_numel, *, gpus_per_cluster=1, device=None, **codec):
    """Build a NCCL-transport context for this torch.distributed rank."""
    import torch
    import torch.distributed as dist
    P, c, l = topology_for_rank(dist.get_rank(), dist.get_world_size(), gpus_per_cluster)
    uid = broadcast_unique_id()
    if device is None:
        device = torch.cuda.current_device()
    return SyncContext(bucket_numel, num_clusters=P, cluster_id=c, gpus_per_cluster=gpus_per_cluster,
                       local_rank=l, transport=NCCL, device=device, unique_id=uid, **codec)


class SvdCodec:
    """One ``nebula_svd`` handle: the FP16(SVD(rho)) compressor of an m x n fp32 matrix
    (NEXT-1; Eq. 1-5).  ``r`` = kept singular triples (or pass ``rho`` for R29's
    r = clamp(floor(rho min(m, n) + 0.5), 1, min(m, n)))."""

    def __init__(self, m: int, n: int, r: int | None = None, *, rho: float | None = None, device=0, stream=None):
        L = load()
        self._L = L
        self.m, self.n, self.device = int(m), int(n), device
        h = ctypes.c_void_p()
        if r is None:   # R29 is computed by the library (nebula_svd_init_density)
            s = L.nebula_svd_init_density(ctypes.byref(h), self.m, self.n, float(rho), device,
                                          _stream_handle(stream, device))
            r = L.nebula_svd_rank(self.m, self.n, float(rho))
        else:
            s = L.nebula_svd_init(ctypes.byref(h), self.m, self.n, int(r), device, _stream_handle(stream, device))
        if s:
            raise NebulaError(s, L.nebula_svd_last_error(None).decode())
        self.r = int(r)
        self._h = h

    def _ck(self, s):
        if s:
            raise NebulaError(s, self._L.nebula_svd_last_error(self._h).decode())

    def payload_bytes(self) -> int:
        b = ctypes.c_uint64()
        self._ck(self._L.nebula_svd_payload_bytes(self._h, ctypes.byref(b)))
        return b.value

    def compress(self, A, payload):
        """A: fp32 [m, n] CUDA tensor (row-major); payload: uint8 CUDA tensor of payload_bytes()."""
        self._ck(self._L.nebula_svd_compress(self._h, _ptr(A), _ptr(payload)))

    def decompress(self, payload, out):
        self._ck(self._L.nebula_svd_decompress(self._h, _ptr(payload), _ptr(out)))

    def set_stream(self, stream):
        self._ck(self._L.nebula_svd_set_stream(self._h, _stream_handle(stream, self.device)))

    def check(self):
        self._ck(self._L.nebula_svd_check(self._h))

    def kernel_launches(self) -> int:
        return self._L.nebula_svd_kernel_launches(self._h)

    def set_eigensolver(self, which: str, gram: str = "dmma"):
        """which: 'syevd' (default, divide and conquer) | 'syevj' (Jacobi); gram: 'dmma' (FP64
        tensor cores, default) | 'simt' (fp64 FMA)."""
        self._ck(self._L.nebula_svd_set_eigensolver(self._h, {"syevd": 0, "syevj": 1}[which] +
                                                    2 * {"dmma": 0, "simt": 1}[gram]))

    def destroy(self):
        if getattr(self, "_h", None):
            self._L.nebula_svd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass
