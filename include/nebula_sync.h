/*
 * nebula_sync.h — C ABI of the B200-native compressed gradient sync (Nebula-I hot path).
 *
 * What the library computes (arXiv 2205.09470, "Nebula-I"; PAPER.md = /root/reference/PAPER.md,
 * SPEC.md = /root/reference/SPEC.md; R-numbers are DESIGN.md readings == SURVEY.md §8(c) C-numbers):
 *
 *   For every cluster c (a group of G GPUs; P clusters), every gradient bucket b of n fp32
 *   elements, and optimisation step t:
 *     method = IDENTITY if t < start_step else codec.method
 *     p      = fl(g + r)                                             error feedback, R15
 *     payload_c = C(p)   FP16  : RNE binary16                        PAPER.md:125-130 Eq. 5
 *                        INT8  : per-bucket symmetric max-abs scale
 *                        TOPK  : k largest |p|, ties -> lower index  PAPER.md:63, :99 (cited), R11-R14
 *     r      = fl(p - D(C(p)))                                       R15
 *     exchange payload_c between clusters                            PAPER.md:76 "gradients are aggregated",
 *                                                                    PAPER.md:95 data parallelism across clusters
 *     out    = fl(tree_sum_c D(payload_c) / P)                       R16 (fixed pairwise tree over cluster ids)
 *
 *   With G > 1 (hierarchical): the cluster gradient is the fp32 mean of its G GPUs, summed in
 *   local-rank order then divided by G (R20: an intra-cluster reduce-scatter over NVLink peer
 *   memory; NCCL ReduceScatter(avg), whose order is NCCL's, only when the peers cannot be
 *   mapped), GPU l codes shard l (n/G elements) with its own residual, exchanges it with the
 *   P-1 peers of the same local rank, and the averaged shards are all-gathered inside the
 *   cluster (R20).
 *
 * Payload body (R18): 16-byte preamble {u32 method, u32 count (n or k), f32 scale (1.0 if
 * unused), u32 aux (TOPK value type, else 0)}, then sections zero-padded to 16 bytes:
 * IDENTITY f32[n] | FP16 binary16[n] | INT8 / QSGD int8[n] | FP8 E4M3 / E5M2 u8[n] | TOPK u32 idx[k] (ascending) then
 * val[k] (f32 | binary16 | int8).  All little-endian.  Identical on every transport.
 *
 * Conventions for every entry point:
 *   - Pointers named dev_* are CUDA device pointers on the context's device; host_* are
 *     host pointers.  Nothing is retained past the call except through the context.
 *   - Every call only ENQUEUES work on the context's stream and returns, except
 *     nebula_check, nebula_payload_copy, nebula_topk_stats and nebula_step_host, which
 *     synchronise that stream.  One host thread per context.
 *   - Host-validated errors return immediately with nothing enqueued.  Device-detected
 *     errors (non-finite p, fp16 overflow, a P2P peer timeout) set a sticky device flag returned
 *     by nebula_check (which clears it) and, without any synchronisation, by the next
 *     compress / step call once the step that raised it has completed: every step and
 *     decompress_reduce ends with an asynchronous 4-byte copy of the flag word into pinned
 *     host memory, which the next stage call reads before enqueuing anything.  After a device error the affected buckets' residuals
 *     and dev_out are unspecified (the caller skips the step and zeroes or restores the
 *     residual via nebula_residual_ptr); INT8 writes no payload for such a bucket.
 *   - No C++ exception crosses the ABI.  nebula_last_error() describes the last failure.
 *   - Per bucket the order must be compress -> exchange -> decompress_reduce; anything
 *     else returns NEBULA_ERR_STATE.  nebula_step runs all three.
 *   - bucket == NEBULA_ALL_BUCKETS (-1) applies a call to every bucket in one segmented
 *     launch per stage; the buckets are then laid out back to back (in init order) in the
 *     caller's flat buffers.
 */
#ifndef NEBULA_SYNC_H_
#define NEBULA_SYNC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NEBULA_ABI_VERSION 1
#define NEBULA_ALL_BUCKETS (-1)
#define NEBULA_MAX_CLUSTERS 8
#define NEBULA_UNIQUE_ID_BYTES 128

typedef struct nebula_ctx nebula_ctx; /* opaque, library-owned */

typedef enum {
  NEBULA_OK = 0,
  NEBULA_ERR_INVALID_ARG = 1, /* host-validated; nothing enqueued */
  NEBULA_ERR_STATE = 2,       /* call order violated for a bucket */
  NEBULA_ERR_OOM = 3,
  NEBULA_ERR_CUDA = 4,
  NEBULA_ERR_NCCL = 5,
  NEBULA_ERR_NONFINITE = 6,   /* device-detected NaN/Inf in p = g + r   (sticky) */
  NEBULA_ERR_OVERFLOW = 7,    /* device-detected fp16 overflow |p| >= 65520 (R10) */
  NEBULA_ERR_UNSUPPORTED = 8  /* e.g. NCCL transport in a build/box without peers */
} nebula_status;

/* NEBULA_FP8 (NEXT-4; R27, "8-bit floating point to represent each gradient"):
 * OCP E4M3, one per-bucket scale s = fl(max|p| / 448) (s := 1 if max == 0 or underflow),
 * code = RNE-to-E4M3(fl(p / s)) saturating at +-448, D = fl(E4M3(code) * s).  Body: u8[n]. */
/* NEBULA_QSGD (NEXT-4; R32, QSGD is cited at PAPER.md:63, :99): INT8's scale and payload
 * (method id 6), with stochastic instead of nearest rounding: x = fl(p / s),
 * q = floor(x) + [u < x - floor(x)] clamped to [-127, 127], u the counter-based SplitMix64
 * uniform (2^-24 grid) of (seed = NEBULA_OPT_SR_SEED, step, cluster, bucket, shard, element):
 * base = sm(seed ^ sm(step ^ sm(((cluster * 65536 + shard) << 32) | bucket))),
 * h_j = sm(base + j * 0x9E3779B97F4A7C15), u_{2j} = (h_j >> 40) * 2^-24,
 * u_{2j+1} = ((h_j >> 16) & 0xFFFFFF) * 2^-24.  E[D] = p (unbiased).
 * (5 is the FP16(SVD) payload id, not a bucket method.) */
/* NEBULA_FP8_E5M2 (NEXT-4; R33): OCP E5M2, s = fl(max|p| / 57344) (R4 rules),
 * code = RNE-to-E5M2(fl(p / s)) saturating at +-57344 (never an infinity code),
 * D = fl(E5M2(code) * s).  Body: u8[n]. */
typedef enum { NEBULA_IDENTITY = 0, NEBULA_FP16 = 1, NEBULA_INT8 = 2, NEBULA_TOPK = 3, NEBULA_FP8 = 4,
               NEBULA_QSGD = 6, NEBULA_FP8_E5M2 = 7 } nebula_method;
typedef enum { NEBULA_VAL_F32 = 0, NEBULA_VAL_F16 = 1, NEBULA_VAL_I8 = 2 } nebula_value_type;
/* Transports.  NCCL: one process per GPU (torchrun); peers' buffers are mapped with CUDA IPC
 * when every rank can reach every peer (NVLink), else NCCL collectives move the bytes.
 * LOOPBACK: one context simulates all P clusters (G = 1) on its device.  SELF: one context per
 * (cluster, GPU) inside ONE process, all created with the same 128-byte group id in
 * nccl_unique_id (any bytes; the group is these contexts) — the contexts reach each other's
 * buffers directly (same device, or peer-accessible devices), so the P2P exchange, the flag
 * protocol and the intra-cluster hop run exactly as across processes.  SELF rules: the first
 * stage call needs every member to exist (else NEBULA_ERR_STATE); members run on their own
 * streams and the caller enqueues each stage for every member before waiting on any (a
 * member's exchange waits for its peers' compress); nebula_step runs the staged kernels;
 * destroy every member only after synchronising all of them. */
typedef enum { NEBULA_TRANSPORT_NCCL = 0, NEBULA_TRANSPORT_LOOPBACK = 1, NEBULA_TRANSPORT_SELF = 2 } nebula_transport;

/* Codec (SPEC.md:111-122 CodecMethod / CodecSchedule, extended with TOPK and error feedback). */
typedef struct {
  int32_t method;          /* nebula_method */
  int32_t topk_values;     /* nebula_value_type; TOPK only (R13) */
  uint64_t topk_k;         /* >0: exact k per coded bucket (capped at n); 0: derive from density */
  double topk_density;     /* rho in (0,1]; k = clamp(floor(rho*n + 0.5), 1, n)  (R12) */
  int32_t error_feedback;  /* 1: p = g + r and r <- p - D(C(p)) (R15); 0: p = g, no residual */
  int32_t flags;           /* NEBULA_CODEC_* bits (0 = defaults) */
  uint64_t start_step;     /* IDENTITY while step < start_step */
} nebula_codec;

/* NEBULA_CODEC_EXACT_TOPK (NEXT-3, R34; TOPK with G > 1): the selection is the top-k of the
 * WHOLE cluster bucket (k from the bucket's numel) instead of k/G per GPU shard (R20).  Every
 * GPU of the cluster all-gathers the fixed-order cluster mean, codes the whole bucket with the
 * cluster's full residual (replicated on the G GPUs, bit-identical), exchanges the full payload
 * with its inter-cluster peers and averages the whole bucket (no intra all-gather afterwards).
 * Cost: G x the per-GPU codec work and inter-cluster bytes of the per-shard reading.  Ignored
 * when G == 1 (the same thing).  Residual length (nebula_residual_ptr): numel. */
#define NEBULA_CODEC_EXACT_TOPK 1

/* Topology: P clusters x G GPUs.  Global rank = cluster_id * G + local_rank. */
typedef struct {
  int32_t num_clusters;     /* P, 1..NEBULA_MAX_CLUSTERS */
  int32_t cluster_id;       /* 0..P-1 (ignored for LOOPBACK: this device hosts all P) */
  int32_t gpus_per_cluster; /* G >= 1; G > 1 => hierarchical (NCCL or SELF; every numel % G == 0;
                               the P2P intra-cluster hop needs G <= 8) */
  int32_t local_rank;       /* 0..G-1 */
  int32_t transport;        /* nebula_transport */
  int32_t device;           /* CUDA device ordinal the context lives on */
  const void* nccl_unique_id; /* NEBULA_UNIQUE_ID_BYTES, identical on all P*G ranks (SELF: the group
                                 id); NULL for LOOPBACK */
} nebula_topology;

/* Integer order statistics of one top-k selection (R25 "ranks"). */
typedef struct {
  uint64_t k;           /* number of selected elements */
  uint32_t threshold;   /* key T = |p| bits of the k-th largest (sign cleared) */
  uint32_t reserved;
  uint64_t count_above; /* #{key > T} */
  uint64_t need;        /* k - count_above: how many key == T elements (lowest indices) were taken */
  uint64_t candidates;  /* diagnostic: elements that went through the exact resolution stage */
  uint32_t path;        /* diagnostic: 0 = sampled bracket, 1 = widened bracket */
  uint32_t reserved2;
} nebula_topk_info;

/* ABI version of the loaded library (== NEBULA_ABI_VERSION it was built with). */
int32_t nebula_abi_version(void);

/* Static string for a status code. Never NULL. */
const char* nebula_status_string(nebula_status s);

/* Writes an NCCL unique id (NEBULA_UNIQUE_ID_BYTES) to host_out128; rank 0 calls it and
 * broadcasts the bytes to all ranks out of band (the Python binding uses torch.distributed). */
nebula_status nebula_get_unique_id(void* host_out128);

/* Creates a context.  bucket_numel[num_buckets] are element counts (each < 2^31; 0 allowed).
 * Allocates and zeroes the residuals (library-owned, one per (cluster, bucket[, shard])),
 * payload slots and scratch; for NCCL builds the communicators (collective across all
 * P*G ranks).  stream is a cudaStream_t (NULL = legacy default stream) the context enqueues
 * on; it may be changed with nebula_set_stream.  On failure *out is NULL. */
nebula_status nebula_sync_init(nebula_ctx** out, const nebula_topology* topo, const nebula_codec* codec,
                               const uint64_t* bucket_numel, int32_t num_buckets, void* stream);

nebula_status nebula_set_stream(nebula_ctx* ctx, void* stream);

/* Stage 1 — EF-accumulate + compress + pack (+ the G>1 intra-cluster reduce-scatter).
 * NEBULA_ERR_STATE if a bucket of the call is not idle (compress twice without the other
 * stages would apply the residual twice) or, for ALL, the buckets are at different step
 * counts (a mix of per-bucket and ALL calls); nothing is enqueued then.
 * dev_grad: fp32 gradient of the bucket (or of all buckets, back to back, for
 * NEBULA_ALL_BUCKETS).  LOOPBACK: P stacked copies, cluster-major: [P][bucket elems]
 * (for ALL: [P][sum of all bucket elems]).  16-byte alignment enables the vector path;
 * any alignment is accepted.  Not modified.  May be freed once the stream work completes. */
nebula_status nebula_compress(nebula_ctx* ctx, int32_t bucket, const float* dev_grad, uint64_t step);

/* Stage 2 — move every cluster's payload to every cluster (NCCL AllGather over the
 * inter-cluster communicator, in place; LOOPBACK: nothing to move). */
nebula_status nebula_exchange(nebula_ctx* ctx, int32_t bucket);

/* Stage 3 — decode all P payload slots, tree-sum, divide by P, write dev_out (fp32, the
 * bucket's elements; ALL: back to back) (+ the G>1 intra-cluster all-gather).  dev_out may
 * alias dev_grad (non-LOOPBACK) . */
nebula_status nebula_decompress_reduce(nebula_ctx* ctx, int32_t bucket, float* dev_out);

/* Decode ONE cluster's payload slot into dev_out without averaging: fp32, the bucket's
 * elements (ALL: back to back), +0.0 where top-k did not select.  The pipeline-hop use of the
 * codecs ("FP16 quantization was used for feed-forward
 * activation compression ... INT8 quantization was used for back propagation gradient
 * compression", across the Scenario-II boundary PAPER.md:259) — compress with error_feedback
 * 0, exchange, then decompress the peer's slot.  Allowed after exchange (any slot) or after
 * compress (own slot; every slot for LOOPBACK).  Does not change the bucket's state.  With
 * G > 1 the shards are gathered with NCCL (NEBULA_ERR_UNSUPPORTED on SELF). */
nebula_status nebula_decompress(nebula_ctx* ctx, int32_t bucket, int32_t slot, float* dev_out);

/* All three stages.  Same results, bit for bit, as compress + exchange + decompress_reduce.
 * For INT8 / FP8 / QSGD with 16-B aligned pointers, buckets averaging >= 1M elements, G = 1 and
 * a LOOPBACK or (NCCL-transport) P2P pull exchange, the three stages run as ONE cooperative kernel
 * (NEBULA_OPT_STEP_FUSION): reduce warps average bucket b — pulling the peers' payloads over
 * NVLink once their system-scope arrival flags say they are complete — while the compress
 * warps of the same kernel stream bucket b+1.  A peer that never arrives sets the peer-timeout
 * flag after 60 s (nebula_check reports it). */
nebula_status nebula_step(nebula_ctx* ctx, int32_t bucket, const float* dev_grad, float* dev_out, uint64_t step);

/* All buckets, host buffers: copies host_grad (LOOPBACK: [P][total]) to the device, runs the
 * step, copies the average back to host_out ([total]) and synchronises.  Pipelined per bucket
 * over two copy streams and the context stream (bucket b+1 copies in while b is reduced and
 * b-1 copies out), so both PCIe directions overlap the GPU work.  Pinned host memory gives
 * full PCIe bandwidth and overlap; pageable works. */
nebula_status nebula_step_host(nebula_ctx* ctx, const float* host_grad, float* host_out, uint64_t step);

/* Synchronises the stream; returns and clears the sticky device error
 * (NEBULA_ERR_NONFINITE takes precedence over NEBULA_ERR_OVERFLOW), else NEBULA_OK. */
nebula_status nebula_check(nebula_ctx* ctx);

/* Size in bytes of one cluster's payload for a bucket (preamble + padded sections). */
nebula_status nebula_payload_bytes(const nebula_ctx* ctx, int32_t bucket, uint64_t* bytes);

/* Synchronises, then copies payload slot `slot` (cluster id 0..P-1) of a bucket to host
 * memory (cap >= nebula_payload_bytes).  Valid after compress (own slot; all slots for
 * LOOPBACK) or after exchange (all slots).  For oracle comparison and export. */
nebula_status nebula_payload_copy(nebula_ctx* ctx, int32_t bucket, int32_t slot, void* host_dst, uint64_t cap);

/* Device pointer to the residual of (bucket, cluster) — the caller saves / restores it with
 * its optimizer state (checkpointing) or zeroes it after a device error.  cluster is the
 * simulated cluster for LOOPBACK and must be the context's own cluster otherwise.  Length:
 * the coded elements of the bucket (numel, or numel/G when hierarchical without
 * NEBULA_CODEC_EXACT_TOPK). */
nebula_status nebula_residual_ptr(nebula_ctx* ctx, int32_t bucket, int32_t cluster, float** dev_residual);

/* Synchronises and returns the order statistics of the last TOPK compress of (bucket, cluster). */
nebula_status nebula_topk_stats(nebula_ctx* ctx, int32_t bucket, int32_t cluster, nebula_topk_info* out);

/* Number of library kernels enqueued since the context was created (bench accounting). */
uint64_t nebula_kernel_launches(const nebula_ctx* ctx);

/* Tuning knobs (results are bit-identical whichever kernel runs).
 *   NEBULA_OPT_INT8_KERNEL (INT8, FP8 E4M3 / E5M2 and QSGD): 0 auto (default), 1 two-pass streaming
 *   (max-abs pass + quantise pass, 21 B/elem of HBM traffic), 2 single pass: the
 *   warp-specialised TMA kernel (cooperative grid of one CTA per SM: a producer warp feeding
 *   two cp.async.bulk rings, max/park warps, quantise warps; 13 B/elem algorithmic; needs
 *   16-B aligned pointers, else two-pass).  Auto = 2 when buckets average >= 1M elements
 *   and pointers are 16-B aligned, else 1. */
#define NEBULA_OPT_INT8_KERNEL 1
/*   NEBULA_OPT_EXCHANGE (NCCL transport): 0 auto (default), 1 ncclAllGather of the payloads
 *   after the compress, 2 P2P push: the compress kernels store every payload word into the
 *   same slot of every peer's (CUDA-IPC-mapped) slot buffer over NVLink while they compute,
 *   3 P2P pull: compress writes locally, the decompress-reduce kernel loads each peer's slot
 *   directly from the peer over NVLink.  In 2 and 3 the exchange is a per-bucket flag
 *   handshake (release/acquire at system scope) and slots are double-buffered by step parity.
 *   Auto (every rank can map every peer, decided collectively at init): 2 for TOPK and, at
 *   P = 2, for IDENTITY / INT8 / FP8; 3 otherwise (P > 2, and FP16 / QSGD at P = 2); else 1.
 *   Only between steps. */
#define NEBULA_OPT_EXCHANGE 2
/*   NEBULA_OPT_FP16_KERNEL: 0 (default) TMA-ring streaming kernel for 16-B aligned calls,
 *   1 plain 128-bit-load streaming kernel. */
#define NEBULA_OPT_FP16_KERNEL 3
/*   NEBULA_OPT_STEP_FUSION: 0 (default) nebula_step fuses INT8 / FP8 / QSGD compress + exchange
 *   + reduce into one kernel where eligible (see nebula_step), 1 never (three stage launches),
 *   2..12 fused with warp split 0..10 of the kernel's tuning sweep (6 = split 4, the P2P-pull
 *   reducer with register loads; FP8 / QSGD take splits 0 and 4). */
#define NEBULA_OPT_STEP_FUSION 4
/*   NEBULA_OPT_EXACT_SCALE (NEXT-3, R28; hierarchical G > 1 only): 0 (default) every GPU's
 *   shard has its own INT8 / FP8 scale (R20); 1 the scale of the WHOLE cluster bucket: the
 *   max-abs pass runs on the shard, a 4-byte-per-bucket ncclAllReduce(max) over the
 *   intra-cluster communicator combines the G shards' maxima, then every shard quantises with
 *   that scale (two streaming passes instead of the single-pass INT8 kernel).  Payloads and
 *   residuals then equal the G = 1 compress of the cluster's mean gradient, shard by shard.
 *   Only between steps. */
#define NEBULA_OPT_EXACT_SCALE 5
/*   NEBULA_OPT_SR_SEED: the 64-bit seed of NEBULA_QSGD's uniforms (default 0); any time. */
#define NEBULA_OPT_SR_SEED 6
/*   NEBULA_OPT_TOPK_REDUCE: sparse decompress-average kernel, 0 tile-interleaved (per-tile run
 *   starts found in parallel, CTAs walk 2048-element tiles grid-stride), 1 (default) warps own
 *   contiguous ranges of 512-element sub-tiles (measured 0.30 vs 0.345 ms at BASELINE config 2).
 *   Same results. */
#define NEBULA_OPT_TOPK_REDUCE 7
/*   NEBULA_OPT_INTRA (G > 1): 0 (default) the intra-cluster reduce-scatter / all-gather over
 *   NVLink peer memory with a fixed summation order when every GPU of the cluster is mapped
 *   (SM-issued NVLink stores / loads), 1 NCCL ReduceScatter(avg) / AllGather (NCCL transport
 *   only).  Only between steps. */
#define NEBULA_OPT_INTRA 8
/*   NEBULA_OPT_PIPELINE: 1 (default) an ALL-bucket nebula_step over >= 2 buckets runs its two
 *   halves of buckets on two streams when that helps — TOPK (G = 1, LOOPBACK or P2P exchange):
 *   the latency-bound selection kernels of one half overlap the streaming pass of the other.
 *   2 = also G > 1 with the P2P intra-cluster hop (every codec; one half's intra-cluster
 *   traffic against the other half's codec — measured 1-9 % slower at 2 x 2 / 1 x 4, so not
 *   the default).  Same bits; 0 = one stream.  The context's stream waits for both halves. */
#define NEBULA_OPT_PIPELINE 9
/*   NEBULA_OPT_TOPK_STAGE: top-k streaming pass (p = g + r, classify, stage) for 16-B aligned
 *   calls, 1 (default) a producer warp feeds the tiles through a TMA shared-memory ring, 0 plain
 *   vector loads.  Same results; any time between steps. */
#define NEBULA_OPT_TOPK_STAGE 10
nebula_status nebula_set_option(nebula_ctx* ctx, int32_t option, int64_t value);

/* Exchange transport in use: 0 LOOPBACK, 1 NCCL all-gather, 2 P2P push, 3 P2P pull; -1 for NULL. */
int32_t nebula_exchange_mode(const nebula_ctx* ctx);
/* Intra-cluster hop in use: 0 none (G = 1), 1 NCCL ReduceScatter(avg) / AllGather, 2 P2P
 * fixed-order reduce-scatter / all-gather over NVLink peer memory; -1 for NULL. */
int32_t nebula_intra_mode(const nebula_ctx* ctx);

/* Per-kernel device timers.  When enabled, every kernel / collective the context enqueues is
 * bracketed by a CUDA event pair recorded on the context's stream (the stream the kernel
 * runs on).  nebula_timing_read synchronises, returns per-phase sums since the last read
 * (one entry per phase that ran; phase ids named by nebula_phase_name) and resets them. */
typedef struct {
  uint32_t phase;  /* kernel / collective id */
  uint32_t count;  /* launches timed */
  double ms;       /* summed event-to-event time */
} nebula_phase_time;

nebula_status nebula_timing_enable(nebula_ctx* ctx, int32_t on);
nebula_status nebula_timing_read(nebula_ctx* ctx, nebula_phase_time* out, int32_t cap, int32_t* n_out);
const char* nebula_phase_name(uint32_t phase);

/* ---------------------------------------------------------------------------------------
 * FP16(SVD(rho)) low-rank compressor of ONE fp32 matrix (PAPER.md:105-130
 * Eq. 1-5; readings R29-R31).  The paper applies it to the Scenario-II forward activations
 * (Table 5 "FP16(SVD(r))"): A (m x n) -> U_r, S_r, V_r (top r singular
 * triples, Eq. 2), each encoded as binary16 (Eq. 5); the receiver rebuilds A' = U_r S_r V_r^T
 * (Eq. 3).  Value bytes = 2 (m r + r + r n) = Eq. 4 x 4 m n / 2.
 *
 * Payload (R31): 16-byte preamble {u32 5, u32 m, u32 n, u32 r}, then binary16 sections
 * zero-padded to 16 bytes: U_r [m][r] row-major, S_r [r] (descending), V_r [n][r] row-major.
 * Sign convention (R30): the largest-magnitude entry of every U_r column is positive.
 * Computation: G = B^T B (B = A if m >= n else A^T) in fp64 on the GPU, a dense symmetric
 * eigensolver (cuSOLVER syevd) for the top r eigenpairs, U/V = B W_r / sigma, binary16 pack —
 * all on the handle's stream, no host synchronisation (nebula_svd_check synchronises).
 * Errors: host-validated arguments return immediately; a non-finite entry of A, a binary16
 * overflow of a singular value (>= 65520) or an eigensolver failure are reported by
 * nebula_svd_check (the payload is then unspecified). */
typedef struct nebula_svd nebula_svd; /* opaque, library-owned workspace for one (m, n, r) */

/* m, n >= 1, min(m, n) <= 16384, 1 <= r <= min(m, n).  Allocates the workspace (fp64 Gram
 * min(m,n)^2, fp32 max(m,n) x r, solver buffers) on `device`; stream = cudaStream_t. */
nebula_status nebula_svd_init(nebula_svd** out, int64_t m, int64_t n, int32_t r, int32_t device, void* stream);
/* R29: the kept rank for a ratio rho in (0, 1]: r = clamp(floor(rho * min(m, n) + 1/2), 1,
 * min(m, n)) ("r is the used ratio of the total singular values");
 * 0 for invalid arguments.  nebula_svd_init_density = nebula_svd_init with that r. */
int32_t nebula_svd_rank(int64_t m, int64_t n, double rho);
nebula_status nebula_svd_init_density(nebula_svd** out, int64_t m, int64_t n, double rho, int32_t device, void* stream);
nebula_status nebula_svd_set_stream(nebula_svd* h, void* stream);
/* Payload size in bytes (preamble + padded sections). */
nebula_status nebula_svd_payload_bytes(const nebula_svd* h, uint64_t* bytes);
/* dev_A: fp32 m x n row-major (caller-owned, unmodified); dev_payload: nebula_svd_payload_bytes
 * bytes of device memory (caller-owned), written completely. */
nebula_status nebula_svd_compress(nebula_svd* h, const float* dev_A, void* dev_payload);
/* dev_payload as written by nebula_svd_compress (or by any encoder of the R31 layout with the
 * handle's m, n, r); dev_out: fp32 m x n row-major, A'[i][j] = sum_q fl(U[i][q] S[q]) V[j][q]
 * accumulated in fp32 with fused multiply-adds. */
nebula_status nebula_svd_decompress(nebula_svd* h, const void* dev_payload, float* dev_out);
/* Synchronises the stream; returns (and clears) NEBULA_ERR_NONFINITE / NEBULA_ERR_OVERFLOW or
 * NEBULA_ERR_CUDA for an eigensolver failure, else NEBULA_OK. */
nebula_status nebula_svd_check(nebula_svd* h);
uint64_t nebula_svd_kernel_launches(const nebula_svd* h);
/* Bit 0: eigensolver of the Gram matrix, 0 (default) cuSOLVER syevd (divide and conquer), 1
 * cuSOLVER syevj (Jacobi, tolerance 1e-14, <= 30 sweeps).  Bit 1: Gram kernel, 0 (default) FP64
 * tensor cores (mma.sync m8n8k4 f64), 1 SIMT fp64 FMA.  All give the same factors to binary16. */
nebula_status nebula_svd_set_eigensolver(nebula_svd* h, int32_t which);
nebula_status nebula_svd_destroy(nebula_svd* h);
const char* nebula_svd_last_error(const nebula_svd* h);

/* Frees everything the context owns (synchronises first).  NULL is a no-op.  COLLECTIVE for
 * the NCCL transport when peers are mapped (P2P exchange or intra-cluster hop): every rank must
 * call it, since peers may still read this rank's buffers over NVLink until all ranks arrive
 * (a 4-byte all-reduce quiesces them before the mappings are closed and the memory freed). */
nebula_status nebula_sync_destroy(nebula_ctx* ctx);

/* Last error message of ctx (or of the last failed nebula_sync_init when ctx is NULL). */
const char* nebula_last_error(const nebula_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* NEBULA_SYNC_H_ */
