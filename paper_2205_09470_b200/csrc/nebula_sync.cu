// nebula_sync.cu — the C ABI (include/nebula_sync.h): context, argument validation, memory
// plan, the three stages, NCCL transport over NVLink, LOOPBACK transport.
//
// Stage map:
//   compress           a0 method gate -> [G>1: intra-cluster mean of the G GPUs'
//                      buckets: fixed-order P2P reduce-scatter (kernels_intra.cu),
//                      or ncclReduceScatter(avg) when the peers cannot be mapped]
//                      -> a2..a6 EF + codec kernels (kernels_dense.cu / kernels_ws.cu / kernels_topk.cu)
//   exchange           a7 payloads between clusters (slot c = cluster c): P2P
//                      push / pull over NVLink with arrival flags, or an in-place ncclAllGather;
//                      LOOPBACK: nothing moves
//   decompress_reduce  a8 tree-average of the P slots -> [G>1: P2P all-gather of the shards]
//
// Transports: NCCL (one process per GPU; CUDA IPC maps the peers' buffers), LOOPBACK (all P
// clusters simulated in one context), SELF (one context per (cluster, GPU) in ONE process —
// the contexts reach each other's buffers directly, so every P2P code path runs on one GPU).
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/nebula_sync.h"

// NVTX ranges around the public stage calls (nsys / ncu --nvtx show them as "nebula_*"; header-
// only NVTX 3: without a tool attached each push / pop is one predictable branch)
namespace {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace
#include "kernels.h"

using namespace nb;

namespace {

thread_local std::string g_init_error;

enum BucketState { ST_IDLE = 0, ST_COMPRESSED = 1, ST_EXCHANGED = 2 };

struct BucketInfo {
  uint64_t n = 0;      // caller elements
  uint64_t cn = 0;     // coded elements (n / G)
  uint64_t off = 0;    // element offset in the caller's flat ALL buffers
  uint64_t coff = 0;   // element offset in library coded buffers (multiple of 4)
  uint64_t sn = 0;     // intra-cluster shard elements (n / G)
  uint64_t soff = 0;   // element offset in the shard buffers (multiple of 4)
  uint64_t k = 0;      // TOPK entries
  uint64_t pb[2] = {0, 0};  // payload bytes per slot, per layout (0: codec method, 1: IDENTITY phase)
  uint64_t so[2] = {0, 0};  // byte offset of this bucket's [P][pb] slot block, per layout
  int state = ST_IDLE;
  int method = -1;     // method used by the last compress (after the start-step gate)
  uint64_t seq = 0;    // compresses so far (P2P push: slot parity = seq & 1, arrival flag value)
};

struct Table {         // one launch's work list, resident in d_items / d_ritems
  int first = 0, count = 0;
  uint64_t chunks = 0;
  uint64_t entries = 0, tiles = 0;  // TOPK reduce: sum(k + 1), sum(ceil(n / 2048))
  bool aligned = true; // every g_off (or out_off) is a multiple of 4 elements
};

struct ITable {        // one intra-cluster call's bucket list, resident in d_iitems
  int first = 0, count = 0;
  uint64_t chunks = 0;
  bool aligned = true;  // every off and cn a multiple of 4 elements
};

struct DevGuard {
  int old = -1, dev;
  explicit DevGuard(int d) : dev(d) {
    cudaGetDevice(&old);
    if (old != dev) cudaSetDevice(dev);
  }
  ~DevGuard() {
    if (old >= 0 && old != dev) cudaSetDevice(old);
  }
};

}  // namespace

struct nebula_ctx {
  nebula_topology topo{};
  nebula_codec codec{};
  int P = 1, G = 1, Ploc = 1, me = 0, local_rank = 0, device = 0, num_sms = 148;
  bool loopback = false;
  std::vector<BucketInfo> b;
  uint64_t total_n = 0, total_cn = 0, total_sn = 0, total_slots = 0;
  bool xtopk = false;            // NEXT-3 (R34): G > 1 top-k over the whole cluster bucket
  cudaStream_t stream = nullptr;

  float* d_resid = nullptr;      // [Ploc][total_cn]
  uint8_t* d_slots = nullptr;    // [sum_b P * pb_b]
  uint32_t* d_flags = nullptr;   // sticky device error bits
  uint32_t* h_flags = nullptr;   // pinned host mirror of d_flags, refreshed by an async 4-byte copy
                                 // after every step / reduce: later calls see a device error
                                 // without synchronising (ABI "host-mapped word")
  uint32_t* d_scratch = nullptr; // [Ploc * B] per-item max-abs bits
  // Two slot layouts: [0] for the codec's method, [1] for the IDENTITY phase before
  // start_step (only built when start_step > 0 and the method is lossy).  Slots are sized
  // per method so the exchange moves exactly the payload bytes of the method in use.
  int nlayouts = 1;
  Item* d_items[2] = {nullptr, nullptr};   // all compress tables back to back
  RItem* d_ritems[2] = {nullptr, nullptr}; // all reduce tables back to back
  std::vector<Table> ctab[2];              // [0] = ALL, [1+b] = bucket b
  std::vector<Table> rtab[2];
  float* d_shard_in = nullptr;   // G > 1
  float* d_shard_out = nullptr;

  // ---- intra-cluster hop over NVLink peer memory (G > 1; kernels_intra.cu)
  bool intra_p2p = false;        // every GPU of the cluster mapped (NCCL: IPC, SELF: same process)
  int intra_opt = 0;             // NEBULA_OPT_INTRA: 0 auto (P2P when mapped), 1 NCCL RS/AG
  float* d_recv = nullptr;       // [G][total_sn]: slot j = GPU j's slice of this GPU's shard
  float* d_full = nullptr;       // xtopk: the whole cluster-mean bucket(s) [total_n]
  float* ip_in[8] = {};          // the cluster's GPUs' mean shards (xtopk all-gather)
  unsigned long long* d_arr_rs = nullptr;   // [B][G] arrival words: RS slices, AG shards, scale mail
  unsigned long long* d_arr_ag = nullptr;
  unsigned long long* d_arr_sc = nullptr;
  uint32_t* d_mail = nullptr;    // [B][G] max-abs words of the G shards (exact cluster scale)
  IItem* d_iitems = nullptr;
  std::vector<ITable> itab;      // [0] = ALL, [1+b] = bucket b
  float* ip_recv[8] = {};        // the cluster's GPUs' buffers, indexed by local rank
  float* ip_out[8] = {};
  unsigned long long* ip_arr_rs[8] = {};
  unsigned long long* ip_arr_ag[8] = {};
  unsigned long long* ip_arr_sc[8] = {};
  uint32_t* ip_mail[8] = {};
  std::vector<void*> ipc_opened; // CUDA IPC mappings to close at destroy

  // ---- SELF transport: the group (unique id) this context belongs to
  bool self = false;
  bool peers_resolved = false;
  std::string group;
  float* d_hgrad = nullptr;      // nebula_step_host staging (bucket-major)
  float* d_hout = nullptr;
  cudaStream_t h2d = nullptr, d2h = nullptr;   // nebula_step_host copy streams
  std::vector<cudaEvent_t> ev_in, ev_done;

  TopkBuffers tk{};
  uint2* tk_stage2 = nullptr;          // staging of the second half of a pipelined top-k step
  int topk_pipe = 1;                   // NEBULA_OPT_TOPK_PIPELINE
  cudaStream_t side = nullptr;         // second stream of the pipelined top-k step
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_wide = nullptr;       // pipelined top-k: first half's multi-CTA resolve section done
  void* d_topk_mem = nullptr;
  std::vector<uint64_t> tk_mtiles;   // merge tiles per call type ([0] ALL, [1+b])
  std::vector<uint64_t> tk_host_mt0; // per item
  std::vector<uint64_t> tk_sample_off; // [items + 1]
  std::vector<uint64_t> tk_ccap;       // per item candidate capacity

  ncclComm_t world = nullptr, inter = nullptr, intra = nullptr;
  uint64_t launches = 0;

  // exchange transport: 0 LOOPBACK (nothing moves), 1 NCCL in-place all-gather, 2 P2P push (the
  // compress kernels store every payload into all peers' slots over NVLink; exchange = flags),
  // 3 P2P pull (exchange = flags; the reducer reads every peer's own slot over NVLink)
  int xmode = 0;
  int xopt = 0;                            // NEBULA_OPT_EXCHANGE: 0 auto, 1 NCCL, 2 P2P
  bool p2p_ok = false;
  uint64_t slot_span = 0;                  // bytes of one parity half of d_slots
  uint8_t* peer_slots[NEBULA_MAX_CLUSTERS] = {};            // IPC-mapped d_slots of each cluster
  unsigned long long* peer_arrive[NEBULA_MAX_CLUSTERS] = {}; // IPC-mapped arrival flags
  unsigned long long* d_arrive = nullptr;  // [B][P] last seq received from each sender
  std::string err;

  // INT8 single-pass on-chip kernel (cooperative grid)
  int int8_kernel = 0;          // NEBULA_OPT_INT8_KERNEL
  int fp16_kernel = 0;          // NEBULA_OPT_FP16_KERNEL: 0 TMA ring, 1 plain streaming
  int step_fusion = 0;          // NEBULA_OPT_STEP_FUSION: 0 fuse INT8 steps where eligible, 1 never
  uint64_t sr_seed = 0;         // NEBULA_OPT_SR_SEED (QSGD uniforms, R32)
  int topk_reduce = 1;          // NEBULA_OPT_TOPK_REDUCE: 0 tile-interleaved, 1 per-warp ranges (default)
  int exact_scale = 0;          // NEBULA_OPT_EXACT_SCALE: 1 = cluster-wide INT8/FP8 scale when G > 1 (R28)
  bool ready = false;           // init completed (destroy may then run the collective quiesce)
  bool onchip_ok = false;
  int onchip_grid = 0;
  size_t onchip_smem = 0;
  uint64_t onchip_elems = 0;
  uint32_t* d_bar = nullptr;

  // per-kernel event timers (nebula_timing_*)
  bool timing = false;
  std::vector<cudaEvent_t> evs;
  size_t ev_next = 0;
  struct Rec { int ph, a, b; };
  std::vector<Rec> recs;
  std::vector<std::pair<int, int>> open;  // (phase, start event) stack
};

static void timing_mark(void* p, int ph, int end) {
  nebula_ctx* ctx = static_cast<nebula_ctx*>(p);
  if (ctx->ev_next >= ctx->evs.size()) {
    for (int i = 0; i < 256; ++i) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return;
      ctx->evs.push_back(e);
    }
  }
  const int id = (int)ctx->ev_next++;
  cudaEventRecord(ctx->evs[id], ctx->stream);
  if (!end) {
    ctx->open.push_back({ph, id});
  } else if (!ctx->open.empty()) {
    auto o = ctx->open.back();
    ctx->open.pop_back();
    ctx->recs.push_back({o.first, o.second, id});
  }
}

// ============================================================================ helpers
#define CKC(call)                                                                      \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);                   \
      return NEBULA_ERR_CUDA;                                                          \
    }                                                                                  \
  } while (0)
#define CKN(call)                                                                      \
  do {                                                                                 \
    ncclResult_t r_ = (call);                                                          \
    if (r_ != ncclSuccess) {                                                           \
      ctx->err = std::string(#call) + ": " + ncclGetErrorString(r_);                   \
      return NEBULA_ERR_NCCL;                                                          \
    }                                                                                  \
  } while (0)

static nebula_status fail(nebula_ctx* ctx, nebula_status s, const std::string& msg) {
  if (ctx) ctx->err = msg;
  else g_init_error = msg;
  return s;
}

// Device errors seen by the host mirror (no synchronisation): the sticky bits the kernels raised
// up to the last completed mirror copy.  Returned by every stage call until nebula_check.
static nebula_status pending_device_error(nebula_ctx* ctx) {
  const uint32_t f = ctx->h_flags ? *reinterpret_cast<volatile uint32_t*>(ctx->h_flags) : 0u;
  if (f & kFlagPeerTimeout) return fail(ctx, NEBULA_ERR_NCCL, "P2P exchange: a peer's payload did not arrive (timeout); call nebula_check");
  if (f & kFlagNonfinite) return fail(ctx, NEBULA_ERR_NONFINITE, "non-finite element in g + r (a previous step); call nebula_check");
  if (f & kFlagOverflow) return fail(ctx, NEBULA_ERR_OVERFLOW, "fp16 overflow (a previous step); call nebula_check");
  return NEBULA_OK;
}
static void mirror_flags(nebula_ctx* ctx) {
  cudaMemcpyAsync(ctx->h_flags, ctx->d_flags, 4, cudaMemcpyDeviceToHost, ctx->stream);
}

static uint64_t topk_k_of(uint64_t n, const nebula_codec& c) {
  // R12: k = clamp(floor(rho*n + 0.5), 1, n) in double, or the caller's k (capped at n)
  if (n == 0) return 0;
  if (c.topk_k > 0) return std::min<uint64_t>(c.topk_k, n);
  double k = std::floor(c.topk_density * (double)n + 0.5);
  if (k < 1) k = 1;
  if (k > (double)n) k = (double)n;
  return (uint64_t)k;
}

static uint64_t value_bytes(int vt) { return vt == V_F32 ? 4 : (vt == V_F16 ? 2 : 1); }

static uint64_t payload_bytes_for(int method, uint64_t n, uint64_t k, int vt) {
  switch (method) {
    case M_IDENTITY: return 16 + pad16(4 * n);
    case M_FP16: return 16 + pad16(2 * n);
    case M_INT8:
    case M_QSGD:
    case M_FP8:
    case M_FP8_E5M2: return 16 + pad16(n);
    default: return 16 + pad16(4 * k) + pad16(value_bytes(vt) * k);
  }
}

static uint64_t nchunks_of(uint64_t n) { return std::max<uint64_t>(1, (n + kChunkElems - 1) / kChunkElems); }

// Host-side validation; no CUDA call is made before it passes (tested on CPU).
static nebula_status validate(const nebula_topology* t, const nebula_codec* c, const uint64_t* numel, int nb_) {
  if (!t || !c || !numel) return fail(nullptr, NEBULA_ERR_INVALID_ARG, "null topology/codec/bucket_numel");
  if (nb_ < 1) return fail(nullptr, NEBULA_ERR_INVALID_ARG, "num_buckets must be >= 1");
  if (t->num_clusters < 1 || t->num_clusters > NEBULA_MAX_CLUSTERS)
    return fail(nullptr, NEBULA_ERR_INVALID_ARG, "num_clusters must be in [1, 8]");
  if (t->transport != NEBULA_TRANSPORT_NCCL && t->transport != NEBULA_TRANSPORT_LOOPBACK &&
      t->transport != NEBULA_TRANSPORT_SELF)
    return fail(nullptr, NEBULA_ERR_INVALID_ARG, "unknown transport");
  if (t->gpus_per_cluster < 1 || t->gpus_per_cluster > 64)
    return fail(nullptr, NEBULA_ERR_INVALID_ARG, "gpus_per_cluster must be >= 1");
  if (t->transport == NEBULA_TRANSPORT_LOOPBACK && t->gpus_per_cluster != 1)
    return fail(nullptr, NEBULA_ERR_INVALID_ARG, "LOOPBACK simulates P clusters x 1 GPU (gpus_per_cluster must be 1)");
  if (t->transport == NEBULA_TRANSPORT_SELF && t->gpus_per_cluster > 8)
    return fail(nullptr, NEBULA_ERR_INVALID_ARG, "SELF transport: gpus_per_cluster must be <= 8");
  if (t->transport != NEBULA_TRANSPORT_LOOPBACK) {
    if (!t->nccl_unique_id) return fail(nullptr, NEBULA_ERR_INVALID_ARG, "NCCL / SELF transport needs nccl_unique_id (the group id)");
    if (t->cluster_id < 0 || t->cluster_id >= t->num_clusters)
      return fail(nullptr, NEBULA_ERR_INVALID_ARG, "cluster_id out of range");
    if (t->local_rank < 0 || t->local_rank >= t->gpus_per_cluster)
      return fail(nullptr, NEBULA_ERR_INVALID_ARG, "local_rank out of range");
  }
  if (t->device < 0) return fail(nullptr, NEBULA_ERR_INVALID_ARG, "device must be >= 0");
  if (c->method < NEBULA_IDENTITY || c->method > NEBULA_FP8_E5M2 || c->method == 5)
    return fail(nullptr, NEBULA_ERR_INVALID_ARG, "unknown method");
  if (c->error_feedback != 0 && c->error_feedback != 1)
    return fail(nullptr, NEBULA_ERR_INVALID_ARG, "error_feedback must be 0 or 1");
  if (c->flags & ~NEBULA_CODEC_EXACT_TOPK) return fail(nullptr, NEBULA_ERR_INVALID_ARG, "unknown codec flags");
  if (c->method == NEBULA_TOPK) {
    if (c->topk_values < NEBULA_VAL_F32 || c->topk_values > NEBULA_VAL_I8)
      return fail(nullptr, NEBULA_ERR_INVALID_ARG, "unknown topk value type");
    if (c->topk_k == 0 && !(c->topk_density > 0.0 && c->topk_density <= 1.0))
      return fail(nullptr, NEBULA_ERR_INVALID_ARG, "topk_density must be in (0, 1] when topk_k == 0");
  }
  for (int i = 0; i < nb_; ++i) {
    if (numel[i] >= (1ull << 31)) return fail(nullptr, NEBULA_ERR_INVALID_ARG, "bucket numel must be < 2^31");
    if (numel[i] % (uint64_t)t->gpus_per_cluster)
      return fail(nullptr, NEBULA_ERR_INVALID_ARG, "hierarchical mode needs every bucket numel % gpus_per_cluster == 0");
  }
  return NEBULA_OK;
}

// Method of a compress at `step` (Identity when step < start_step).
static int method_at(const nebula_ctx* ctx, uint64_t step) {
  return step < ctx->codec.start_step ? M_IDENTITY : ctx->codec.method;
}

static int layout_of(const nebula_ctx* ctx, int method) {
  return (ctx->nlayouts == 2 && method == M_IDENTITY) ? 1 : 0;
}

static Launch launch_of(nebula_ctx* ctx) {
  return Launch{ctx->stream, ctx->num_sms, &ctx->launches, ctx->timing ? timing_mark : nullptr, ctx};
}

// Call ids ("t"): 0 = ALL buckets, 1 + b = bucket b alone, B + 1 / B + 2 = the first / second
// half of the buckets (internal: the pipelined top-k step).  ALL and the halves address the
// caller's flat buffers at the buckets' offsets ("flat"); a single-bucket call at offset 0.
static int tab_of(int32_t bucket) { return bucket == NEBULA_ALL_BUCKETS ? 0 : 1 + bucket; }
static bool flat_of(const nebula_ctx* ctx, int t) { return t == 0 || t > (int)ctx->b.size(); }
static void call_range(const nebula_ctx* ctx, int t, int* lo, int* hi) {
  const int B = (int)ctx->b.size(), mid = B / 2;
  if (t == 0) { *lo = 0; *hi = B; }
  else if (t <= B) { *lo = t - 1; *hi = t; }
  else if (t == B + 1) { *lo = 0; *hi = mid; }
  else { *lo = mid; *hi = B; }
}

// Bucket range of a call: ALL -> [0, B), b -> [b, b+1).
static bool range_of(nebula_ctx* ctx, int32_t bucket, int* lo, int* hi) {
  const int B = (int)ctx->b.size();
  if (bucket == NEBULA_ALL_BUCKETS) { *lo = 0; *hi = B; return true; }
  if (bucket < 0 || bucket >= B) return false;
  *lo = bucket; *hi = bucket + 1;
  return true;
}

static uint64_t elems_of(const nebula_ctx* ctx, int lo, int hi) {
  uint64_t s = 0;
  for (int i = lo; i < hi; ++i) s += ctx->b[i].n;
  return s;
}

// ============================================================================ init
static nebula_status build_tables(nebula_ctx* ctx, int lay) {
  const int B = (int)ctx->b.size();
  std::vector<Item> items;
  std::vector<RItem> ritems;
  const uint64_t rtotal = ctx->total_cn;
  std::vector<uint64_t> sbase(B + 1, 0);  // absolute start-offset bases (TOPK reduce)
  for (int bi = 0; bi < B; ++bi) sbase[bi + 1] = sbase[bi] + (uint64_t)ctx->P * ((ctx->b[bi].cn + 2047) / 2048 + 1);
  for (int t = 0; t <= B + 2; ++t) {  // every call id (tab_of / call_range)
    Table ct, rt;
    ct.first = (int)items.size();
    rt.first = (int)ritems.size();
    int blo, bhi;
    call_range(ctx, t, &blo, &bhi);
    const bool flat = flat_of(ctx, t);
    for (int bi = blo; bi < bhi; ++bi) {
      const BucketInfo& bk = ctx->b[bi];
      for (int c = 0; c < ctx->Ploc; ++c) {  // bucket-major, cluster-minor
        Item it{};
        if (ctx->G > 1 && !ctx->xtopk) it.g_off = bk.soff;
        else if (ctx->loopback) it.g_off = flat ? (uint64_t)c * ctx->total_n + bk.off : (uint64_t)c * bk.n;
        else it.g_off = flat ? bk.off : 0;
        it.r_off = (uint64_t)c * rtotal + bk.coff;
        const int cl = ctx->loopback ? c : ctx->me;
        it.slot_off = bk.so[lay] + (uint64_t)cl * bk.pb[lay];
        it.n = bk.cn;
        it.chunk0 = ct.chunks;
        it.sidx = (uint32_t)(c * B + bi);
        ct.chunks += nchunks_of(bk.cn);
        ct.aligned &= (it.g_off % 4) == 0;
        items.push_back(it);
      }
      RItem ri{};
      ri.slot_off = bk.so[lay];
      ri.pb = bk.pb[lay];
      ri.out_off = (ctx->G > 1 && !ctx->xtopk) ? bk.soff : (flat ? bk.off : 0);
      ri.n = bk.cn;
      ri.k = bk.k;
      ri.chunk0 = rt.chunks;
      ri.e0 = rt.entries;
      ri.t0 = rt.tiles;
      ri.sbase = sbase[bi];
      rt.chunks += nchunks_of(bk.cn);
      rt.entries += bk.k + 1;
      rt.tiles += (bk.cn + 2047) / 2048;
      rt.aligned &= (ri.out_off % 4) == 0;
      ritems.push_back(ri);
    }
    ct.count = (int)items.size() - ct.first;
    rt.count = (int)ritems.size() - rt.first;
    ctx->ctab[lay].push_back(ct);
    ctx->rtab[lay].push_back(rt);
  }
  CKC(cudaMalloc(&ctx->d_items[lay], items.size() * sizeof(Item)));
  CKC(cudaMalloc(&ctx->d_ritems[lay], ritems.size() * sizeof(RItem)));
  CKC(cudaMemcpy(ctx->d_items[lay], items.data(), items.size() * sizeof(Item), cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(ctx->d_ritems[lay], ritems.data(), ritems.size() * sizeof(RItem), cudaMemcpyHostToDevice));
  return NEBULA_OK;
}

nebula_status topk_setup(nebula_ctx* ctx);  // below

// ---- SELF transport registry: the contexts of one group (same unique id) in this process.
struct SelfGroup {
  std::map<int, nebula_ctx*> members;   // global rank (cluster * G + local rank) -> context
};
static std::mutex g_self_mu;
static std::map<std::string, SelfGroup> g_self;

static void self_unregister(nebula_ctx* ctx) {
  if (!ctx->self) return;
  std::lock_guard<std::mutex> lk(g_self_mu);
  auto it = g_self.find(ctx->group);
  if (it == g_self.end()) return;
  const int rank = ctx->topo.cluster_id * ctx->G + ctx->topo.local_rank;
  auto m = it->second.members.find(rank);
  if (m != it->second.members.end() && m->second == ctx) it->second.members.erase(m);
  if (it->second.members.empty()) g_self.erase(it);
}

static void release(nebula_ctx* ctx) {
  if (!ctx) return;
  DevGuard g(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  // Collective quiesce (NCCL transport with peer mappings): a peer may still be reading our
  // exported buffers over NVLink (P2P pull reducer, all-gather pull), so nobody unmaps or frees
  // before every rank reached destroy.  nebula_sync_destroy is collective in that case.
  if (ctx->ready && ctx->world && (ctx->p2p_ok || ctx->intra_p2p)) {
    int32_t* d = nullptr;
    if (cudaMalloc(&d, sizeof(int32_t)) == cudaSuccess) {
      cudaMemset(d, 0, sizeof(int32_t));
      ncclAllReduce(d, d, 1, ncclInt32, ncclSum, ctx->world, ctx->stream);
      cudaStreamSynchronize(ctx->stream);
      cudaFree(d);
    }
  }
  self_unregister(ctx);
  for (void* p : ctx->ipc_opened) cudaIpcCloseMemHandle(p);
  cudaFree(ctx->d_resid);
  cudaFree(ctx->d_slots);
  cudaFree(ctx->d_flags);
  if (ctx->h_flags) cudaFreeHost(ctx->h_flags);
  cudaFree(ctx->d_scratch);
  for (int l = 0; l < 2; ++l) {
    cudaFree(ctx->d_items[l]);
    cudaFree(ctx->d_ritems[l]);
  }
  cudaFree(ctx->d_shard_in);
  cudaFree(ctx->d_shard_out);
  cudaFree(ctx->d_recv);
  cudaFree(ctx->d_full);
  cudaFree(ctx->d_arr_rs);
  cudaFree(ctx->d_arr_ag);
  cudaFree(ctx->d_arr_sc);
  cudaFree(ctx->d_mail);
  cudaFree(ctx->d_iitems);
  cudaFree(ctx->d_hgrad);
  cudaFree(ctx->d_hout);
  for (cudaEvent_t e : ctx->ev_in) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->ev_done) cudaEventDestroy(e);
  if (ctx->h2d) cudaStreamDestroy(ctx->h2d);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->ev_wide) cudaEventDestroy(ctx->ev_wide);
  if (ctx->d2h) cudaStreamDestroy(ctx->d2h);
  cudaFree(ctx->d_topk_mem);
  cudaFree(ctx->d_bar);
  for (cudaEvent_t e : ctx->evs) cudaEventDestroy(e);
  cudaFree(ctx->d_arrive);
  if (ctx->intra) ncclCommDestroy(ctx->intra);
  if (ctx->inter && ctx->inter != ctx->world) ncclCommDestroy(ctx->inter);
  if (ctx->world) ncclCommDestroy(ctx->world);
  delete ctx;
}

// ---- NCCL transport: peer mappings (collective over all P*G ranks).  Every rank exports CUDA
// IPC handles of its slot buffer and arrival words (inter-cluster exchange) and of its receive
// buffer, averaged shard, intra arrival words and scale mailbox (intra-cluster hop); the
// handles travel through one ncclAllGather.  Each rank OPENS its peers' handles first, then all
// ranks agree (ncclMin) on whether every rank mapped every peer; if not, everybody closes its
// mappings and keeps the NCCL collectives, so all ranks always use the same transport.
struct P2PInfo {
  cudaIpcMemHandle_t h[9];   // slots, arrive, recv, shard_out, arr_rs, arr_ag, arr_sc, mail, shard_in
  int32_t device, ok, pad0, pad1;
};

static void* ipc_open(nebula_ctx* ctx, const cudaIpcMemHandle_t& h, bool* ok) {
  void* p = nullptr;
  if (!*ok) return nullptr;
  if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    cudaGetLastError();
    *ok = false;
    return nullptr;
  }
  ctx->ipc_opened.push_back(p);
  return p;
}

static nebula_status p2p_setup(nebula_ctx* ctx) {
  const int P = ctx->P, G = ctx->G, N = P * G;
  const int cl = ctx->topo.cluster_id, lr = ctx->local_rank, me = cl * G + lr;
  P2PInfo mine{};
  mine.device = ctx->device;
  void* bufs[9] = {ctx->d_slots, ctx->d_arrive, ctx->d_recv, ctx->d_shard_out, ctx->d_arr_rs, ctx->d_arr_ag,
                   ctx->d_arr_sc, ctx->d_mail, ctx->d_shard_in};
  mine.ok = 1;
  for (int k = 0; k < 9; ++k)
    if (bufs[k] && cudaIpcGetMemHandle(&mine.h[k], bufs[k]) != cudaSuccess) mine.ok = 0;
  cudaGetLastError();
  P2PInfo* d_info = nullptr;
  CKC(cudaMalloc(&d_info, sizeof(P2PInfo) * N));
  CKC(cudaMemcpy(d_info + me, &mine, sizeof(P2PInfo), cudaMemcpyHostToDevice));
  CKN(ncclAllGather(d_info + me, d_info, sizeof(P2PInfo), ncclUint8, ctx->world, ctx->stream));
  CKC(cudaStreamSynchronize(ctx->stream));
  std::vector<P2PInfo> all(N);
  CKC(cudaMemcpy(all.data(), d_info, sizeof(P2PInfo) * N, cudaMemcpyDeviceToHost));
  cudaFree(d_info);
  // inter-cluster peers: same local rank in every other cluster
  bool inter_ok = P > 1;
  const size_t inter_mark = ctx->ipc_opened.size();
  for (int c = 0; c < P && inter_ok; ++c) {
    const P2PInfo& q = all[c * G + lr];
    if (c == cl) {
      ctx->peer_slots[c] = ctx->d_slots;
      ctx->peer_arrive[c] = ctx->d_arrive;
      continue;
    }
    inter_ok = q.ok && mine.ok && q.device != ctx->device;
    ctx->peer_slots[c] = static_cast<uint8_t*>(ipc_open(ctx, q.h[0], &inter_ok));
    ctx->peer_arrive[c] = static_cast<unsigned long long*>(ipc_open(ctx, q.h[1], &inter_ok));
  }
  const size_t intra_mark = ctx->ipc_opened.size();
  bool intra_ok = G > 1 && G <= 8;
  for (int j = 0; j < G && intra_ok; ++j) {
    const P2PInfo& q = all[cl * G + j];
    if (j == lr) {
      ctx->ip_recv[j] = ctx->d_recv;
      ctx->ip_out[j] = ctx->d_shard_out;
      ctx->ip_arr_rs[j] = ctx->d_arr_rs;
      ctx->ip_arr_ag[j] = ctx->d_arr_ag;
      ctx->ip_arr_sc[j] = ctx->d_arr_sc;
      ctx->ip_mail[j] = ctx->d_mail;
      ctx->ip_in[j] = ctx->d_shard_in;
      continue;
    }
    intra_ok = q.ok && mine.ok && q.device != ctx->device;
    ctx->ip_recv[j] = static_cast<float*>(ipc_open(ctx, q.h[2], &intra_ok));
    ctx->ip_out[j] = static_cast<float*>(ipc_open(ctx, q.h[3], &intra_ok));
    ctx->ip_arr_rs[j] = static_cast<unsigned long long*>(ipc_open(ctx, q.h[4], &intra_ok));
    ctx->ip_arr_ag[j] = static_cast<unsigned long long*>(ipc_open(ctx, q.h[5], &intra_ok));
    ctx->ip_arr_sc[j] = static_cast<unsigned long long*>(ipc_open(ctx, q.h[6], &intra_ok));
    ctx->ip_mail[j] = static_cast<uint32_t*>(ipc_open(ctx, q.h[7], &intra_ok));
    ctx->ip_in[j] = static_cast<float*>(ipc_open(ctx, q.h[8], &intra_ok));
  }
  // agree (every rank mapped every peer), else everybody unmaps and keeps NCCL
  int32_t ok2[2] = {inter_ok ? 1 : 0, intra_ok ? 1 : 0};
  int32_t* d_ok = nullptr;
  CKC(cudaMalloc(&d_ok, sizeof(ok2)));
  CKC(cudaMemcpy(d_ok, ok2, sizeof(ok2), cudaMemcpyHostToDevice));
  CKN(ncclAllReduce(d_ok, d_ok, 2, ncclInt32, ncclMin, ctx->world, ctx->stream));
  CKC(cudaStreamSynchronize(ctx->stream));
  CKC(cudaMemcpy(ok2, d_ok, sizeof(ok2), cudaMemcpyDeviceToHost));
  cudaFree(d_ok);
  auto close_from = [&](size_t a, size_t b) {
    for (size_t k = a; k < b; ++k) cudaIpcCloseMemHandle(ctx->ipc_opened[k]);
    for (size_t k = a; k < b; ++k) ctx->ipc_opened[k] = nullptr;
  };
  if (!ok2[1]) close_from(intra_mark, ctx->ipc_opened.size());
  if (!ok2[0]) close_from(inter_mark, intra_mark);
  ctx->ipc_opened.erase(std::remove(ctx->ipc_opened.begin(), ctx->ipc_opened.end(), nullptr), ctx->ipc_opened.end());
  ctx->p2p_ok = ok2[0] != 0;
  ctx->intra_p2p = ok2[1] != 0;
  if (!ctx->p2p_ok)
    for (int c = 0; c < NEBULA_MAX_CLUSTERS; ++c) ctx->peer_slots[c] = nullptr, ctx->peer_arrive[c] = nullptr;
  return NEBULA_OK;
}

// ---- SELF transport: resolve the group's buffers (all P*G contexts must exist by the first
// stage call; their devices must be peer-accessible, the same device always is).
static nebula_status self_resolve(nebula_ctx* ctx) {
  if (!ctx->self || ctx->peers_resolved) return NEBULA_OK;
  std::lock_guard<std::mutex> lk(g_self_mu);
  auto it = g_self.find(ctx->group);
  const int P = ctx->P, G = ctx->G, cl = ctx->topo.cluster_id, lr = ctx->local_rank;
  if (it == g_self.end() || (int)it->second.members.size() != P * G)
    return fail(ctx, NEBULA_ERR_STATE, "SELF transport: not every (cluster, GPU) context of the group exists yet");
  auto& m = it->second.members;
  auto reach = [&](const nebula_ctx* q) -> bool {
    if (q->device == ctx->device) return true;
    int can = 0;
    if (cudaDeviceCanAccessPeer(&can, ctx->device, q->device) != cudaSuccess || !can) return false;
    cudaError_t e = cudaDeviceEnablePeerAccess(q->device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return false;
    cudaGetLastError();
    return true;
  };
  for (int c = 0; c < P; ++c) {
    const nebula_ctx* q = m[c * G + lr];
    if (q->P != P || q->G != G || q->codec.method != ctx->codec.method || q->b.size() != ctx->b.size() || !reach(q))
      return fail(ctx, NEBULA_ERR_INVALID_ARG, "SELF transport: group members disagree (topology / codec / buckets) or cannot reach each other");
    ctx->peer_slots[c] = q->d_slots;
    ctx->peer_arrive[c] = q->d_arrive;
  }
  for (int j = 0; j < G; ++j) {
    const nebula_ctx* q = m[cl * G + j];
    if (q->P != P || q->G != G || q->b.size() != ctx->b.size() || !reach(q))
      return fail(ctx, NEBULA_ERR_INVALID_ARG, "SELF transport: group members disagree or cannot reach each other");
    ctx->ip_recv[j] = q->d_recv;
    ctx->ip_out[j] = q->d_shard_out;
    ctx->ip_arr_rs[j] = q->d_arr_rs;
    ctx->ip_arr_ag[j] = q->d_arr_ag;
    ctx->ip_arr_sc[j] = q->d_arr_sc;
    ctx->ip_mail[j] = q->d_mail;
    ctx->ip_in[j] = q->d_shard_in;
  }
  ctx->p2p_ok = P > 1;
  ctx->intra_p2p = G > 1;
  ctx->peers_resolved = true;
  return NEBULA_OK;
}

// Auto exchange mode: P = 2 -> push (one peer: the compress kernel's NVLink stores hide inside
// it); P > 2 -> pull for the dense codecs (NVLink loads outrun SM-issued stores once every GPU
// feeds P - 1 peers, and the fused step overlaps them with the compress) but push for TOPK (its
// payload is small and the sparse reducer's scattered window loads would each pay the NVLink
// latency: 0.90 ms at P = 4 pulling, r02).
// Measured at N = 2 / 4 (profiles/r02/p2_policy, bench_n4f_*): top-k pushes (its payloads are
// written once, the pull reducer's window loads each paid the NVLink latency); at P = 2 INT8 /
// FP8 push and pull tie (1.145 / 1.13 ms) and push is kept, while FP16 and QSGD gain from the
// fused step over pull (FP16 1.61 -> 1.28 ms, QSGD 1.53 -> 1.40 ms); P > 2 pulls.
static int auto_xmode(const nebula_ctx* ctx) {
  const int m = ctx->codec.method;
  if (m == NEBULA_TOPK) return 2;
  // (a 4 MiB bucket too: FP16 pull 43.7 us vs push 46.0 us, profiles/r02/config1_n2_*.jsonl)
  if (ctx->P == 2 && m != NEBULA_FP16 && m != NEBULA_QSGD) return 2;
  return 3;
}

// Slot buffer of a bucket's exchange `seq` (the P2P modes double-buffer by seq parity).
static uint8_t* slots_at(const nebula_ctx* ctx, uint64_t seq) {
  return ctx->d_slots + (ctx->xmode >= 2 ? (seq & 1) * ctx->slot_span : 0);
}
static uint8_t* slots_of(const nebula_ctx* ctx, const BucketInfo& bk) { return slots_at(ctx, bk.seq); }

// Payload destinations of a compress `seq`: own slot buffer, plus every peer's for the P2P push.
static Dests dests_of(const nebula_ctx* ctx, uint64_t seq) {
  Dests d{};
  d.p[0] = slots_at(ctx, seq);
  d.n = 1;
  if (ctx->xmode == 2) {
    const uint64_t half = (seq & 1) * ctx->slot_span;
    for (int c = 0; c < ctx->P; ++c)
      if (c != ctx->me) d.p[d.n++] = ctx->peer_slots[c] + half;
  }
  return d;
}

// Where the reducer finds cluster c's payload: the local slot buffer, or (P2P pull) cluster
// c's own buffer (IPC-mapped, or the group member's for SELF).
static Dests sources_of(const nebula_ctx* ctx, const BucketInfo& bk) {
  Dests d{};
  d.n = ctx->P;
  for (int c = 0; c < ctx->P; ++c)
    d.p[c] = ctx->xmode == 3 ? ctx->peer_slots[c] + (bk.seq & 1) * ctx->slot_span : slots_of(ctx, bk);
  return d;
}

static Peers inter_peers(const nebula_ctx* ctx) {
  Peers pe{};
  for (int c = 0; c < ctx->P; ++c) pe.arrive[c] = ctx->peer_arrive[c];
  pe.n = ctx->P;
  pe.me = ctx->me;
  return pe;
}
static Peers intra_peers(const nebula_ctx* ctx, unsigned long long* const* arr) {
  Peers pe{};
  for (int j = 0; j < ctx->G; ++j) pe.arrive[j] = arr[j];
  pe.n = ctx->G;
  pe.me = ctx->local_rank;
  return pe;
}
static bool intra_p2p_on(const nebula_ctx* ctx) { return ctx->G > 1 && ctx->intra_p2p && ctx->intra_opt != 1; }

// Intra-cluster tables: per call type one IItem per bucket (ALL: caller offsets bk.off).
static nebula_status build_itables(nebula_ctx* ctx) {
  const int B = (int)ctx->b.size();
  std::vector<IItem> items;
  for (int t = 0; t <= B + 2; ++t) {
    ITable T;
    T.first = (int)items.size();
    int blo, bhi;
    call_range(ctx, t, &blo, &bhi);
    for (int bi = blo; bi < bhi; ++bi) {
      const BucketInfo& bk = ctx->b[bi];
      IItem it{};
      it.off = flat_of(ctx, t) ? bk.off : 0;
      it.coff = bk.soff;
      it.cn = bk.sn;
      it.chunk0 = T.chunks;
      T.chunks += (bk.sn + 4095) / 4096;
      T.aligned &= (it.off % 4 == 0) && (bk.sn % 4 == 0);
      items.push_back(it);
    }
    T.count = (int)items.size() - T.first;
    ctx->itab.push_back(T);
  }
  CKC(cudaMalloc(&ctx->d_iitems, std::max<size_t>(1, items.size()) * sizeof(IItem)));
  CKC(cudaMemcpy(ctx->d_iitems, items.data(), items.size() * sizeof(IItem), cudaMemcpyHostToDevice));
  return NEBULA_OK;
}

extern "C" {

int32_t nebula_abi_version(void) { return NEBULA_ABI_VERSION; }

const char* nebula_status_string(nebula_status s) {
  switch (s) {
    case NEBULA_OK: return "NEBULA_OK";
    case NEBULA_ERR_INVALID_ARG: return "NEBULA_ERR_INVALID_ARG";
    case NEBULA_ERR_STATE: return "NEBULA_ERR_STATE";
    case NEBULA_ERR_OOM: return "NEBULA_ERR_OOM";
    case NEBULA_ERR_CUDA: return "NEBULA_ERR_CUDA";
    case NEBULA_ERR_NCCL: return "NEBULA_ERR_NCCL";
    case NEBULA_ERR_NONFINITE: return "NEBULA_ERR_NONFINITE";
    case NEBULA_ERR_OVERFLOW: return "NEBULA_ERR_OVERFLOW";
    case NEBULA_ERR_UNSUPPORTED: return "NEBULA_ERR_UNSUPPORTED";
  }
  return "NEBULA_ERR_UNKNOWN";
}

nebula_status nebula_get_unique_id(void* out128) {
  if (!out128) return fail(nullptr, NEBULA_ERR_INVALID_ARG, "null output buffer");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, NEBULA_ERR_NCCL, ncclGetErrorString(r));
  static_assert(sizeof(id) == NEBULA_UNIQUE_ID_BYTES, "ncclUniqueId size");
  std::memcpy(out128, &id, sizeof(id));
  return NEBULA_OK;
}

nebula_status nebula_sync_init(nebula_ctx** out, const nebula_topology* topo, const nebula_codec* codec,
                               const uint64_t* bucket_numel, int32_t num_buckets, void* stream) {
  if (!out) return fail(nullptr, NEBULA_ERR_INVALID_ARG, "null out");
  *out = nullptr;
  nebula_status v = validate(topo, codec, bucket_numel, num_buckets);
  if (v != NEBULA_OK) return v;

  nebula_ctx* ctx = new (std::nothrow) nebula_ctx();
  if (!ctx) return fail(nullptr, NEBULA_ERR_OOM, "host allocation failed");
  ctx->topo = *topo;
  ctx->topo.nccl_unique_id = nullptr;
  ctx->codec = *codec;
  ctx->P = topo->num_clusters;
  ctx->G = topo->gpus_per_cluster;
  ctx->loopback = topo->transport == NEBULA_TRANSPORT_LOOPBACK;
  ctx->self = topo->transport == NEBULA_TRANSPORT_SELF;
  if (ctx->self) ctx->group.assign(static_cast<const char*>(topo->nccl_unique_id), NEBULA_UNIQUE_ID_BYTES);
  ctx->Ploc = ctx->loopback ? ctx->P : 1;
  ctx->me = ctx->loopback ? 0 : topo->cluster_id;
  ctx->local_rank = ctx->loopback ? 0 : topo->local_rank;
  ctx->device = topo->device;
  ctx->stream = (cudaStream_t)stream;

  auto bail = [&](nebula_status s) {
    g_init_error = ctx->err;
    release(ctx);
    return s;
  };

  {
    DevGuard dg(ctx->device);
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev <= ctx->device) {
      ctx->err = std::string("no CUDA device ") + std::to_string(ctx->device) + ": " + cudaGetErrorString(e);
      return bail(NEBULA_ERR_CUDA);
    }
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device);
    preload_kernels();   // no lazy kernel load may ever wait behind a spinning flag kernel

    // ---- memory plan
    ctx->b.resize(num_buckets);
    ctx->xtopk = ctx->G > 1 && codec->method == NEBULA_TOPK && (codec->flags & NEBULA_CODEC_EXACT_TOPK);
    uint64_t off = 0, coff = 0, soff = 0, so = 0, so1 = 0;
    for (int i = 0; i < num_buckets; ++i) {
      BucketInfo& bk = ctx->b[i];
      bk.n = bucket_numel[i];
      bk.sn = bk.n / ctx->G;
      bk.cn = ctx->xtopk ? bk.n : bk.sn;   // coded elements: the shard, or (R34) the whole bucket
      bk.off = off;
      bk.coff = coff;
      bk.soff = soff;
      soff += (bk.sn + 3) / 4 * 4;
      bk.k = codec->method == NEBULA_TOPK ? topk_k_of(bk.cn, *codec) : 0;
      bk.pb[0] = payload_bytes_for(codec->method, bk.cn, bk.k, codec->topk_values);
      bk.pb[1] = payload_bytes_for(M_IDENTITY, bk.cn, 0, 0);
      bk.so[0] = so;
      bk.so[1] = so1;
      off += bk.n;
      coff += (bk.cn + 3) / 4 * 4;
      so += (uint64_t)ctx->P * bk.pb[0];
      so1 += (uint64_t)ctx->P * bk.pb[1];
    }
    ctx->nlayouts = (codec->start_step > 0 && codec->method != NEBULA_IDENTITY) ? 2 : 1;
    ctx->total_n = off;
    ctx->total_cn = coff;
    ctx->total_sn = soff;
    ctx->total_slots = ctx->nlayouts == 2 ? std::max(so, so1) : so;

    size_t rbytes = std::max<uint64_t>(16, (uint64_t)ctx->Ploc * ctx->total_cn * sizeof(float));
    if (cudaMalloc(&ctx->d_resid, rbytes) != cudaSuccess) { ctx->err = "residual allocation failed"; return bail(NEBULA_ERR_OOM); }
    ctx->slot_span = pad16(std::max<uint64_t>(16, ctx->total_slots));
    const int halves = (!ctx->loopback && ctx->P > 1) ? 2 : 1;   // double buffer for the P2P push
    if (cudaMalloc(&ctx->d_slots, halves * ctx->slot_span) != cudaSuccess) { ctx->err = "payload allocation failed"; return bail(NEBULA_ERR_OOM); }
    if (cudaMalloc(&ctx->d_flags, 16) != cudaSuccess) { ctx->err = "flag allocation failed"; return bail(NEBULA_ERR_OOM); }
    if (cudaHostAlloc(&ctx->h_flags, 16, cudaHostAllocDefault) != cudaSuccess) { ctx->err = "host flag allocation failed"; return bail(NEBULA_ERR_OOM); }
    std::memset(ctx->h_flags, 0, 16);
    if (cudaMalloc(&ctx->d_scratch, sizeof(uint32_t) * ctx->Ploc * num_buckets) != cudaSuccess) { ctx->err = "scratch allocation failed"; return bail(NEBULA_ERR_OOM); }
    if (cudaMemset(ctx->d_resid, 0, rbytes) != cudaSuccess || cudaMemset(ctx->d_slots, 0, halves * ctx->slot_span) != cudaSuccess ||
        cudaMemset(ctx->d_flags, 0, 16) != cudaSuccess) { ctx->err = "memset failed"; return bail(NEBULA_ERR_CUDA); }
    if (ctx->G > 1) {
      if (cudaMalloc(&ctx->d_shard_in, std::max<uint64_t>(16, ctx->total_sn * 4)) != cudaSuccess ||
          cudaMalloc(&ctx->d_shard_out, std::max<uint64_t>(16, ctx->total_sn * 4)) != cudaSuccess ||
          (ctx->xtopk && cudaMalloc(&ctx->d_full, std::max<uint64_t>(16, ctx->total_n * 4)) != cudaSuccess)) {
        ctx->err = "shard allocation failed";
        return bail(NEBULA_ERR_OOM);
      }
      if (ctx->G <= 8) {   // intra-cluster P2P hop buffers (used when every peer can be mapped)
        const size_t aw = sizeof(unsigned long long) * (size_t)num_buckets * ctx->G;
        if (cudaMalloc(&ctx->d_recv, std::max<uint64_t>(16, (uint64_t)ctx->G * ctx->total_sn * 4)) != cudaSuccess ||
            cudaMalloc(&ctx->d_arr_rs, aw) != cudaSuccess || cudaMalloc(&ctx->d_arr_ag, aw) != cudaSuccess ||
            cudaMalloc(&ctx->d_arr_sc, aw) != cudaSuccess ||
            cudaMalloc(&ctx->d_mail, sizeof(uint32_t) * (size_t)num_buckets * ctx->G) != cudaSuccess) {
          ctx->err = "intra-cluster buffer allocation failed";
          return bail(NEBULA_ERR_OOM);
        }
        if (cudaMemset(ctx->d_arr_rs, 0, aw) != cudaSuccess || cudaMemset(ctx->d_arr_ag, 0, aw) != cudaSuccess ||
            cudaMemset(ctx->d_arr_sc, 0, aw) != cudaSuccess) { ctx->err = "memset failed"; return bail(NEBULA_ERR_CUDA); }
        nebula_status si = build_itables(ctx);
        if (si != NEBULA_OK) return bail(si);
      }
    }
    if (!ctx->loopback && ctx->P > 1) {   // inter-cluster arrival words [B][P] (P2P exchange)
      const size_t aw = sizeof(unsigned long long) * (size_t)num_buckets * ctx->P;
      if (cudaMalloc(&ctx->d_arrive, aw) != cudaSuccess || cudaMemset(ctx->d_arrive, 0, aw) != cudaSuccess) {
        ctx->err = "arrival-word allocation failed";
        return bail(NEBULA_ERR_OOM);
      }
    }
    nebula_status s = NEBULA_OK;
    for (int l = 0; l < ctx->nlayouts && s == NEBULA_OK; ++l) s = build_tables(ctx, l);
    if (s != NEBULA_OK) return bail(s);
    if (codec->method == NEBULA_TOPK) {
      s = topk_setup(ctx);
      if (s != NEBULA_OK) return bail(s);
    }
    if (codec->method == NEBULA_INT8 || codec->method == NEBULA_FP8 || codec->method == NEBULA_QSGD ||
        codec->method == NEBULA_FP8_E5M2 || codec->method == NEBULA_FP16) {
      ctx->onchip_ok = int8_onchip_capacity(ctx->device, &ctx->onchip_elems, &ctx->onchip_grid, &ctx->onchip_smem);
      if (ctx->onchip_ok && cudaMalloc(&ctx->d_bar, sizeof(uint32_t) * (2 * ctx->Ploc * num_buckets + 1)) != cudaSuccess) {
        ctx->err = "barrier allocation failed";
        return bail(NEBULA_ERR_OOM);
      }
      cudaGetLastError();
    }

    // ---- communicators (collective over all P*G ranks)
    if (!ctx->loopback && !ctx->self) {
      ncclUniqueId id;
      std::memcpy(&id, topo->nccl_unique_id, sizeof(id));
      const int nranks = ctx->P * ctx->G, rank = topo->cluster_id * ctx->G + topo->local_rank;
      ncclResult_t r = ncclCommInitRank(&ctx->world, nranks, id, rank);
      if (r != ncclSuccess) { ctx->err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r); return bail(NEBULA_ERR_NCCL); }
      if (ctx->G == 1) {
        ctx->inter = ctx->world;
      } else {
        r = ncclCommSplit(ctx->world, topo->local_rank, topo->cluster_id, &ctx->inter, nullptr);
        if (r == ncclSuccess) r = ncclCommSplit(ctx->world, topo->cluster_id, topo->local_rank, &ctx->intra, nullptr);
        if (r != ncclSuccess) { ctx->err = std::string("ncclCommSplit: ") + ncclGetErrorString(r); return bail(NEBULA_ERR_NCCL); }
      }
    }
    if (!ctx->loopback) {
      ctx->xmode = 1;
      if (ctx->self) {
        // peers are the other contexts of the group in this process (resolved at the first
        // stage call, once every member exists); the exchange is always P2P
        std::lock_guard<std::mutex> lk(g_self_mu);
        SelfGroup& grp = g_self[ctx->group];
        const int rank = topo->cluster_id * ctx->G + topo->local_rank;
        if (grp.members.count(rank)) {
          ctx->err = "SELF transport: this (cluster, local rank) already has a context in the group";
          ctx->self = false;   // not registered: release must not unregister the other context
          return bail(NEBULA_ERR_INVALID_ARG);
        }
        grp.members[rank] = ctx;
        ctx->p2p_ok = ctx->P > 1;
        ctx->intra_p2p = ctx->G > 1;
      } else if (ctx->P > 1 || ctx->G > 1) {
        nebula_status ps = p2p_setup(ctx);
        if (ps != NEBULA_OK) return bail(ps);
      }
      // auto (auto_xmode): push for top-k and at P = 2 (one peer: the NVLink egress hides inside
      // the compress kernel) except FP16 / QSGD; otherwise pull (NVLink loads outrun SM-issued
      // stores once every GPU feeds P - 1 peers)
      if (ctx->p2p_ok && ctx->P > 1) ctx->xmode = auto_xmode(ctx);
    }
    if (cudaDeviceSynchronize() != cudaSuccess) { ctx->err = "device sync after init failed"; return bail(NEBULA_ERR_CUDA); }
  }
  ctx->ready = true;
  *out = ctx;
  return NEBULA_OK;
}

nebula_status nebula_set_stream(nebula_ctx* ctx, void* stream) {
  if (!ctx) return NEBULA_ERR_INVALID_ARG;
  ctx->stream = (cudaStream_t)stream;
  return NEBULA_OK;
}

// NEXT-3 (R28): the max-abs words of this GPU's shards (scratch[b], Ploc == 1 when G > 1;
// |p| bits order like the floats, NaN/Inf bits above every finite one) -> the max over the G
// shards of the cluster, so every shard quantises with the scale of the whole cluster bucket.
// P2P: a mailbox + flag kernel over the cluster's GPUs; else one 4-byte-per-bucket
// ncclAllReduce(max) on the intra-cluster communicator.
static nebula_status cluster_scale(nebula_ctx* ctx, const Launch& L, int lo, int hi, uint64_t seq) {
  if (intra_p2p_on(ctx)) {
    PeerU mails{};
    for (int j = 0; j < ctx->G; ++j) mails.p[j] = ctx->ip_mail[j];
    launch_scale_mail(L, intra_peers(ctx, ctx->ip_arr_sc), mails, ctx->d_scratch, ctx->d_mail, ctx->d_arr_sc, lo, hi,
                      seq, ctx->d_flags);
    CKC(cudaGetLastError());
    return NEBULA_OK;
  }
  Mark mk(L, PH_NCCL_SCALE);
  uint32_t* w = ctx->d_scratch + lo;   // Ploc == 1 when G > 1: word b is bucket b
  CKN(ncclAllReduce(w, w, (size_t)(hi - lo), ncclUint32, ncclMax, ctx->intra, ctx->stream));
  return NEBULA_OK;
}

// G > 1: this GPU's shard of the cluster mean (R20).  P2P: push the peers' slices, flag
// handshake, fixed-order sum / G (bit-identical to the oracle for any input); else NCCL
// ReduceScatter(avg) (order and pre-scaling are NCCL's).
static nebula_status intra_reduce_scatter(nebula_ctx* ctx, const Launch& L, int t, int lo, int hi,
                                          const float* g, uint64_t seq) {
  if (intra_p2p_on(ctx)) {
    const ITable& T = ctx->itab[t];
    const IItem* it = ctx->d_iitems + T.first;
    const bool vec = T.aligned && (uintptr_t)g % 16 == 0;
    {
      PeerF recv{};
      for (int j = 0; j < ctx->G; ++j) recv.p[j] = ctx->ip_recv[j];
      recv.n = ctx->G;
      recv.me = ctx->local_rank;
      launch_rs_push(L, vec, it, T.count, T.chunks, g, recv, ctx->total_sn);
    }
    launch_exchange_flags(L, intra_peers(ctx, ctx->ip_arr_rs), ctx->d_arr_rs, lo, hi, seq, ctx->d_flags, PH_P2P_FLAGS_RS);
    launch_rs_reduce(L, vec, it, T.count, T.chunks, g, ctx->d_recv, ctx->total_sn, ctx->G, ctx->local_rank,
                     ctx->d_shard_in);
    CKC(cudaGetLastError());
    return NEBULA_OK;
  }
  if (!ctx->intra) return fail(ctx, NEBULA_ERR_UNSUPPORTED, "no intra-cluster transport (peers not mapped, no NCCL)");
  Mark mk(L, PH_NCCL_RS);
  CKN(ncclGroupStart());
  for (int i = lo; i < hi; ++i) {
    const BucketInfo& bk = ctx->b[i];
    if (!bk.sn) continue;
    const float* src = g + (flat_of(ctx, t) ? bk.off : 0);
    CKN(ncclReduceScatter(src, ctx->d_shard_in + bk.soff, bk.sn, ncclFloat32, ncclAvg, ctx->intra, ctx->stream));
  }
  CKN(ncclGroupEnd());
  return NEBULA_OK;
}

// G > 1: every GPU of the cluster gathers the P2P-averaged shards into dev_out.  P2P: flag
// handshake, then NVLink loads of the peers' shards; else NCCL AllGather.
static nebula_status intra_all_gather(nebula_ctx* ctx, const Launch& L, int t, int lo, int hi, float* dev_out,
                                      uint64_t seq, bool from_in = false) {
  // from_in (xtopk): gather the G mean shards (d_shard_in) instead of the averaged ones
  float* const* srcs = from_in ? ctx->ip_in : ctx->ip_out;
  float* own = from_in ? ctx->d_shard_in : ctx->d_shard_out;
  if (intra_p2p_on(ctx)) {
    const ITable& T = ctx->itab[t];
    launch_exchange_flags(L, intra_peers(ctx, ctx->ip_arr_ag), ctx->d_arr_ag, lo, hi, seq, ctx->d_flags, PH_P2P_FLAGS_AG);
    PeerF outs{};
    for (int j = 0; j < ctx->G; ++j) outs.p[j] = srcs[j];
    outs.n = ctx->G;
    outs.me = ctx->local_rank;
    launch_ag_pull(L, T.aligned && (uintptr_t)dev_out % 16 == 0, ctx->d_iitems + T.first, T.count, T.chunks, outs, dev_out);
    CKC(cudaGetLastError());
    return NEBULA_OK;
  }
  if (!ctx->intra) return fail(ctx, NEBULA_ERR_UNSUPPORTED, "no intra-cluster transport (peers not mapped, no NCCL)");
  Mark mk(L, PH_NCCL_AG);
  CKN(ncclGroupStart());
  for (int i = lo; i < hi; ++i) {
    const BucketInfo& bk = ctx->b[i];
    if (!bk.sn) continue;
    float* dst = dev_out + (flat_of(ctx, t) ? bk.off : 0);
    CKN(ncclAllGather(own + bk.soff, dst, bk.sn, ncclFloat32, ctx->intra, ctx->stream));
  }
  CKN(ncclGroupEnd());
  return NEBULA_OK;
}

static nebula_status zero_scratch(nebula_ctx* ctx, const Launch& L, int lo, int hi) {
  Mark mk(L, PH_MEMSET);
  for (int c = 0; c < ctx->Ploc; ++c)
    CKC(cudaMemsetAsync(ctx->d_scratch + (size_t)c * ctx->b.size() + lo, 0, sizeof(uint32_t) * (size_t)(hi - lo),
                        ctx->stream));
  return NEBULA_OK;
}

// Call preconditions shared by compress and the fused step: every bucket of the call is idle
// (a second compress would apply the residual twice) and, for ALL calls, at the same
// step count, so one sequence number names the exchange of every bucket of the call.
static nebula_status stage_start(nebula_ctx* ctx, int lo, int hi) {
  for (int i = lo; i < hi; ++i)
    if (ctx->b[i].state != ST_IDLE)
      return fail(ctx, NEBULA_ERR_STATE, "compress: bucket " + std::to_string(i) +
                                             " is mid-step (compress -> exchange -> decompress_reduce)");
  for (int i = lo + 1; i < hi; ++i)
    if (ctx->b[i].seq != ctx->b[lo].seq)
      return fail(ctx, NEBULA_ERR_STATE, "ALL-bucket call over buckets at different step counts");
  return self_resolve(ctx);
}

// ============================================================================ stages
static nebula_status compress_t(nebula_ctx* ctx, int t, const float* dev_grad, uint64_t step) {
  int lo, hi;
  call_range(ctx, t, &lo, &hi);
  if (!dev_grad && elems_of(ctx, lo, hi)) return fail(ctx, NEBULA_ERR_INVALID_ARG, "null dev_grad");
  nebula_status st0 = stage_start(ctx, lo, hi);
  if (st0 != NEBULA_OK) return st0;
  st0 = pending_device_error(ctx);
  if (st0 != NEBULA_OK) return st0;
  DevGuard dg(ctx->device);
  const int method = method_at(ctx, step);
  const bool ef = ctx->codec.error_feedback != 0;
  const int lay = layout_of(ctx, method);
  const Table& T = ctx->ctab[lay][t];
  const Launch L = launch_of(ctx);
  const uint64_t seq = ctx->b[lo].seq + 1;   // this exchange; committed once everything is enqueued
  const Dests dst = dests_of(ctx, seq);

  const float* gbase = dev_grad;
  if (ctx->G > 1) {  // intra-cluster mean of the G GPUs' buckets -> this GPU's shard (R20)
    nebula_status s = intra_reduce_scatter(ctx, L, t, lo, hi, dev_grad, seq);
    if (s != NEBULA_OK) return s;
    gbase = ctx->d_shard_in;
    if (ctx->xtopk) {   // R34: every GPU of the cluster codes the whole cluster-mean bucket
      s = intra_all_gather(ctx, L, t, lo, hi, ctx->d_full, seq, true);
      if (s != NEBULA_OK) return s;
      gbase = ctx->d_full;
    }
  }
  const bool vec = T.aligned && ((uintptr_t)gbase % 16 == 0);
  const Item* items = ctx->d_items[lay] + T.first;
  const bool xscale = ctx->exact_scale && ctx->G > 1;

  switch (method) {
    case M_IDENTITY:
      launch_identity(L, vec, items, T.count, T.chunks, gbase, dst, ctx->d_flags);
      break;
    case M_FP16:
      if (vec && ctx->fp16_kernel == 0)
        launch_fp16_tma(L, ef, items, T.count, T.chunks, gbase, ctx->d_resid, dst, ctx->d_flags);
      else
        launch_fp16(L, ef, vec, items, T.count, T.chunks, gbase, ctx->d_resid, dst, ctx->d_flags);
      break;
    case M_INT8:
    case M_FP8:
    case M_FP8_E5M2:
    case M_QSGD: {
      // one per-bucket scale: max-abs words zeroed, then either the single-pass warp-specialised
      // kernel (16-B aligned, buckets averaging >= 1M elements, no cluster-wide scale) or the
      // max-abs pass, [the cluster-wide max (R28)], and the quantise pass
      { nebula_status zs = zero_scratch(ctx, L, lo, hi); if (zs != NEBULA_OK) return zs; }
      const int kind = method == M_FP8 ? 1 : (method == M_QSGD ? 2 : (method == M_FP8_E5M2 ? 3 : 0));
      const SrArgs sr{ctx->sr_seed, step, (uint32_t)ctx->me, (uint32_t)ctx->local_rank, (uint32_t)ctx->b.size()};
      // (SELF: auto never picks the cooperative kernel — group members' grids share one GPU)
      const bool single = ctx->onchip_ok && vec && !xscale &&
                          (ctx->int8_kernel == 2 ||
                           (ctx->int8_kernel == 0 && !ctx->self &&
                            elems_of(ctx, lo, hi) / ctx->G >= (uint64_t)(hi - lo) * (1ull << 20)));
      if (single) {
        // done words of the call's own items: the two halves of a pipelined step run concurrently
        launch_ws_compress(L, ef, kind, items, T.count, gbase, ctx->d_resid, dst, ctx->d_scratch, ctx->d_flags,
                           ctx->d_bar + (size_t)lo * ctx->Ploc, sr);
        break;
      }
      launch_absmax(L, ef, vec, items, T.count, T.chunks, gbase, ctx->d_resid, ctx->d_scratch);
      if (xscale) { nebula_status xs = cluster_scale(ctx, L, lo, hi, seq); if (xs != NEBULA_OK) return xs; }
      if (kind == 1 || kind == 3)
        launch_fp8_quant(L, ef, vec, items, T.count, T.chunks, gbase, ctx->d_resid, dst, ctx->d_scratch, ctx->d_flags,
                         kind == 3 ? 2 : 1);
      else if (kind == 2) launch_qsgd_quant(L, ef, vec, items, T.count, T.chunks, gbase, ctx->d_resid, dst, ctx->d_scratch, ctx->d_flags, sr);
      else launch_int8_quant(L, ef, vec, items, T.count, T.chunks, gbase, ctx->d_resid, dst, ctx->d_scratch, ctx->d_flags);
      break;
    }
    case M_TOPK: {
      const int item0 = lo * ctx->Ploc;
      TopkBuffers tkb = ctx->tk;
      if (t > (int)ctx->b.size()) {
        // pipelined halves: the second half's multi-CTA resolve section waits for the first
        // half's.  Run concurrently, the two sections faulted (illegal address) or diverged at
        // 2-10 % density with more buckets on that path (profiles/r02/topk/README.md); ordered
        // they pass — the conflict is not understood, so they never overlap.
        if (!ctx->ev_wide) CKC(cudaEventCreateWithFlags(&ctx->ev_wide, cudaEventDisableTiming));
        if (t == (int)ctx->b.size() + 1) tkb.wide_rec = ctx->ev_wide;
        else tkb.wide_wait = ctx->ev_wide;
      }
      if (t == (int)ctx->b.size() + 2) {   // second half of a pipelined step: own counters / staging
        tkb.ctrs = ctx->tk.ctrs + 8;
        tkb.stage = ctx->tk_stage2;
      }
      launch_topk(L, ef, vec, tkb, item0, T.count, T.chunks, items, gbase, ctx->d_resid, dst,
                  ctx->d_flags, ctx->codec.topk_values, ctx->tk_mtiles[t]);
      break;
    }
  }
  CKC(cudaGetLastError());
  for (int i = lo; i < hi; ++i) {
    ctx->b[i].seq = seq;
    ctx->b[i].state = ST_COMPRESSED;
    ctx->b[i].method = method;
  }
  return NEBULA_OK;
}

nebula_status nebula_compress(nebula_ctx* ctx, int32_t bucket, const float* dev_grad, uint64_t step) {
  NvtxRange nvtx_range("nebula_compress");
  if (!ctx) return NEBULA_ERR_INVALID_ARG;
  int lo, hi;
  if (!range_of(ctx, bucket, &lo, &hi)) return fail(ctx, NEBULA_ERR_INVALID_ARG, "bucket index out of range");
  return compress_t(ctx, tab_of(bucket), dev_grad, step);
}

static nebula_status exchange_t(nebula_ctx* ctx, int t) {
  int lo, hi;
  call_range(ctx, t, &lo, &hi);
  for (int i = lo; i < hi; ++i)
    if (ctx->b[i].state != ST_COMPRESSED) return fail(ctx, NEBULA_ERR_STATE, "exchange before compress");
  DevGuard dg(ctx->device);
  if (ctx->xmode >= 2) {   // push: payloads already in our slots; pull: peers' own slots ready
    const Launch L = launch_of(ctx);
    launch_exchange_flags(L, inter_peers(ctx), ctx->d_arrive, lo, hi, ctx->b[lo].seq, ctx->d_flags);
    CKC(cudaGetLastError());
  } else if (!ctx->loopback && ctx->P > 1) {
    const Launch L = launch_of(ctx);
    Mark mk(L, PH_NCCL_EXCHANGE);
    CKN(ncclGroupStart());
    for (int i = lo; i < hi; ++i) {
      const BucketInfo& bk = ctx->b[i];
      // in place: rank c's contribution already sits in slot c (ncclAllGather in-place rule)
      const int lay = layout_of(ctx, bk.method);
      uint8_t* base = slots_of(ctx, bk) + bk.so[lay];
      CKN(ncclAllGather(base + (uint64_t)ctx->me * bk.pb[lay], base, bk.pb[lay], ncclUint8, ctx->inter, ctx->stream));
    }
    CKN(ncclGroupEnd());
  }
  for (int i = lo; i < hi; ++i) ctx->b[i].state = ST_EXCHANGED;
  return NEBULA_OK;
}

nebula_status nebula_exchange(nebula_ctx* ctx, int32_t bucket) {
  NvtxRange nvtx_range("nebula_exchange");
  if (!ctx) return NEBULA_ERR_INVALID_ARG;
  int lo, hi;
  if (!range_of(ctx, bucket, &lo, &hi)) return fail(ctx, NEBULA_ERR_INVALID_ARG, "bucket index out of range");
  return exchange_t(ctx, tab_of(bucket));
}

static nebula_status reduce_t(nebula_ctx* ctx, int t, float* dev_out) {
  int lo, hi;
  call_range(ctx, t, &lo, &hi);
  if (!dev_out && elems_of(ctx, lo, hi)) return fail(ctx, NEBULA_ERR_INVALID_ARG, "null dev_out");
  for (int i = lo; i < hi; ++i)
    if (ctx->b[i].state != ST_EXCHANGED) return fail(ctx, NEBULA_ERR_STATE, "decompress_reduce before exchange");
  const int method = ctx->b[lo].method;
  for (int i = lo; i < hi; ++i)
    if (ctx->b[i].method != method) return fail(ctx, NEBULA_ERR_STATE, "buckets compressed with different methods");
  DevGuard dg(ctx->device);
  const int lay = layout_of(ctx, method);
  const Table& T = ctx->rtab[lay][t];
  const bool sharded = ctx->G > 1 && !ctx->xtopk;   // reduce this GPU's shard, then all-gather
  float* obase = sharded ? ctx->d_shard_out : dev_out;
  const bool vec = T.aligned && ((uintptr_t)obase % 16 == 0);
  const Launch L = launch_of(ctx);
  const RItem* items = ctx->d_ritems[lay] + T.first;
  if (method == M_TOPK)
  {
    // output range of this call: buckets [lo, hi) are contiguous in the out buffer
    float* zb;
    uint64_t zc;
    if (sharded) {
      zb = obase + ctx->b[lo].soff;
      zc = (hi == (int)ctx->b.size() ? ctx->total_sn : ctx->b[hi].soff) - ctx->b[lo].soff;
    } else {
      zb = obase;
      zc = elems_of(ctx, lo, hi);
    }
    uint64_t sc = 0;
    for (int i = lo; i < hi; ++i) sc += (uint64_t)ctx->P * ((ctx->b[i].cn + 2047) / 2048 + 1);
    launch_reduce_topk(L, ctx->codec.topk_values, ctx->P, vec, items, T.count, T.entries, T.tiles, sources_of(ctx, ctx->b[lo]),
                       ctx->tk.start, obase, zb, zc, sc, ctx->topk_reduce);
  }
  else
    launch_reduce_dense(L, method, ctx->P, vec, items, T.count, T.chunks, sources_of(ctx, ctx->b[lo]), obase);
  CKC(cudaGetLastError());
  if (sharded) {
    nebula_status s = intra_all_gather(ctx, L, t, lo, hi, dev_out, ctx->b[lo].seq);
    if (s != NEBULA_OK) return s;
  }
  mirror_flags(ctx);
  for (int i = lo; i < hi; ++i) ctx->b[i].state = ST_IDLE;
  return NEBULA_OK;
}

nebula_status nebula_decompress_reduce(nebula_ctx* ctx, int32_t bucket, float* dev_out) {
  NvtxRange nvtx_range("nebula_decompress_reduce");
  if (!ctx) return NEBULA_ERR_INVALID_ARG;
  int lo, hi;
  if (!range_of(ctx, bucket, &lo, &hi)) return fail(ctx, NEBULA_ERR_INVALID_ARG, "bucket index out of range");
  return reduce_t(ctx, tab_of(bucket), dev_out);
}

// Decode ONE cluster's payload (no averaging) — the pipeline-hop use of the codecs (SURVEY.md
// NEXT-2; PAPER.md:418 FP16 forward activations / INT8 backward gradients across the
// Scenario-II boundary).  Reuses the reducer kernels with P = 1 on that slot.
nebula_status nebula_decompress(nebula_ctx* ctx, int32_t bucket, int32_t slot, float* dev_out) {
  if (!ctx) return NEBULA_ERR_INVALID_ARG;
  int lo, hi;
  if (!range_of(ctx, bucket, &lo, &hi)) return fail(ctx, NEBULA_ERR_INVALID_ARG, "bucket index out of range");
  if (slot < 0 || slot >= ctx->P) return fail(ctx, NEBULA_ERR_INVALID_ARG, "slot out of range");
  if (!dev_out && elems_of(ctx, lo, hi)) return fail(ctx, NEBULA_ERR_INVALID_ARG, "null dev_out");
  for (int i = lo; i < hi; ++i) {
    const int st = ctx->b[i].state;
    const bool own = ctx->loopback || slot == ctx->me;
    if (!(st == ST_EXCHANGED || (st == ST_COMPRESSED && own)))
      return fail(ctx, NEBULA_ERR_STATE, "decompress needs the slot's payload (compress / exchange first)");
  }
  const bool sharded = ctx->G > 1 && !ctx->xtopk;
  if (sharded && !ctx->intra)   // the shards are gathered with NCCL (no P2P sequence for this call)
    return fail(ctx, NEBULA_ERR_UNSUPPORTED, "single-slot decompress with G > 1 needs the NCCL transport");
  DevGuard dg(ctx->device);
  const Launch L = launch_of(ctx);
  for (int i = lo; i < hi; ++i) {
    const BucketInfo& bk = ctx->b[i];
    const int method = bk.method, lay = layout_of(ctx, method);
    const Table& T = ctx->rtab[lay][1 + i];
    const RItem* items = ctx->d_ritems[lay] + T.first;
    float* out_b = dev_out + (bucket == NEBULA_ALL_BUCKETS ? bk.off : 0);
    float* obase = sharded ? ctx->d_shard_out : out_b;
    const bool vec = T.aligned && ((uintptr_t)obase % 16 == 0);
    Dests src{};
    src.n = 1;
    src.p[0] = sources_of(ctx, bk).p[slot] + (uint64_t)slot * bk.pb[lay];   // slot c read as "cluster 0"
    if (method == M_TOPK) {
      float* zb = sharded ? obase + bk.soff : obase;
      launch_reduce_topk(L, ctx->codec.topk_values, 1, vec, items, T.count, T.entries, T.tiles, src, ctx->tk.start,
                         obase, zb, bk.cn, (bk.cn + 2047) / 2048 + 1, ctx->topk_reduce);
    } else {
      launch_reduce_dense(L, method, 1, vec, items, T.count, T.chunks, src, obase);
    }
    CKC(cudaGetLastError());
    if (sharded && bk.sn) {
      Mark mk(L, PH_NCCL_AG);
      CKN(ncclAllGather(ctx->d_shard_out + bk.soff, out_b, bk.sn, ncclFloat32, ctx->intra, ctx->stream));
    }
  }
  return NEBULA_OK;
}

// The fused INT8 step (one cooperative kernel for compress + exchange + reduce), when the
// call is one the warp-specialised kernel serves and the exchange is LOOPBACK or P2P.
static bool step_fusable(const nebula_ctx* ctx, int lo, int hi, int32_t bucket, const float* g, const float* out,
                         uint64_t step) {
  const int m = method_at(ctx, step);
  if (ctx->step_fusion == 1 || (m != M_INT8 && m != M_FP8 && m != M_QSGD && m != M_FP8_E5M2 && m != M_FP16) ||
      ctx->G != 1 || !ctx->onchip_ok)
    return false;
  if (m == M_FP16 && ctx->fp16_kernel != 0) return false;   // the plain FP16 kernel option stays staged
  // SELF: the peers' cooperative kernels share this GPU — two grid-wide kernels waiting on each
  // other's flags could never be co-resident, so SELF always runs the staged stages
  if (ctx->self) return false;
  // LOOPBACK, or P2P pull (the reduce warps load the peers' payloads); with P2P push the
  // compress kernel's NVLink stores are cheaper outside the fused kernel (fewer quantise warps)
  if (!(ctx->loopback || ctx->P == 1 || ctx->xmode == 3)) return false;
  if (!(ctx->int8_kernel == 0 || ctx->int8_kernel == 2)) return false;
  if (ctx->int8_kernel == 0 && elems_of(ctx, lo, hi) < (uint64_t)(hi - lo) * (1ull << 20)) return false;
  const int lay = layout_of(ctx, M_INT8), t = bucket == NEBULA_ALL_BUCKETS ? 0 : 1 + bucket;
  const Table& T = ctx->ctab[lay][t];
  const Table& R = ctx->rtab[lay][t];
  if (!T.aligned || !R.aligned || (uintptr_t)g % 16 || (uintptr_t)out % 16) return false;
  return true;
}

static nebula_status int8_step_fused(nebula_ctx* ctx, int lo, int hi, int32_t bucket, const float* dev_grad,
                                     float* dev_out, int method, uint64_t step) {
  const bool ef = ctx->codec.error_feedback != 0;
  const int lay = layout_of(ctx, M_INT8), t = bucket == NEBULA_ALL_BUCKETS ? 0 : 1 + bucket;
  const Table& T = ctx->ctab[lay][t];
  const Table& R = ctx->rtab[lay][t];
  const Launch L = launch_of(ctx);
  nebula_status st0 = stage_start(ctx, lo, hi);
  if (st0 != NEBULA_OK) return st0;
  st0 = pending_device_error(ctx);
  if (st0 != NEBULA_OK) return st0;
  const uint64_t seq = ctx->b[lo].seq + 1;
  { nebula_status zs = zero_scratch(ctx, L, lo, hi); if (zs != NEBULA_OK) return zs; }
  Peers pe{};
  if (!ctx->loopback && ctx->P > 1) pe = inter_peers(ctx);
  BucketInfo probe = ctx->b[lo];
  probe.seq = seq;
  if (method == M_FP16) {
    launch_fp16_step(L, ef, ctx->d_items[lay] + T.first, T.count, dev_grad, ctx->d_resid, dests_of(ctx, seq),
                     ctx->d_flags, ctx->d_bar, ctx->d_ritems[lay] + R.first, lo, ctx->Ploc, sources_of(ctx, probe),
                     dev_out, pe, ctx->d_arrive, seq, ctx->xmode == 3 ? 1 : 0);
  } else
  launch_int8_step(L, ef, ctx->d_items[lay] + T.first, T.count, dev_grad, ctx->d_resid, dests_of(ctx, seq),
                   ctx->d_scratch, ctx->d_flags, ctx->d_bar, ctx->d_ritems[lay] + R.first, lo, ctx->Ploc,
                   sources_of(ctx, probe), dev_out, pe, ctx->d_arrive, seq,
                   ctx->step_fusion >= 2 ? ctx->step_fusion - 2 : (ctx->xmode == 3 ? 4 : 0),
                   method == M_FP8 ? 1 : (method == M_QSGD ? 2 : (method == M_FP8_E5M2 ? 3 : 0)),
                   SrArgs{ctx->sr_seed, step, (uint32_t)ctx->me, (uint32_t)ctx->local_rank, (uint32_t)ctx->b.size()});
  CKC(cudaGetLastError());
  mirror_flags(ctx);
  for (int i = lo; i < hi; ++i) {
    ctx->b[i].seq = seq;
    ctx->b[i].state = ST_IDLE;
    ctx->b[i].method = method;
  }
  return NEBULA_OK;
}

// Pipelined step: the buckets split into two halves, each a full compress -> exchange ->
// reduce on its own stream.  TOPK: the latency-bound selection kernels of one half (bracket,
// scan, resolve, merge: one CTA per bucket or small grids) overlap the HBM-bound stage pass of
// the other.  G > 1 (every codec): one half's NVLink-bound intra-cluster reduce-scatter /
// all-gather overlaps the other half's HBM-bound codec.  Same kernels, same per-bucket state,
// same bits.  P2P / LOOPBACK transports only (two NCCL collectives on one communicator from two
// streams could interleave differently on different ranks); SELF runs the staged calls as its
// rules say.
static bool step_pipelinable(const nebula_ctx* ctx, int32_t bucket, uint64_t step) {
  if (!ctx->topk_pipe || bucket != NEBULA_ALL_BUCKETS || ctx->b.size() < 2 || ctx->self) return false;
  if (ctx->P > 1 && ctx->xmode == 1) return false;
  const int m = method_at(ctx, step);
  if (m == M_TOPK && ctx->topk_reduce == 0) return false;   // variant 0's start offsets are shared
  // G > 1 only when asked for (value 2): measured at 2 x 2 and 1 x 4 it was 1-9 % slower than
  // one stream (profiles/r02/g_gt1_pipeline) — the halves' intra-cluster kernels contend
  if (ctx->G > 1) return ctx->topk_pipe == 2 && intra_p2p_on(ctx);
  return m == M_TOPK;
}

static nebula_status step_pipelined(nebula_ctx* ctx, const float* dev_grad, float* dev_out, uint64_t step) {
  DevGuard dg(ctx->device);
  if (!ctx->side) {
    CKC(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
    CKC(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
  }
  const int B = (int)ctx->b.size();
  for (int i = 1; i < B; ++i)   // validate before anything is enqueued (as the ALL call would)
    if (ctx->b[i].state != ST_IDLE || ctx->b[i].seq != ctx->b[0].seq || ctx->b[0].state != ST_IDLE)
      return fail(ctx, NEBULA_ERR_STATE, "ALL-bucket step over buckets that are mid-step or at different step counts");
  CKC(cudaEventRecord(ctx->ev_fork, ctx->stream));
  CKC(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
  nebula_status s = compress_t(ctx, B + 1, dev_grad, step);
  if (s == NEBULA_OK) s = exchange_t(ctx, B + 1);
  if (s == NEBULA_OK) s = reduce_t(ctx, B + 1, dev_out);
  if (s != NEBULA_OK) return s;
  cudaStream_t main = ctx->stream;
  ctx->stream = ctx->side;
  s = compress_t(ctx, B + 2, dev_grad, step);
  if (s == NEBULA_OK) s = exchange_t(ctx, B + 2);
  if (s == NEBULA_OK) s = reduce_t(ctx, B + 2, dev_out);
  ctx->stream = main;
  CKC(cudaEventRecord(ctx->ev_join, ctx->side));
  CKC(cudaStreamWaitEvent(main, ctx->ev_join, 0));
  return s;
}

nebula_status nebula_step(nebula_ctx* ctx, int32_t bucket, const float* dev_grad, float* dev_out, uint64_t step) {
  NvtxRange nvtx_range("nebula_step");
  if (ctx && step_pipelinable(ctx, bucket, step) && dev_grad && dev_out) return step_pipelined(ctx, dev_grad, dev_out, step);
  if (ctx) {
    int lo, hi;
    if (range_of(ctx, bucket, &lo, &hi) && hi > lo && dev_grad && dev_out &&
        step_fusable(ctx, lo, hi, bucket, dev_grad, dev_out, step)) {
      DevGuard dg(ctx->device);
      return int8_step_fused(ctx, lo, hi, bucket, dev_grad, dev_out, method_at(ctx, step), step);
    }
  }
  nebula_status s = nebula_compress(ctx, bucket, dev_grad, step);
  if (s != NEBULA_OK) return s;
  s = nebula_exchange(ctx, bucket);
  if (s != NEBULA_OK) return s;
  return nebula_decompress_reduce(ctx, bucket, dev_out);
}

// Host-buffer step, pipelined per bucket over three streams so both PCIe directions and the
// GPU work overlap:  h2d stream: copy bucket b in -> event;  ctx stream: wait, step(b) ->
// event;  d2h stream: wait, copy bucket b's average out.  Device staging is bucket-major
// ([P][n_b] per bucket for LOOPBACK, as a per-bucket call expects).
nebula_status nebula_step_host(nebula_ctx* ctx, const float* host_grad, float* host_out, uint64_t step) {
  NvtxRange nvtx_range("nebula_step_host");
  if (!ctx) return NEBULA_ERR_INVALID_ARG;
  if ((!host_grad || !host_out) && ctx->total_n) return fail(ctx, NEBULA_ERR_INVALID_ARG, "null host buffer");
  DevGuard dg(ctx->device);
  const int Pl = ctx->loopback ? ctx->P : 1;
  const uint64_t gelems = (uint64_t)Pl * ctx->total_n;
  const int B = (int)ctx->b.size();
  if (!ctx->d_hgrad) {
    CKC(cudaMalloc(&ctx->d_hgrad, std::max<uint64_t>(16, gelems * 4)));
    CKC(cudaMalloc(&ctx->d_hout, std::max<uint64_t>(16, ctx->total_n * 4)));
    CKC(cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking));
    CKC(cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking));
    ctx->ev_in.resize(B);
    ctx->ev_done.resize(B);
    for (int i = 0; i < B; ++i) {
      CKC(cudaEventCreateWithFlags(&ctx->ev_in[i], cudaEventDisableTiming));
      CKC(cudaEventCreateWithFlags(&ctx->ev_done[i], cudaEventDisableTiming));
    }
  }
  // the copies may only start once earlier work on the context stream is done with the staging
  cudaEvent_t start;
  CKC(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  CKC(cudaEventRecord(start, ctx->stream));
  CKC(cudaStreamWaitEvent(ctx->h2d, start, 0));
  cudaEventDestroy(start);
  for (int i = 0; i < B; ++i) {
    const BucketInfo& bk = ctx->b[i];
    float* dst = ctx->d_hgrad + (uint64_t)Pl * bk.off;
    for (int c = 0; c < Pl; ++c)
      CKC(cudaMemcpyAsync(dst + (uint64_t)c * bk.n, host_grad + (uint64_t)c * ctx->total_n + bk.off, bk.n * 4,
                          cudaMemcpyHostToDevice, ctx->h2d));
    CKC(cudaEventRecord(ctx->ev_in[i], ctx->h2d));
  }
  for (int i = 0; i < B; ++i) {
    const BucketInfo& bk = ctx->b[i];
    CKC(cudaStreamWaitEvent(ctx->stream, ctx->ev_in[i], 0));
    nebula_status s = nebula_step(ctx, i, ctx->d_hgrad + (uint64_t)Pl * bk.off, ctx->d_hout + bk.off, step);
    if (s != NEBULA_OK) {
      cudaStreamSynchronize(ctx->h2d);
      return s;
    }
    CKC(cudaEventRecord(ctx->ev_done[i], ctx->stream));
    CKC(cudaStreamWaitEvent(ctx->d2h, ctx->ev_done[i], 0));
    CKC(cudaMemcpyAsync(host_out + bk.off, ctx->d_hout + bk.off, bk.n * 4, cudaMemcpyDeviceToHost, ctx->d2h));
  }
  CKC(cudaStreamSynchronize(ctx->d2h));
  CKC(cudaStreamSynchronize(ctx->stream));
  return NEBULA_OK;
}

nebula_status nebula_check(nebula_ctx* ctx) {
  if (!ctx) return NEBULA_ERR_INVALID_ARG;
  DevGuard dg(ctx->device);
  CKC(cudaStreamSynchronize(ctx->stream));
  uint32_t f = 0;
  CKC(cudaMemcpy(&f, ctx->d_flags, 4, cudaMemcpyDeviceToHost));
  CKC(cudaMemset(ctx->d_flags, 0, 4));
  *reinterpret_cast<volatile uint32_t*>(ctx->h_flags) = 0u;
  if (!ctx->loopback && ctx->world) {
    ncclResult_t async_err = ncclSuccess;
    ncclCommGetAsyncError(ctx->world, &async_err);
    if (async_err != ncclSuccess) return fail(ctx, NEBULA_ERR_NCCL, ncclGetErrorString(async_err));
  }
  if (f & kFlagPeerTimeout) return fail(ctx, NEBULA_ERR_NCCL, "P2P exchange: a peer's payload did not arrive (timeout)");
  if (f & kFlagNonfinite) return fail(ctx, NEBULA_ERR_NONFINITE, "non-finite element in g + r");
  if (f & kFlagOverflow) return fail(ctx, NEBULA_ERR_OVERFLOW, "fp16 overflow (|p| >= 65520)");
  return NEBULA_OK;
}

nebula_status nebula_payload_bytes(const nebula_ctx* ctx, int32_t bucket, uint64_t* bytes) {
  if (!ctx || !bytes || bucket < 0 || bucket >= (int)ctx->b.size()) return NEBULA_ERR_INVALID_ARG;
  const BucketInfo& bk = ctx->b[bucket];
  const int m = bk.method >= 0 ? bk.method : (ctx->codec.start_step == 0 ? ctx->codec.method : M_IDENTITY);
  *bytes = payload_bytes_for(m, bk.cn, bk.k, ctx->codec.topk_values);
  return NEBULA_OK;
}

nebula_status nebula_payload_copy(nebula_ctx* ctx, int32_t bucket, int32_t slot, void* host_dst, uint64_t cap) {
  if (!ctx || !host_dst || bucket < 0 || bucket >= (int)ctx->b.size() || slot < 0 || slot >= ctx->P)
    return fail(ctx, NEBULA_ERR_INVALID_ARG, "bad payload_copy arguments");
  uint64_t nbytes = 0;
  nebula_payload_bytes(ctx, bucket, &nbytes);
  if (cap < nbytes) return fail(ctx, NEBULA_ERR_INVALID_ARG, "cap smaller than payload bytes");
  DevGuard dg(ctx->device);
  CKC(cudaStreamSynchronize(ctx->stream));
  const BucketInfo& bk = ctx->b[bucket];
  const int lay = layout_of(ctx, bk.method >= 0 ? bk.method : ctx->codec.method);
  // P2P pull: cluster `slot`'s payload lives in that cluster's own (IPC-mapped) buffer
  const uint8_t* base = sources_of(ctx, bk).p[slot];
  CKC(cudaMemcpy(host_dst, base + bk.so[lay] + (uint64_t)slot * bk.pb[lay], nbytes, cudaMemcpyDeviceToHost));
  return NEBULA_OK;
}

nebula_status nebula_residual_ptr(nebula_ctx* ctx, int32_t bucket, int32_t cluster, float** dev_residual) {
  if (!ctx || !dev_residual || bucket < 0 || bucket >= (int)ctx->b.size())
    return fail(ctx, NEBULA_ERR_INVALID_ARG, "bad residual_ptr arguments");
  int c;
  if (ctx->loopback) {
    if (cluster < 0 || cluster >= ctx->P) return fail(ctx, NEBULA_ERR_INVALID_ARG, "cluster out of range");
    c = cluster;
  } else {
    if (cluster != ctx->topo.cluster_id) return fail(ctx, NEBULA_ERR_INVALID_ARG, "not this context's cluster");
    c = 0;
  }
  *dev_residual = ctx->d_resid + (uint64_t)c * ctx->total_cn + ctx->b[bucket].coff;
  return NEBULA_OK;
}

uint64_t nebula_kernel_launches(const nebula_ctx* ctx) { return ctx ? ctx->launches : 0; }

nebula_status nebula_set_option(nebula_ctx* ctx, int32_t option, int64_t value) {
  if (!ctx) return NEBULA_ERR_INVALID_ARG;
  if (option == NEBULA_OPT_INT8_KERNEL) {
    if (value < 0 || value > 2) return fail(ctx, NEBULA_ERR_INVALID_ARG, "INT8 kernel option must be in [0, 2]");
    if (value == 2 && (ctx->codec.method == NEBULA_INT8 || ctx->codec.method == NEBULA_FP8 ||
                       ctx->codec.method == NEBULA_FP8_E5M2 ||
                       ctx->codec.method == NEBULA_QSGD) && !ctx->onchip_ok)
      return fail(ctx, NEBULA_ERR_UNSUPPORTED, "cooperative on-chip INT8 kernel not available on this device");
    ctx->int8_kernel = (int)value;
    return NEBULA_OK;
  }
  if (option == NEBULA_OPT_STEP_FUSION) {
    if (value < 0 || value > 12) return fail(ctx, NEBULA_ERR_INVALID_ARG, "step fusion option must be in [0, 12]");
    ctx->step_fusion = (int)value;
    return NEBULA_OK;
  }
  if (option == NEBULA_OPT_FP16_KERNEL) {
    if (value < 0 || value > 1) return fail(ctx, NEBULA_ERR_INVALID_ARG, "FP16 kernel option must be 0 or 1");
    ctx->fp16_kernel = (int)value;
    return NEBULA_OK;
  }
  if (option == NEBULA_OPT_TOPK_REDUCE) {
    if (value < 0 || value > 1) return fail(ctx, NEBULA_ERR_INVALID_ARG, "top-k reduce option must be 0 or 1");
    ctx->topk_reduce = (int)value;
    return NEBULA_OK;
  }
  if (option == NEBULA_OPT_SR_SEED) {
    ctx->sr_seed = (uint64_t)value;
    return NEBULA_OK;
  }
  if (option == NEBULA_OPT_EXACT_SCALE) {
    if (value < 0 || value > 1) return fail(ctx, NEBULA_ERR_INVALID_ARG, "exact-scale option must be 0 or 1");
    for (const auto& bk : ctx->b)
      if (bk.state != ST_IDLE) return fail(ctx, NEBULA_ERR_STATE, "change the scale mode only between steps");
    ctx->exact_scale = (int)value;
    return NEBULA_OK;
  }
  if (option == NEBULA_OPT_EXCHANGE) {
    if (value < 0 || value > 3) return fail(ctx, NEBULA_ERR_INVALID_ARG, "exchange option must be in [0, 3]");
    if (ctx->loopback) return NEBULA_OK;   // nothing moves
    if (value >= 2 && !ctx->p2p_ok) return fail(ctx, NEBULA_ERR_UNSUPPORTED, "P2P not available (peers not mappable)");
    if (value == 1 && ctx->self && ctx->P > 1)
      return fail(ctx, NEBULA_ERR_UNSUPPORTED, "SELF transport has no NCCL communicator");
    for (const auto& bk : ctx->b)
      if (bk.state != ST_IDLE) return fail(ctx, NEBULA_ERR_STATE, "change the exchange only between steps");
    ctx->xopt = (int)value;
    ctx->xmode = (value == 1 || !ctx->p2p_ok || ctx->P == 1) ? 1 : (value == 0 ? auto_xmode(ctx) : (int)value);
    return NEBULA_OK;
  }
  if (option == NEBULA_OPT_TOPK_STAGE) {
    if (value < 0 || value > 1) return fail(ctx, NEBULA_ERR_INVALID_ARG, "top-k stage option must be 0 or 1");
    ctx->tk.stage_tma = value == 1;
    return NEBULA_OK;
  }
  if (option == NEBULA_OPT_PIPELINE) {
    if (value < 0 || value > 2) return fail(ctx, NEBULA_ERR_INVALID_ARG, "pipeline option must be in [0, 2]");
    ctx->topk_pipe = (int)value;
    return NEBULA_OK;
  }
  if (option == NEBULA_OPT_INTRA) {
    if (value < 0 || value > 1) return fail(ctx, NEBULA_ERR_INVALID_ARG, "intra option must be 0 or 1");
    if (value == 1 && ctx->G > 1 && !ctx->intra)
      return fail(ctx, NEBULA_ERR_UNSUPPORTED, "no intra-cluster NCCL communicator (SELF transport)");
    for (const auto& bk : ctx->b)
      if (bk.state != ST_IDLE) return fail(ctx, NEBULA_ERR_STATE, "change the intra-cluster hop only between steps");
    ctx->intra_opt = (int)value;
    return NEBULA_OK;
  }
  return fail(ctx, NEBULA_ERR_INVALID_ARG, "unknown option");
}

int32_t nebula_exchange_mode(const nebula_ctx* ctx) { return ctx ? ctx->xmode : -1; }

int32_t nebula_intra_mode(const nebula_ctx* ctx) {
  if (!ctx) return -1;
  if (ctx->G == 1) return 0;
  return intra_p2p_on(ctx) ? 2 : 1;
}

nebula_status nebula_timing_enable(nebula_ctx* ctx, int32_t on) {
  if (!ctx) return NEBULA_ERR_INVALID_ARG;
  ctx->timing = on != 0;
  return NEBULA_OK;
}

nebula_status nebula_timing_read(nebula_ctx* ctx, nebula_phase_time* out, int32_t cap, int32_t* n_out) {
  if (!ctx || !n_out || (cap > 0 && !out)) return NEBULA_ERR_INVALID_ARG;
  DevGuard dg(ctx->device);
  CKC(cudaStreamSynchronize(ctx->stream));
  double ms[PH_COUNT] = {0};
  uint32_t cnt[PH_COUNT] = {0};
  for (const auto& r : ctx->recs) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, ctx->evs[r.a], ctx->evs[r.b]) == cudaSuccess) {
      ms[r.ph] += t;
      cnt[r.ph] += 1;
    }
  }
  ctx->recs.clear();
  ctx->open.clear();
  ctx->ev_next = 0;
  int n = 0;
  for (int p = 0; p < PH_COUNT; ++p) {
    if (!cnt[p]) continue;
    if (n < cap) out[n] = nebula_phase_time{(uint32_t)p, cnt[p], ms[p]};
    ++n;
  }
  *n_out = n;
  return NEBULA_OK;
}

const char* nebula_phase_name(uint32_t phase) {
  static const char* names[PH_COUNT] = {
      "identity_pack", "fp16_ef_pack", "int8_ef_absmax", "int8_ef_quant_pack", "topk_ef_sample",
      "topk_bracket", "topk_classify", "topk_resolve", "topk_fallback", "topk_merge_pack",
      "dense_decompress_reduce", "topk_offsets", "sparse_decompress_reduce", "nccl_allgather_payload",
      "nccl_reducescatter_intra", "nccl_allgather_intra", "memset", "int8_fused_ef_quant_pack",
      "p2p_exchange_flags", "int8_fused_step", "fp8_ef_quant_pack", "nccl_allreduce_cluster_scale", "qsgd_ef_quant_pack",
      "intra_rs_push", "intra_rs_reduce", "intra_ag_pull", "intra_scale_mail", "p2p_flags_intra_rs", "p2p_flags_intra_ag",
      "fp16_fused_step"};
  return phase < PH_COUNT ? names[phase] : "unknown";
}

nebula_status nebula_sync_destroy(nebula_ctx* ctx) {
  release(ctx);
  return NEBULA_OK;
}

const char* nebula_last_error(const nebula_ctx* ctx) { return ctx ? ctx->err.c_str() : g_init_error.c_str(); }

}  // extern "C"

// ============================================================================ top-k plumbing
nebula_status topk_setup(nebula_ctx* ctx);
nebula_status nebula_topk_stats(nebula_ctx* ctx, int32_t bucket, int32_t cluster, nebula_topk_info* out);
#include "topk_host.inc"
