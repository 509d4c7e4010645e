// kernels.h — host-side launchers of the sm_100a kernels (internal to libnebula_sync.so).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "nebula_internal.cuh"

namespace nb {

// Phase ids of the per-kernel timers (nebula_timing_read); names in nebula_phase_name.
enum Phase : int {
  PH_IDENTITY = 0, PH_FP16, PH_ABSMAX, PH_INT8_QUANT, PH_TOPK_A, PH_TOPK_BRACKET, PH_TOPK_CLASSIFY,
  PH_TOPK_RESOLVE, PH_TOPK_FALLBACK, PH_TOPK_MERGE, PH_REDUCE_DENSE, PH_TOPK_OFFSETS, PH_TOPK_REDUCE,
  PH_NCCL_EXCHANGE, PH_NCCL_RS, PH_NCCL_AG, PH_MEMSET, PH_INT8_ONCHIP, PH_P2P_FLAGS, PH_INT8_STEP, PH_FP8_QUANT,
  PH_NCCL_SCALE, PH_QSGD_QUANT, PH_RS_PUSH, PH_RS_REDUCE, PH_AG_PULL, PH_SCALE_MAIL,
  PH_P2P_FLAGS_RS, PH_P2P_FLAGS_AG, PH_FP16_STEP, PH_COUNT
};

struct Launch {
  cudaStream_t stream;
  int num_sms;
  uint64_t* launches;                       // incremented once per kernel enqueued
  void (*mark)(void*, int phase, int end);  // optional CUDA-event timer hook
  void* mctx;
};

// Persistent-grid size for a grid-stride kernel: exactly the resident CTAs (SMs x the
// kernel's occupancy), never more than the work — a grid larger than one wave leaves a
// partial second wave (the tail effect ncu showed on the reducer).
int occupancy_per_sm(const void* kernel, int threads, size_t smem);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for the CURRENT device, once per
// (device, kernel, bytes) — the attribute is per device context (thread-safe cache).
void ensure_smem_attr(const void* kernel, size_t bytes);
inline unsigned persistent_grid(const Launch& L, uint64_t chunks, const void* kernel, int threads, size_t smem = 0) {
  uint64_t g = (uint64_t)L.num_sms * (uint64_t)occupancy_per_sm(kernel, threads, smem);
  if (chunks < g) g = chunks;
  return (unsigned)(g ? g : 1);
}

// RAII timer around one launch site: records an event pair on the launch stream.
struct Mark {
  const Launch& L;
  int ph;
  Mark(const Launch& l, int p) : L(l), ph(p) { if (L.mark) L.mark(L.mctx, ph, 0); }
  ~Mark() { if (L.mark) L.mark(L.mctx, ph, 1); }
};

// Load every kernel of the library into the current device's context (called by
// nebula_sync_init).  CUDA's lazy loading would otherwise load a kernel at its first launch,
// which may wait for the kernels already running — and the P2P flag kernels spin until a peer
// (another stream or process) runs: a launch-time load behind such a spin can deadlock.
void preload_kernels();
void preload_dense();
void preload_ws();
void preload_intra();
void preload_topk();

// ---- dense codecs (kernels_dense.cu) ----
// IDENTITY: payload <- g (+ non-finite check).  Residual untouched (R15).
void launch_identity(const Launch& L, bool vec, const Item* items, int nitems, uint64_t chunks,
                     const float* g, const Dests& slots, uint32_t* flags);
// FP16 + EF, single pass: p = g + r; h = RNE16(p); r <- p - h; flags.
void launch_fp16(const Launch& L, bool ef, bool vec, const Item* items, int nitems, uint64_t chunks,
                 const float* g, float* r, const Dests& slots, uint32_t* flags);
// FP16 + EF with a TMA ring (16-B aligned calls; one CTA per SM, producer warp + 31 consumers).
bool launch_fp16_tma(const Launch& L, bool ef, const Item* items, int nitems, uint64_t chunks, const float* g,
                     float* r, const Dests& slots, uint32_t* flags);
// INT8 pass 1: scratch[sidx] <- max over the item of |g + r| bits (atomicMax; zeroed by caller).
void launch_absmax(const Launch& L, bool ef, bool vec, const Item* items, int nitems, uint64_t chunks,
                   const float* g, const float* r, uint32_t* scratch);
// INT8 pass 2: scale from scratch, quantize + pack, r <- p - q*s.
void launch_int8_quant(const Launch& L, bool ef, bool vec, const Item* items, int nitems, uint64_t chunks,
                       const float* g, float* r, const Dests& slots, const uint32_t* scratch, uint32_t* flags);
// FP8 pass 2 (NEXT-4): fmt 1 = E4M3 (scale fl(m/448)), 2 = E5M2 (fl(m/57344)); quantise + pack,
// r <- p - D.
void launch_fp8_quant(const Launch& L, bool ef, bool vec, const Item* items, int nitems, uint64_t chunks,
                      const float* g, float* r, const Dests& slots, const uint32_t* scratch, uint32_t* flags, int fmt);
// QSGD pass 2 (NEXT-4, R32): INT8 scale, stochastic rounding with counter-based uniforms.
void launch_qsgd_quant(const Launch& L, bool ef, bool vec, const Item* items, int nitems, uint64_t chunks,
                       const float* g, float* r, const Dests& slots, const uint32_t* scratch, uint32_t* flags,
                       const SrArgs& sr);
// INT8 (kind 0) / FP8 E4M3 (kind 1) / QSGD (kind 2) / FP8 E5M2 (kind 3) single HBM pass: the warp-specialised TMA
// kernel with that quantiser (16-B aligned calls; cooperative, one CTA per SM; done_words >=
// nitems words, zeroed by the launcher).
void launch_ws_compress(const Launch& L, bool ef, int kind, const Item* items, int nitems, const float* g, float* r,
                        const Dests& slots, uint32_t* scratch, uint32_t* flags, uint32_t* done_words,
                        const SrArgs& sr);
// capacity(): false when the device cannot host the single-pass kernels' cooperative grid
// (one 1024-thread CTA per SM with the TMA rings); the caller then uses the two-pass kernels.
bool int8_onchip_capacity(int device, uint64_t* max_elems, int* grid, size_t* smem);
// Dense decompress + tree-average over P slots.
void launch_reduce_dense(const Launch& L, int method, int P, bool vec, const RItem* items, int nitems,
                         uint64_t chunks, const Dests& slots, float* out);

// ---- P2P push exchange (kernels_dense.cu) ----
struct Peers {
  unsigned long long* arrive[8];  // every cluster's arrival flags (IPC-mapped; own at [me])
  int n, me;
};
// Fused INT8 step (compress + P2P/loopback exchange + average in one cooperative kernel).
// items/nitems: the compress table of the call (bucket-major, PL items per bucket); ritems: the
// reduce table (one per bucket); src.n = P sources; pe.n > 1 = P2P peers to signal / wait for.
void launch_int8_step(const Launch& L, bool ef, const Item* items, int nitems, const float* g, float* r,
                      const Dests& dst, uint32_t* scratch, uint32_t* flags, uint32_t* bar_words, const RItem* ritems,
                      int b0, int PL, const Dests& src, float* obase, const Peers& pe, unsigned long long* local_arrive,
                      uint64_t seq, int config, int kind, const SrArgs& sr);   // kind 0 INT8, 1 E4M3, 2 QSGD, 3 E5M2

// Fused FP16 step (compress + LOOPBACK / P2P-pull exchange + average in one cooperative kernel);
// config 0 LOOPBACK warp split, 1 P2P pull.  bar_words: nitems words.
void launch_fp16_step(const Launch& L, bool ef, const Item* items, int nitems, const float* g, float* r,
                      const Dests& dst, uint32_t* flags, uint32_t* bar_words, const RItem* ritems, int b0, int PL,
                      const Dests& src, float* obase, const Peers& pe, unsigned long long* local_arrive, uint64_t seq,
                      int config);

// For buckets [lo, hi): tell every peer that this cluster's payloads of exchange `seq` are in
// its slots (system-scope release), then wait until every peer said the same to us.
void launch_exchange_flags(const Launch& L, const Peers& pe, unsigned long long* local_arrive, int lo, int hi,
                           uint64_t seq, uint32_t* flags, int phase = PH_P2P_FLAGS);

// ---- intra-cluster hop over NVLink peer memory, G > 1 (kernels_intra.cu) ----
struct IItem {          // one bucket of an intra-cluster call
  uint64_t off;         // element offset of the bucket in the caller's buffers (gradient / output)
  uint64_t coff;        // element offset of the shard in library coded buffers (multiple of 4)
  uint64_t cn;          // shard elements (bucket numel / G)
  uint64_t chunk0;      // first 4096-element chunk of this item in the launch
};
struct PeerF { float* p[8]; int n, me; };   // a float buffer of every GPU of the cluster (own at [me])
struct PeerU { uint32_t* p[8]; };
// RS step 1: slice j of this GPU's gradient -> peer j's receive buffer, slot me (NVLink stores).
void launch_rs_push(const Launch& L, bool vec, const IItem* items, int nitems, uint64_t chunks, const float* g,
                    const PeerF& recv, uint64_t stride);
// RS step 2 (after the flags): shard = fl(sum in local-rank order) / G.
void launch_rs_reduce(const Launch& L, bool vec, const IItem* items, int nitems, uint64_t chunks, const float* g,
                      const float* recv, uint64_t stride, int G, int me, float* shard);
// AG (after the flags): out[slice j] = GPU j's averaged shard (NVLink loads).
void launch_ag_pull(const Launch& L, bool vec, const IItem* items, int nitems, uint64_t chunks, const PeerF& shards,
                    float* out);
// NEXT-3 exact cluster scale: scratch[b] <- max over the G GPUs' scratch[b] (mailbox + flags).
void launch_scale_mail(const Launch& L, const Peers& pe, const PeerU& mails, uint32_t* scratch, uint32_t* my_mail,
                       unsigned long long* local_arrive, int lo, int hi, uint64_t seq, uint32_t* flags);

// ---- top-k (kernels_topk.cu) ----
struct TopkItem {       // per (cluster, bucket) top-k state, device resident
  uint64_t n, k;
  uint64_t r_off, g_off, slot_off;
  uint64_t chunk0;      // classify-pass chunk base
  uint64_t nchunks;
  uint64_t sample_off;  // into sample buffer (u32 keys)
  uint64_t nsample;
  uint32_t stride;      // sample stride S
  uint32_t sidx;
  uint64_t list_off;    // into winner / candidate lists (entries)
  uint64_t wcap, ccap;  // capacities
  uint64_t status_off;  // into tile-status words
  uint64_t mt0;         // prefix of merge tiles over the launch's items (absolute)
  uint64_t stage_off;   // into the staging buffer (entries); capacity wcap + ccap
  uint32_t value_type;
  uint32_t pad;
};
struct TopkState {      // per item, device resident, rewritten every step
  uint32_t t_lo, t_hi;  // bracket: winners key > t_hi, candidates t_lo <= key <= t_hi
  uint32_t mode;        // 0 bracket, 1 exact (t_lo == t_hi == T, need known)
  uint32_t failed;      // resolve found the bracket invalid -> exact fallback
  uint64_t wcount, ccount;
  uint32_t threshold;   // final T
  uint32_t hist_prefix; // fallback radix state
  uint64_t count_above, need;
  uint64_t rank_left;   // fallback radix: rank still to find inside the prefix
  uint32_t wide;        // resolve on the multi-CTA path (candidate list too long for one CTA)
  uint32_t path;
  float scale;
  uint32_t maxbits;
  unsigned long long wide_above;  // multi-CTA resolve: candidates above the running prefix
  uint32_t stage_ovf;             // pass A ran out of staging space for this bucket -> fallback
  uint32_t wchunk0;               // multi-CTA resolve: first work unit of this item (prefix over items)
};
struct TopkBuffers {
  TopkItem* items;      // [nitems] (bucket-major, cluster-minor: same order as the Item tables)
  TopkState* state;     // [nitems]
  uint32_t* sample;
  uint2* wlist;         // (idx, p bits)
  uint2* clist;
  uint2* clist2;        // compacted candidates of the multi-CTA resolve (merge input for wide items)
  unsigned long long* status;  // per-chunk (winners << 32 | candidates) counts
  unsigned long long* pref;    // per-chunk exclusive prefixes of the counts
  unsigned long long* soff;    // per-chunk offset of its staged entries
  uint2* stage;                // pass-A staging: per chunk W entries then C entries, CTA-private regions
  uint64_t stage_entries;      // staging capacity (split evenly between the pass-A CTAs)
  uint64_t* splits;            // merge-path split points, 2 per merge tile
  uint32_t bracket_smem_keys;  // shared-memory sample capacity of k_topk_bracket
  bool stage_tma = true;       // NEBULA_OPT_TOPK_STAGE: TMA-ring stage pass for 16-B aligned calls
  cudaEvent_t wide_rec = nullptr, wide_wait = nullptr;   // pipelined halves: order their multi-CTA resolve sections
  uint32_t* hist;       // [nitems][2048] fallback histograms
  uint32_t* ctrs;       // [2] any bracket failed, [3] wide-resolve units, [4] any exact-tie bracket
  uint32_t* start;      // sparse-reduce start offsets
  uint64_t* host_mt0;   // host copy of items[].mt0 and merge tiles per item (for grid sizing)
  uint64_t* host_mtiles;
  uint64_t* host_sample_off;  // [nitems + 1] prefix of sample counts
  uint64_t* host_ccap;        // [nitems] candidate capacities (no list longer than kWideMin: no wide resolve)
};
// Runs the whole selection for items [item0, item0 + nitems) (their TopkItem rows), writes
// payloads, updates residuals.  aitems = the call's Item table (same order), g = gradient
// base, r = residual base.
void launch_topk(const Launch& L, bool ef, bool vec, const TopkBuffers& B, int item0, int nitems,
                 uint64_t a_chunks, const Item* aitems, const float* g, float* r, const Dests& slots,
                 uint32_t* flags, int value_type, uint64_t merge_tiles);
// Opt the bracket kernel into `keys` x 4 bytes of dynamic shared memory (once per process).
void topk_prepare_bracket(uint32_t keys);
// Sparse decompress + tree-average (tile merge over the ascending index lists).
// entries = sum over buckets of (k + 1); tiles = sum of ceil(n / 2048).
// zero_begin/zero_count: the output range of the call (filled with +0.0 first).
// start_count = P * sum over the call's buckets of (tiles + 1); variant 0 = tile-interleaved
// (start offsets kernel + CTA tiles), 1 = per-warp contiguous sub-tile ranges.
void launch_reduce_topk(const Launch& L, int value_type, int P, bool vec, const RItem* items, int nitems,
                        uint64_t entries, uint64_t tiles, const Dests& slots, uint32_t* start, float* out,
                        float* zero_begin, uint64_t zero_count, uint64_t start_count, int variant);

}  // namespace nb
