// kernels_topk.cu — exact top-k selection with error feedback, and the sparse reducer.
//
// Selection rule (R11; PAPER.md:63/:99 cite top-k sparsification without defining
// it): the k largest keys key_i = bits(p_i) & 0x7FFFFFFF (|p| order, -0 == +0); equal keys
// resolved by the lower index; payload indices ascending.  The pipeline never sorts:
//
//   S  k_topk_sample   (gather, ~0.5 B/elem) key(fl(g + r)) at every S-th position
//   B  k_topk_bracket  (1 CTA/item) radix-select two ranks of the sample -> bracket
//                       [t_lo, t_hi] that holds the true k-th key with overwhelming odds
//   A  k_topk_stage    (streaming, 12 B/elem) p = g + r -> r; max-abs bits; winners
//                       (key > t_hi) and candidates (t_lo <= key <= t_hi) of each 4096-element
//                       chunk, in index order, staged at a per-chunk slot reserved with one
//                       atomic; per-chunk counts                                  [EF fused]
//   X  k_topk_scan     (1 CTA/item) exclusive scan of the chunk counts -> chunk offsets, totals
//   M  k_topk_move     (one warp per chunk) staged entries -> ascending winner / candidate
//                       lists at the chunk offsets (touches only the entries, ~2% of n)
//   D  k_topk_resolve  (1 CTA/item) verify W < k <= W + C; radix-select the exact threshold T
//                       among the candidates; keep key > T and the first need_T keys == T
//   (fallback, only items whose bracket failed or whose staging overflowed: 3 full
//    radix-histogram passes give the exact T, then a count pass, the scan, an ordered write
//    pass (k_topk_write, positions known up front, so a huge tie set needs no staging) and
//    resolve rerun with t_lo = t_hi = T — bounded memory, exact)
//   F  k_topk_merge    merge-path of the two ascending lists -> payload idx[k], val[k];
//                       residual at the selected positions r = p - D(v)
//
// The reducer scatters each cluster's (idx, val) into shared-memory tiles pre-filled with
// +0.0 and tree-sums them (R16), after a pass that turns each ascending index list into
// per-tile start offsets.
#include <cuda_fp16.h>

#include <algorithm>
#include <new>

#include "dense_common.cuh"
#include "kernels.h"

namespace nb {

constexpr int kSelThreads = 1024;  // single-CTA radix select
constexpr int kMergeThreads = 256, kMergeVT = 8;
constexpr int kMergeTile = kMergeThreads * kMergeVT;   // 2048 outputs per merge CTA
constexpr int kRedTile = 2048;     // elements per sparse-reduce CTA
constexpr uint32_t kWideMin = 131072;  // candidate lists longer than this resolve on many CTAs (one CTA: ~0.1 ms per 75K)

// tile words: (winners << 32) | candidates — per-tile counts, then exclusive prefixes
__device__ __forceinline__ unsigned long long pack_wc(uint64_t w, uint64_t c) { return (w << 32) | c; }

// ---------------------------------------------------------------- block helpers
// Inclusive scan of a 64-bit value over a CTA of NT threads; returns inclusive, *total.
template <int NT>
__device__ __forceinline__ unsigned long long block_incl_scan(unsigned long long v, unsigned long long* smem,
                                                              unsigned long long* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) smem[warp] = v;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = lane < NT / 32 ? smem[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, w, o);
      if (lane >= o) w += t;
    }
    if (lane < NT / 32) smem[lane] = w;
  }
  __syncthreads();
  if (warp > 0) v += smem[warp - 1];
  *total = smem[NT / 32 - 1];
  __syncthreads();
  return v;
}

// hist[nbins] in shared memory (bin value = digit).  Find the bin holding descending rank
// `rank` (1-based): above(b) < rank <= above(b) + hist[b].  Results in *bin/*above (smem).
__device__ void find_bin(const uint32_t* hist, int nbins, uint32_t rank, uint32_t* s_bin, uint32_t* s_above,
                         unsigned long long* scan_smem) {
  // thread t owns descending bins nbins-1-2t, nbins-2-2t
  const int t = threadIdx.x;
  const int b0 = nbins - 1 - 2 * t, b1 = b0 - 1;
  const uint32_t h0 = b0 >= 0 ? hist[b0] : 0, h1 = b1 >= 0 ? hist[b1] : 0;
  unsigned long long tot;
  const unsigned long long incl = block_incl_scan<kSelThreads>((unsigned long long)(h0 + h1), scan_smem, &tot);
  const unsigned long long excl = incl - (h0 + h1);
  if (excl < rank && rank <= incl) {
    if (rank <= excl + h0) { *s_bin = (uint32_t)b0; *s_above = (uint32_t)excl; }
    else { *s_bin = (uint32_t)b1; *s_above = (uint32_t)(excl + h0); }
  }
  __syncthreads();
}

__device__ __forceinline__ void hist_add(uint32_t* hist, bool active, uint32_t bin) {
  // duplicate-heavy input (e.g. all-zero keys) puts a whole warp on one bin: then one lane adds
  // the popcount; otherwise plain per-lane shared atomics (a vote is far cheaper than match.any)
  const unsigned mask = __activemask();
  const unsigned act = __ballot_sync(mask, active);
  if (!act) return;
  const int leader = __ffs(act) - 1;
  const uint32_t b0 = __shfl_sync(mask, bin, leader);
  if (__all_sync(mask, !active || bin == b0)) {
    if ((int)(threadIdx.x & 31) == leader) atomicAdd(&hist[b0], (uint32_t)__popc(act));
  } else if (active) {
    atomicAdd(&hist[bin], 1u);
  }
}

struct Digit { int shift, bits; };
__device__ __forceinline__ Digit digit_of(int d) {
  return d == 0 ? Digit{20, 11} : (d == 1 ? Digit{9, 11} : Digit{0, 9});
}

// Radix select inside one CTA: key at descending rank `rank` (1 <= rank <= m) of keys
// produced by get(i), i < m.  Returns T, and *above = #{key > T}.
// Radix select inside one CTA: key at descending rank `rank` (1 <= rank <= m) of the 31-bit
// keys produced by get(i), i < m.  Returns T, and *above = #{key > T}.  `known` leading key
// bits (value taken from known_val) are shared by every key — e.g. all candidates of a bracket
// [t_lo, t_hi] share the common prefix of t_lo and t_hi — so the digits start below them
// (otherwise the first digits would pile every key into one shared-memory bin).
template <class GetKey>
__device__ uint32_t cta_select(GetKey get, uint32_t m, uint32_t rank, uint32_t* above_out, uint32_t* hist,
                               uint32_t* s_misc, unsigned long long* scan_smem, int known = 0,
                               uint32_t known_val = 0) {
  constexpr int U = 8;   // keys in flight per thread (the loop is latency-bound otherwise)
  int lo_bit = 31 - known;                                   // bits [0, lo_bit) still to resolve
  uint32_t prefix = known > 0 ? (known_val >> lo_bit) : 0u; // value of bits [lo_bit, 31)
  uint32_t above = 0, left = rank;
  while (lo_bit > 0) {
    const int bits = lo_bit < 11 ? lo_bit : 11;
    const int shift = lo_bit - bits, hs = lo_bit;
    const int nb = 1 << bits;
    for (int b = threadIdx.x; b < 2048; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    for (uint32_t i0 = 0; i0 < m; i0 += blockDim.x * U) {
      uint32_t key[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = i0 + u * blockDim.x + threadIdx.x;
        key[u] = i < m ? get(i) : 0u;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = i0 + u * blockDim.x + threadIdx.x;
        const bool act = i < m && ((hs >= 31) || ((key[u] >> hs) == prefix));
        hist_add(hist, act, (key[u] >> shift) & (nb - 1));
      }
    }
    __syncthreads();
    find_bin(hist, nb, left, &s_misc[0], &s_misc[1], scan_smem);
    const uint32_t b = s_misc[0], ab = s_misc[1];
    prefix = (prefix << bits) | b;
    above += ab;
    left -= ab;
    lo_bit = shift;
    __syncthreads();
  }
  *above_out = above;
  return prefix;
}

// ---------------------------------------------------------------- B: bracket from the sample
__global__ void __launch_bounds__(kSelThreads) k_topk_bracket(const TopkItem* __restrict__ titems,
                                                              TopkState* __restrict__ st,
                                                              const uint32_t* __restrict__ sample,
                                                              uint32_t smem_keys, uint32_t* any_tie) {
  extern __shared__ uint32_t s_keys[];   // the item's sample, loaded once for the 6 radix passes
  __shared__ uint32_t hist[2048];
  __shared__ uint32_t misc[4];
  __shared__ unsigned long long scan[32];
  const TopkItem ti = titems[blockIdx.x];
  TopkState& S = st[blockIdx.x];
  const uint32_t ns = (uint32_t)ti.nsample;
  const double ks = (double)ti.k * (double)ns / (double)(ti.n ? ti.n : 1);
  const double delta = 5.0 * sqrt(ks + 1.0) + 16.0;
  const double rh = floor(ks - delta), rl = ceil(ks + delta);
  const uint32_t* smp = sample + ti.sample_off;
  const bool in_smem = ns <= smem_keys;
  if (in_smem) {
    for (uint32_t i = threadIdx.x; i < ns; i += blockDim.x) s_keys[i] = smp[i];
    __syncthreads();
  }
  auto get = [&](uint32_t i) { return in_smem ? s_keys[i] : smp[i]; };
  uint32_t t_hi = 0xFFFFFFFFu, t_lo = 0u, dummy;
  if (ti.k >= ti.n) {          // everything selected: no winners, all candidates
    t_hi = 0xFFFFFFFFu; t_lo = 0u;
  } else {
    if (rh >= 1.0 && ns > 0) t_hi = cta_select(get, ns, (uint32_t)rh, &dummy, hist, misc + 2, scan);
    if (rl <= (double)ns && ns > 0) t_lo = cta_select(get, ns, (uint32_t)rl, &dummy, hist, misc + 2, scan);
    if (t_hi != 0xFFFFFFFFu && t_lo > t_hi) t_lo = t_hi;
  }
  if (threadIdx.x == 0) {
    S.t_lo = t_lo;
    S.t_hi = t_hi;
    S.mode = 0;
    S.path = 0;
    if (t_lo == t_hi) atomicOr(any_tie, 1u);   // k_topk_write's tie pass has work
  }
}

// ---------------------------------------------------------------- S: sample p = g + r
// One thread per sample: key(fl(g_e + r_e)) at e = m * S.  The same binary32 addition as
// pass A, so the sample sees exactly the p the selection will see.
template <bool EF>
__global__ void k_topk_sample(const Item* __restrict__ aitems, const TopkItem* __restrict__ titems, int nitems,
                              uint64_t sbase, uint64_t total, const float* __restrict__ gbase,
                              const float* __restrict__ rbase, uint32_t* __restrict__ sample, uint32_t* ctrs) {
  if (blockIdx.x == 0 && threadIdx.x < 8) ctrs[threadIdx.x] = 0;   // [2] any bracket failed, [3] wide units, [4] any exact-tie bracket
  const uint64_t gi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= total) return;
  const uint64_t a = sbase + gi;
  int lo = 0, hi = nitems - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (titems[mid].sample_off <= a) lo = mid; else hi = mid - 1;
  }
  const TopkItem& ti = titems[lo];
  const uint64_t e = (a - ti.sample_off) * ti.stride;
  const float gv = gbase[aitems[lo].g_off + e];
  const float p = EF ? __fadd_rn(gv, rbase[ti.r_off + e]) : gv;
  sample[a] = abs_bits(p);
}

// ---------------------------------------------------------------- A: EF pass + tile counts
// COUNT_ONLY = false: p = g + r -> r, max-abs, counts.  COUNT_ONLY = true (fallback retry):
// counts over p for the items whose exact threshold was just found.
template <bool COUNT_ONLY, bool EF, bool VEC>
__global__ void __launch_bounds__(kThreads) k_topk_pass(const Item* __restrict__ aitems,
                                                        const TopkItem* __restrict__ titems,
                                                        TopkState* __restrict__ st, int nitems, uint64_t chunks,
                                                        const float* __restrict__ gbase, float* __restrict__ rbase,
                                                        unsigned long long* __restrict__ tiles,
                                                        const uint32_t* any_failed) {
  if (COUNT_ONLY && *((volatile const uint32_t*)any_failed) == 0) return;
  __shared__ unsigned long long s_cnt[kThreads / 32];
  int hint = 0, cur = -1;
  uint32_t m = 0, t_lo = 0, t_hi = 0;
  bool skip = false;
  for (uint64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    const int i = find_item(aitems, nitems, c, hint);
    hint = i;
    if (i != cur) {
      if (!COUNT_ONLY && cur >= 0) {
        const uint32_t w = __reduce_max_sync(0xFFFFFFFFu, m);
        if ((threadIdx.x & 31) == 0 && w) atomicMax(&st[cur].maxbits, w);
      }
      cur = i;
      m = 0;
      t_lo = st[i].t_lo;
      t_hi = st[i].t_hi;
      skip = COUNT_ONLY && st[i].mode != 1;
    }
    if (skip) continue;
    const Item it = aitems[i];
    const TopkItem& ti = titems[i];
    const uint64_t j = c - it.chunk0, n4 = it.n >> 2;
    const float* g = gbase + it.g_off;
    float* r = rbase + it.r_off;
    const float* src = (COUNT_ONLY && EF) ? r : g;
    uint32_t wn = 0, cn = 0;
#pragma unroll
    for (int u = 0; u < kQuadsPerThread; ++u) {
      const uint64_t q = j * kChunkQuads + (uint64_t)u * kThreads + threadIdx.x;
      if (q < n4) {
        float4 p;
        if (VEC || (COUNT_ONLY && EF)) p = ld4_stream(src + 4 * q);
        else p = make_float4(src[4 * q], src[4 * q + 1], src[4 * q + 2], src[4 * q + 3]);
        if constexpr (!COUNT_ONLY && EF) {
          const float4 rv = ld4_stream(r + 4 * q);
          p = make_float4(__fadd_rn(p.x, rv.x), __fadd_rn(p.y, rv.y), __fadd_rn(p.z, rv.z), __fadd_rn(p.w, rv.w));
          st4(r + 4 * q, p);
        }
        const uint32_t k0 = abs_bits(p.x), k1 = abs_bits(p.y), k2 = abs_bits(p.z), k3 = abs_bits(p.w);
        if (!COUNT_ONLY) m = max(m, max(max(k0, k1), max(k2, k3)));
        wn += (k0 > t_hi) + (k1 > t_hi) + (k2 > t_hi) + (k3 > t_hi);
        cn += (k0 >= t_lo && k0 <= t_hi) + (k1 >= t_lo && k1 <= t_hi) + (k2 >= t_lo && k2 <= t_hi) +
              (k3 >= t_lo && k3 <= t_hi);
      }
    }
    if (j == n4 / kChunkQuads && threadIdx.x < (it.n & 3)) {
      const uint64_t e = n4 * 4 + threadIdx.x;
      float p;
      if (COUNT_ONLY) p = src[e];
      else p = EF ? __fadd_rn(g[e], r[e]) : g[e];
      if (!COUNT_ONLY && EF) r[e] = p;
      const uint32_t k0 = abs_bits(p);
      if (!COUNT_ONLY) m = max(m, k0);
      wn += k0 > t_hi;
      cn += (k0 >= t_lo && k0 <= t_hi);
    }
    unsigned long long v = pack_wc(wn, cn);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if ((threadIdx.x & 31) == 0) s_cnt[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t = 0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) t += s_cnt[w];
      tiles[ti.status_off + j] = t;
    }
    __syncthreads();
  }
  if (!COUNT_ONLY && cur >= 0) {
    const uint32_t w = __reduce_max_sync(0xFFFFFFFFu, m);
    if ((threadIdx.x & 31) == 0 && w) atomicMax(&st[cur].maxbits, w);
  }
}

// ---------------------------------------------------------------- A: EF pass + classify + stage
// TMA = false: plain vector loads, kThreads threads, 3 CTAs / SM.  TMA = true (16-B aligned
// calls): one producer warp bulk-loads each chunk's g and r tiles into a kStageNS-deep
// shared-memory ring (cp.async.bulk + mbarrier transaction counts, L2 evict_first) while the
// kThreads consumer threads — the same per-thread code, reading the tiles from shared memory —
// form p, stage and count; consumers synchronise on named barrier 1 (the producer runs ahead).
constexpr int kStageNS = 3;
struct __align__(128) StageTile {
  float4 g[kChunkQuads];
  float4 r[kChunkQuads];
};
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" :: "n"(kThreads) : "memory"); }

template <bool EF, bool VEC, bool TMA>
__global__ void __launch_bounds__(TMA ? kThreads + 32 : kThreads, TMA ? 2 : 3)
    k_topk_stage(const Item* __restrict__ aitems, const TopkItem* __restrict__ titems, TopkState* __restrict__ st,
                 int nitems, uint64_t chunks, const float* __restrict__ gbase, float* __restrict__ rbase,
                 unsigned long long* __restrict__ counts, unsigned long long* __restrict__ soff,
                 uint2* __restrict__ stage, uint64_t region) {
  // warp totals, double-buffered by chunk parity: one barrier per chunk
  __shared__ unsigned long long s_wt[2][kThreads / 32], s_ct[2][kThreads / 32];
  extern __shared__ __align__(128) unsigned char stage_smem[];
  StageTile* ring = reinterpret_cast<StageTile*>(stage_smem);
  __shared__ __align__(8) uint64_t full[kStageNS], empty[kStageNS];
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < kStageNS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], kThreads / 32); }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x < 32) {   // ---------------- producer
      if (threadIdx.x != 0) return;
      const uint64_t pol = l2_evict_first();
      int hint = 0;
      uint32_t f = 0;
      for (uint64_t c = blockIdx.x; c < chunks; c += gridDim.x, ++f) {
        const int i = find_item(aitems, nitems, c, hint);
        hint = i;
        const Item it = aitems[i];
        const uint64_t j = c - it.chunk0, n4 = it.n >> 2, q0 = j * kChunkQuads;
        const uint32_t nq = q0 < n4 ? (uint32_t)min((uint64_t)kChunkQuads, n4 - q0) : 0u;
        const uint32_t sl = f % kStageNS, use = f / kStageNS;
        if (use) mbar_wait(&empty[sl], (use - 1) & 1u);
        if (nq) {
          mbar_expect_tx(&full[sl], nq * (EF ? 32u : 16u));
          bulk_g2s(ring[sl].g, gbase + it.g_off + 4 * q0, nq * 16u, &full[sl], pol);
          if (EF) bulk_g2s(ring[sl].r, rbase + it.r_off + 4 * q0, nq * 16u, &full[sl], pol);
        } else {
          mbar_arrive(&full[sl]);
        }
      }
      return;
    }
  }
  const int tid = TMA ? (int)threadIdx.x - 32 : (int)threadIdx.x;
  // this CTA's private staging region: entries are appended in chunk order, no atomics
  uint64_t pos = (uint64_t)blockIdx.x * region;
  const uint64_t region_end = pos + region;
  int par = 0;
  int hint = 0, cur = -1;
  uint32_t m = 0, t_lo = 0, t_hi = 0;
  const int lane = tid & 31, warp = tid >> 5;
  uint32_t f = 0;
  for (uint64_t c = blockIdx.x; c < chunks; c += gridDim.x, ++f) {
    const int i = find_item(aitems, nitems, c, hint);
    hint = i;
    if (i != cur) {
      if (cur >= 0) {
        const uint32_t w = __reduce_max_sync(0xFFFFFFFFu, m);
        if (lane == 0 && w) atomicMax(&st[cur].maxbits, w);
      }
      cur = i;
      m = 0;
      t_lo = st[i].t_lo;
      t_hi = st[i].t_hi;
    }
    // exact-tie bracket (t_lo == t_hi == the k-th key): the candidates are ties of which only the
    // first need_T by index are wanted — possibly a huge set (e.g. all zeros of an embedding
    // bucket), so they are not staged; the ordered write pass emits them at known offsets
    const bool tie_mode = t_lo == t_hi;
    const Item it = aitems[i];
    const TopkItem& ti = titems[i];
    const uint64_t j = c - it.chunk0, n4 = it.n >> 2;
    const float* g = gbase + it.g_off;
    float* r = rbase + it.r_off;
    uint32_t kb[kQuadsPerThread][4];
    float4 gv[kQuadsPerThread], rv[kQuadsPerThread];
    const uint32_t sl = f % kStageNS;
    if constexpr (TMA) mbar_wait(&full[sl], (f / kStageNS) & 1u);
#pragma unroll
    for (int u = 0; u < kQuadsPerThread; ++u) {
      const uint64_t q = j * kChunkQuads + (uint64_t)u * kThreads + tid;
      if (q < n4) {
        if constexpr (TMA) {
          gv[u] = ring[sl].g[u * kThreads + tid];
          if constexpr (EF) rv[u] = ring[sl].r[u * kThreads + tid];
        } else {
          if constexpr (VEC) gv[u] = ld4_stream(g + 4 * q);
          else gv[u] = make_float4(g[4 * q], g[4 * q + 1], g[4 * q + 2], g[4 * q + 3]);
          if constexpr (EF) rv[u] = ld4_stream(r + 4 * q);
        }
      }
    }
    if constexpr (TMA) {   // the tile is in registers: hand the ring slot back to the producer
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[sl]);
    }
    unsigned long long pw = 0, pc = 0;
#pragma unroll
    for (int u = 0; u < kQuadsPerThread; ++u) {
      const uint64_t q = j * kChunkQuads + (uint64_t)u * kThreads + tid;
      uint32_t wn = 0, cn = 0;
      if (q < n4) {
        float4 p = gv[u];
        if constexpr (EF) {
          p = make_float4(__fadd_rn(p.x, rv[u].x), __fadd_rn(p.y, rv[u].y), __fadd_rn(p.z, rv[u].z),
                          __fadd_rn(p.w, rv[u].w));
          st4(r + 4 * q, p);
        }
        kb[u][0] = __float_as_uint(p.x); kb[u][1] = __float_as_uint(p.y);
        kb[u][2] = __float_as_uint(p.z); kb[u][3] = __float_as_uint(p.w);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t key = kb[u][e] & 0x7FFFFFFFu;
          m = max(m, key);
          wn += key > t_hi;
          cn += (key >= t_lo) & (key <= t_hi);
        }
      } else {
        kb[u][0] = kb[u][1] = kb[u][2] = kb[u][3] = 0;
      }
      pw |= (unsigned long long)wn << (12 * u);
      pc |= (unsigned long long)cn << (12 * u);
    }
    uint32_t tkb = 0, tw = 0, tcn = 0;
    const bool has_tail = (j == n4 / kChunkQuads) && tid < (it.n & 3);
    if (has_tail) {
      const uint64_t e = n4 * 4 + tid;
      const float p = EF ? __fadd_rn(g[e], r[e]) : g[e];
      if constexpr (EF) r[e] = p;
      tkb = __float_as_uint(p);
      const uint32_t key = tkb & 0x7FFFFFFFu;
      m = max(m, key);
      tw = key > t_hi;
      tcn = (key >= t_lo) & (key <= t_hi);
    }
    // element order inside the chunk: (field u = 0..3 then tail, thread, element)
    pw |= (unsigned long long)tw << 48;
    pc |= (unsigned long long)tcn << 48;
    unsigned long long iw = pw, ic = pc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long a1 = __shfl_up_sync(0xFFFFFFFFu, iw, o);
      const unsigned long long a2 = __shfl_up_sync(0xFFFFFFFFu, ic, o);
      if (lane >= o) { iw += a1; ic += a2; }
    }
    if (lane == 31) { s_wt[par][warp] = iw; s_ct[par][warp] = ic; }
    if constexpr (TMA) consumers_sync(); else __syncthreads();
    unsigned long long ew = iw - pw, ec = ic - pc, totw = 0, totc = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
      const unsigned long long a1 = s_wt[par][w], a2 = s_ct[par][w];
      if (w < warp) { ew += a1; ec += a2; }
      totw += a1;
      totc += a2;
    }
    par ^= 1;
    uint32_t baseW[kQuadsPerThread + 1], baseC[kQuadsPerThread + 1];
    uint32_t accW = 0, accC = 0;
#pragma unroll
    for (int u = 0; u <= kQuadsPerThread; ++u) {
      baseW[u] = accW + (uint32_t)((ew >> (12 * u)) & 0xFFF);
      baseC[u] = accC + (uint32_t)((ec >> (12 * u)) & 0xFFF);
      accW += (uint32_t)((totw >> (12 * u)) & 0xFFF);
      accC += (uint32_t)((totc >> (12 * u)) & 0xFFF);
    }
    const uint32_t tileW = accW, tileC = accC;
    const uint32_t staged = tileW + (tie_mode ? 0u : tileC);
    const uint64_t base = pos;                      // identical in every thread of the CTA
    const bool fits = pos + staged <= region_end;
    if (fits) pos += staged;
    if (tid == 0) {
      counts[ti.status_off + j] = pack_wc(tileW, tileC);
      soff[ti.status_off + j] = base;
      if (!fits) atomicOr(&st[i].stage_ovf, 1u);   // this bucket goes to the exact fallback
    }
    if (staged && fits) {
      uint2* S = stage;
#pragma unroll
      for (int u = 0; u < kQuadsPerThread; ++u) {
        const uint64_t q = j * kChunkQuads + (uint64_t)u * kThreads + tid;
        if (q < n4) {
          uint32_t w = baseW[u], cc = baseC[u];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t key = kb[u][e] & 0x7FFFFFFFu;
            const uint32_t idx = (uint32_t)(4 * q + e);
            if (key > t_hi) {
              S[base + w++] = make_uint2(idx, kb[u][e]);
            } else if (key >= t_lo && !tie_mode) {
              S[base + tileW + cc++] = make_uint2(idx, kb[u][e]);
            }
          }
        }
      }
      if (has_tail) {
        const uint32_t key = tkb & 0x7FFFFFFFu;
        const uint32_t idx = (uint32_t)(n4 * 4 + tid);
        if (key > t_hi) S[base + baseW[kQuadsPerThread]] = make_uint2(idx, tkb);
        else if (key >= t_lo && !tie_mode) S[base + tileW + baseC[kQuadsPerThread]] = make_uint2(idx, tkb);
      }
    }
  }
  if (cur >= 0) {
    const uint32_t w = __reduce_max_sync(0xFFFFFFFFu, m);
    if (lane == 0 && w) atomicMax(&st[cur].maxbits, w);
  }
}

// ---------------------------------------------------------------- M: staged -> ordered lists
// One warp per chunk: copy its W staged winners to wl[prefix_W ...] and its C candidates to
// cl[prefix_C ...].  Items whose staging overflowed are skipped (resolve fails them).
__global__ void __launch_bounds__(256) k_topk_move(const Item* __restrict__ aitems, const TopkItem* __restrict__ titems,
                                                   const TopkState* __restrict__ st, int nitems, uint64_t chunks,
                                                   const unsigned long long* __restrict__ counts,
                                                   const unsigned long long* __restrict__ pref,
                                                   const unsigned long long* __restrict__ soff,
                                                   const uint2* __restrict__ stage, uint2* __restrict__ wl,
                                                   uint2* __restrict__ cl) {
  const uint64_t c = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= chunks) return;
  int lo = 0, hi = nitems - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (aitems[mid].chunk0 <= c) lo = mid; else hi = mid - 1;
  }
  const TopkItem& ti = titems[lo];
  const TopkState& S = st[lo];
  if (S.failed == 2 || S.stage_ovf) return;   // overflowed buckets go to the fallback
  const bool tie_mode = S.t_lo == S.t_hi;       // ties are emitted by k_topk_write
  const uint64_t j = c - aitems[lo].chunk0;
  const unsigned long long cnt = counts[ti.status_off + j];
  const uint32_t W = (uint32_t)(cnt >> 32), C = (uint32_t)(cnt & 0xFFFFFFFFu);
  if (!(W + C)) return;
  const unsigned long long pf = pref[ti.status_off + j];
  const uint64_t pw = pf >> 32, pc = pf & 0xFFFFFFFFull;
  const uint2* src = stage + soff[ti.status_off + j];
  uint2* dw = wl + ti.list_off;
  uint2* dc = cl + ti.list_off;
  for (uint32_t x = lane; x < W; x += 32)
    if (pw + x < ti.wcap) dw[pw + x] = src[x];
  if (!tie_mode)
    for (uint32_t x = lane; x < C; x += 32)
      if (pc + x < ti.ccap) dc[pc + x] = src[W + x];
}

// ---------------------------------------------------------------- X: scan tile counts
// 1 CTA per item: exclusive prefix of the (W, C) tile words in place; totals; after pass A
// also the non-finite check and the int8 value scale (both need the bucket's max).
__global__ void __launch_bounds__(kSelThreads) k_topk_scan(const TopkItem* __restrict__ titems,
                                                           TopkState* __restrict__ st,
                                                           const unsigned long long* __restrict__ tiles,
                                                           unsigned long long* __restrict__ pref, int retry,
                                                           uint32_t* flags, int value_type,
                                                           const uint32_t* any_failed) {
  if (retry && *((volatile const uint32_t*)any_failed) == 0) return;
  __shared__ unsigned long long scan[32];
  const TopkItem ti = titems[blockIdx.x];
  TopkState& S = st[blockIdx.x];
  if (retry) {
    if (S.mode != 1 || S.failed == 2) return;
  } else {
    const uint32_t mb = S.maxbits;
    if (nonfinite_bits(mb)) {
      if (threadIdx.x == 0) { S.failed = 2; atomicOr(flags, kFlagNonfinite); }
      return;
    }
    if (threadIdx.x == 0) S.scale = value_type == V_I8 ? int8_scale_from_bits(mb) : 1.0f;
  }
  const unsigned long long* tw = tiles + ti.status_off;
  unsigned long long* pw = pref + ti.status_off;
  unsigned long long carry = 0;
  for (uint64_t j0 = 0; j0 < ti.nchunks; j0 += kSelThreads) {
    const uint64_t j = j0 + threadIdx.x;
    const unsigned long long v = j < ti.nchunks ? tw[j] : 0ull;
    unsigned long long tot;
    const unsigned long long incl = block_incl_scan<kSelThreads>(v, scan, &tot);
    if (j < ti.nchunks) pw[j] = carry + incl - v;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    S.wcount = carry >> 32;
    S.ccount = carry & 0xFFFFFFFFull;
  }
}

// ---------------------------------------------------------------- C: ordered write
template <bool VEC>
__global__ void __launch_bounds__(kThreads) k_topk_write(const Item* __restrict__ aitems,
                                                         const TopkItem* __restrict__ titems,
                                                         const TopkState* __restrict__ st, int nitems, uint64_t chunks,
                                                         const float* __restrict__ pbase, bool p_in_r,
                                                         const float* __restrict__ gbase,
                                                         uint2* __restrict__ wl, uint2* __restrict__ cl,
                                                         const unsigned long long* __restrict__ pref, int retry,
                                                         const uint32_t* any_failed) {
  // retry == 1: fallback buckets (both lists); retry == 2: exact-tie buckets of the first
  // pass (ties only, winners were staged)
  // any_failed: retry 1 -> "some bracket failed", retry 2 -> "some bracket is an exact tie"
  if (*((volatile const uint32_t*)any_failed) == 0) return;
  __shared__ unsigned long long s_wt[kThreads / 32], s_ct[kThreads / 32];
  int hint = 0;
  for (uint64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    const int i = find_item(aitems, nitems, c, hint);
    hint = i;
    const TopkState& S = st[i];
    if (S.failed == 2) continue;
    if (retry == 1 && S.mode != 1) continue;
    if (retry == 2 && (S.t_lo != S.t_hi || S.stage_ovf)) continue;
    const bool ties_only = retry == 2;
    // tie mode: the selection takes the first need_T = k - W ties in index order, so chunks
    // whose tie prefix already reaches need_T write nothing
    const uint64_t cap_c = ties_only ? min((uint64_t)titems[i].ccap, (uint64_t)(titems[i].k > S.wcount ? titems[i].k - S.wcount : 0ull))
                                     : (uint64_t)titems[i].ccap;
    if (ties_only && (pref[titems[i].status_off + (c - aitems[i].chunk0)] & 0xFFFFFFFFull) >= cap_c) continue;
    const Item it = aitems[i];
    const TopkItem& ti = titems[i];
    const uint64_t j = c - it.chunk0, n4 = it.n >> 2;
    const uint32_t t_lo = S.t_lo, t_hi = S.t_hi;
    const float* p = p_in_r ? pbase + it.r_off : gbase + it.g_off;
    const bool vec = p_in_r || VEC;
    uint32_t kb[kQuadsPerThread][4];
    unsigned long long pw = 0, pc = 0;
#pragma unroll
    for (int u = 0; u < kQuadsPerThread; ++u) {
      const uint64_t q = j * kChunkQuads + (uint64_t)u * kThreads + threadIdx.x;
      uint32_t wn = 0, cn = 0;
      if (q < n4) {
        float4 v = vec ? ld4_stream(p + 4 * q) : make_float4(p[4 * q], p[4 * q + 1], p[4 * q + 2], p[4 * q + 3]);
        kb[u][0] = __float_as_uint(v.x); kb[u][1] = __float_as_uint(v.y);
        kb[u][2] = __float_as_uint(v.z); kb[u][3] = __float_as_uint(v.w);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t key = kb[u][e] & 0x7FFFFFFFu;
          wn += key > t_hi;
          cn += (key >= t_lo) & (key <= t_hi);
        }
      } else {
        kb[u][0] = kb[u][1] = kb[u][2] = kb[u][3] = 0;
      }
      pw |= (unsigned long long)wn << (12 * u);
      pc |= (unsigned long long)cn << (12 * u);
    }
    // tail elements (n % 4, after every quad of the item) are a 5th field
    uint32_t tkb = 0, tw = 0, tcn = 0;
    const bool has_tail = (j == n4 / kChunkQuads) && threadIdx.x < (it.n & 3);
    if (has_tail) {
      tkb = __float_as_uint(p[n4 * 4 + threadIdx.x]);
      const uint32_t key = tkb & 0x7FFFFFFFu;
      tw = key > t_hi;
      tcn = (key >= t_lo) & (key <= t_hi);
    }
    // packed 12-bit fields: 0..3 = this thread's quads u, 4 = its tail element; element order
    // inside the tile is (field, thread, element).  Warp-level inclusive scans, one barrier to
    // share the 8 warp totals, every thread folds the totals of the warps before it.
    pw |= (unsigned long long)tw << 48;
    pc |= (unsigned long long)tcn << 48;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long iw = pw, ic = pc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long a1 = __shfl_up_sync(0xFFFFFFFFu, iw, o);
      const unsigned long long a2 = __shfl_up_sync(0xFFFFFFFFu, ic, o);
      if (lane >= o) { iw += a1; ic += a2; }
    }
    if (lane == 31) { s_wt[warp] = iw; s_ct[warp] = ic; }
    __syncthreads();
    unsigned long long ew = iw - pw, ec = ic - pc, totw = 0, totc = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
      const unsigned long long a1 = s_wt[w], a2 = s_ct[w];
      if (w < warp) { ew += a1; ec += a2; }
      totw += a1;
      totc += a2;
    }
    __syncthreads();   // s_wt / s_ct are rewritten by the next chunk
    uint32_t baseW[kQuadsPerThread + 1], baseC[kQuadsPerThread + 1];
    uint32_t accW = 0, accC = 0;
#pragma unroll
    for (int u = 0; u <= kQuadsPerThread; ++u) {
      baseW[u] = accW + (uint32_t)((ew >> (12 * u)) & 0xFFF);
      baseC[u] = accC + (uint32_t)((ec >> (12 * u)) & 0xFFF);
      accW += (uint32_t)((totw >> (12 * u)) & 0xFFF);
      accC += (uint32_t)((totc >> (12 * u)) & 0xFFF);
    }
    const unsigned long long off = pref[ti.status_off + j];
    const uint64_t preW = off >> 32, preC = off & 0xFFFFFFFFull;
    uint2* W = wl + ti.list_off;
    uint2* C = cl + ti.list_off;
#pragma unroll
    for (int u = 0; u < kQuadsPerThread; ++u) {
      const uint64_t q = j * kChunkQuads + (uint64_t)u * kThreads + threadIdx.x;
      if (q < n4) {
        uint32_t w = baseW[u], cc = baseC[u];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t key = kb[u][e] & 0x7FFFFFFFu;
          const uint32_t idx = (uint32_t)(4 * q + e);
          if (key > t_hi) {
            const uint64_t pos = preW + w++;
            if (pos < ti.wcap && !ties_only) W[pos] = make_uint2(idx, kb[u][e]);
          } else if (key >= t_lo) {
            const uint64_t pos = preC + cc++;
            if (pos < cap_c) C[pos] = make_uint2(idx, kb[u][e]);
          }
        }
      }
    }
    if (has_tail) {
      const uint32_t key = tkb & 0x7FFFFFFFu;
      const uint32_t idx = (uint32_t)(n4 * 4 + threadIdx.x);
      if (key > t_hi) {
        const uint64_t pos = preW + baseW[kQuadsPerThread];
        if (pos < ti.wcap && !ties_only) W[pos] = make_uint2(idx, tkb);
      } else if (key >= t_lo) {
        const uint64_t pos = preC + baseC[kQuadsPerThread];
        if (pos < cap_c) C[pos] = make_uint2(idx, tkb);
      }
    }
  }
}

// ---------------------------------------------------------------- D: resolve among candidates
__global__ void __launch_bounds__(kSelThreads) k_topk_resolve(const TopkItem* __restrict__ titems,
                                                              TopkState* __restrict__ st, uint2* __restrict__ cl,
                                                              int retry, uint32_t* any_failed,
                                                              uint32_t wide_min = kWideMin) {
  if (retry && *((volatile uint32_t*)any_failed) == 0) return;
  __shared__ uint32_t hist[2048];
  __shared__ uint32_t misc[4];
  __shared__ unsigned long long scan[32];
  __shared__ uint32_t s_ok;
  const TopkItem ti = titems[blockIdx.x];
  TopkState& S = st[blockIdx.x];
  if (S.failed == 2) return;
  if (retry && S.mode != 1) return;
  const uint64_t k = ti.k, W = S.wcount, C = S.ccount;
  if (threadIdx.x == 0) {
    bool ok = (W < k || k == 0) && (W + C >= k) && (retry || S.stage_ovf == 0);
    if (ok && C > ti.ccap) ok = (S.t_lo == S.t_hi) && (k - W) <= ti.ccap;  // exact tie set: prefix suffices
    s_ok = ok;
    if (!ok) { S.mode = 1; S.failed = 1; atomicOr(any_failed, 1u); }   // -> exact radix fallback
  }
  __syncthreads();
  if (!s_ok || k == 0) {
    if (k == 0 && threadIdx.x == 0) { S.threshold = 0; S.count_above = 0; S.need = 0; }
    return;
  }
  const uint32_t need = (uint32_t)(k - W);
  uint2* cand = cl + ti.list_off;
  const uint32_t m = (uint32_t)(C < ti.ccap ? C : ti.ccap);
  uint32_t T, above_c = 0;
  if (!retry && S.t_lo != S.t_hi && m > wide_min) {
    // long candidate list (a huge bucket, or a large k): the multi-CTA radix select and
    // compaction below (k_topk_wide_*) — one CTA would walk millions of entries
    if (threadIdx.x == 0) {
      const uint32_t hi31 = S.t_hi > 0x7FFFFFFFu ? 0x7FFFFFFFu : S.t_hi;
      const uint32_t x = S.t_lo ^ hi31;
      const int known = x ? (__clz(x) - 1) : 31;
      const int lo_bit = 31 - known;
      S.wide = 1u | ((uint32_t)lo_bit << 8);            // bits [lo_bit, 31) shared by every candidate
      S.hist_prefix = known > 0 ? (S.t_lo >> lo_bit) : 0u;
      S.rank_left = need;
      S.wide_above = 0;
    }
    return;
  }
  if (S.t_lo == S.t_hi) {
    // exact tie set: every candidate == T and the list holds the first need ties in index
    // order (k_topk_write), already the compacted selection
    if (threadIdx.x == 0) {
      S.threshold = S.t_lo;
      S.count_above = W;
      S.need = need;
    }
    return;
  } else {
    auto get = [&](uint32_t i) { return cand[i].y & 0x7FFFFFFFu; };
    // every candidate key lies in [t_lo, min(t_hi, 2^31 - 1)]: their common leading bits are known
    const uint32_t hi31 = S.t_hi > 0x7FFFFFFFu ? 0x7FFFFFFFu : S.t_hi;
    const uint32_t x = S.t_lo ^ hi31;
    const int known = x ? (__clz(x) - 1) : 31;
    T = cta_select(get, m, need, &above_c, hist, misc + 2, scan, known, S.t_lo);
  }
  const uint32_t needT = need - above_c;
  // stable in-place compaction of the selected candidates with ONE packed scan per 4096
  // entries: an entry's output position is (#key > T before it) + min(#key == T before it,
  // need_T), so the (gt, tie) prefix pair decides both selection and position
  uint32_t gt_seen = 0, tie_seen = 0;
  for (uint32_t i0 = 0; i0 < m; i0 += blockDim.x * 4) {
    uint2 e[4];
    uint32_t ngt = 0, ntie = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t i = i0 + 4 * threadIdx.x + u;
      e[u] = i < m ? cand[i] : make_uint2(0u, 0xFFFFFFFFu);
      const uint32_t key = e[u].y & 0x7FFFFFFFu;
      ngt += (i < m) && key > T;
      ntie += (i < m) && key == T;
    }
    const unsigned long long v = ((unsigned long long)ngt << 32) | ntie;
    unsigned long long tot;
    const unsigned long long excl = block_incl_scan<kSelThreads>(v, scan, &tot) - v;
    uint32_t gb = gt_seen + (uint32_t)(excl >> 32), tb = tie_seen + (uint32_t)(excl & 0xFFFFFFFFu);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t i = i0 + 4 * threadIdx.x + u;
      if (i >= m) break;
      const uint32_t key = e[u].y & 0x7FFFFFFFu;
      if (key > T) {
        cand[gb + min(tb, needT)] = e[u];   // reads of this round completed before the scan's barriers
        ++gb;
      } else if (key == T) {
        if (tb < needT) cand[gb + tb] = e[u];
        ++tb;
      }
    }
    gt_seen += (uint32_t)(tot >> 32);
    tie_seen += (uint32_t)(tot & 0xFFFFFFFFu);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    S.threshold = T;
    S.count_above = W + above_c;
    S.need = needT;
  }
}

// ---------------------------------------------------------------- D': multi-CTA resolve
// For candidate lists longer than kWideMin: the radix select of the need-th largest candidate
// key runs as (histogram over all CTAs -> one CTA picks the bin) x up to 3 digits, then a
// stable three-kernel compaction (per-chunk (gt, tie) counts -> per-item scan -> positioned
// writes into clist2).  Same selection as the one-CTA resolve: keys > T, then the first need_T
// keys == T in index order.  S.wide = 1 | lo_bit << 8 (bits still to resolve); the running
// prefix / rank / count-above live in hist_prefix, rank_left, wide_above.
constexpr uint32_t kWideChunk = 4096;

__device__ __forceinline__ bool wide_active(const TopkState& S) { return (S.wide & 1u) && S.failed == 0; }

__device__ __forceinline__ uint32_t wide_m(const TopkItem& ti, const TopkState& S) {
  return (uint32_t)(S.ccount < ti.ccap ? S.ccount : ti.ccap);
}

// 1 CTA: work units (kWideChunk candidates) of every wide item, flattened: S.wchunk0 = exclusive
// prefix of the items' unit counts, *total = their sum (every unit is one CTA-iteration below,
// so the work spreads over all CTAs however the candidates split between items)
__global__ void __launch_bounds__(kSelThreads) k_topk_wide_plan(const TopkItem* __restrict__ titems,
                                                                TopkState* __restrict__ st, int nitems,
                                                                uint32_t* total) {
  __shared__ unsigned long long scan[32];
  unsigned long long carry = 0;
  for (int i0 = 0; i0 < nitems; i0 += kSelThreads) {
    const int i = i0 + threadIdx.x;
    unsigned long long v = 0;
    if (i < nitems && wide_active(st[i])) v = (wide_m(titems[i], st[i]) + kWideChunk - 1) / kWideChunk;
    unsigned long long tot;
    const unsigned long long incl = block_incl_scan<kSelThreads>(v, scan, &tot);
    if (i < nitems) st[i].wchunk0 = (uint32_t)(carry + incl - v);
    carry += tot;
  }
  if (threadIdx.x == 0) *total = (uint32_t)carry;
}

// the item owning work unit u: the last item whose first unit is <= u (items without units
// share their successor's prefix, so the last such item is the one with units)
__device__ __forceinline__ int wide_item_of(const TopkState* st, int nitems, uint32_t u) {
  int lo = 0, hi = nitems - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (st[mid].wchunk0 <= u) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(256) k_topk_wide_hist(const TopkItem* __restrict__ titems,
                                                        const TopkState* __restrict__ st, int nitems,
                                                        const uint2* __restrict__ cl, uint32_t* __restrict__ ghist,
                                                        const uint32_t* total) {
  __shared__ uint32_t hist[2048];
  const uint32_t nu = *total;
  for (uint32_t u = blockIdx.x; u < nu; u += gridDim.x) {
    const int i = wide_item_of(st, nitems, u);
    const TopkState& S = st[i];
    const int lo_bit = (int)(S.wide >> 8);
    if (lo_bit <= 0) continue;
    const int bits = lo_bit < 11 ? lo_bit : 11, shift = lo_bit - bits, hs = lo_bit, nb = 1 << bits;
    const uint32_t prefix = S.hist_prefix;
    const TopkItem& ti = titems[i];
    const uint32_t m = wide_m(ti, S), c = u - S.wchunk0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    const uint2* cand = cl + ti.list_off;
    const uint32_t lim = min(m, (c + 1) * kWideChunk);
#pragma unroll 4
    for (uint32_t x = c * kWideChunk + threadIdx.x; x < lim; x += blockDim.x) {
      const uint32_t key = cand[x].y & 0x7FFFFFFFu;
      hist_add(hist, hs >= 31 || (key >> hs) == prefix, (key >> shift) & (nb - 1));
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += blockDim.x)
      if (hist[b]) atomicAdd(&ghist[(size_t)i * 2048 + b], hist[b]);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kSelThreads) k_topk_wide_pick(TopkState* __restrict__ st, uint32_t* ghist) {
  __shared__ uint32_t hist[2048];
  __shared__ uint32_t misc[4];
  __shared__ unsigned long long scan[32];
  TopkState& S = st[blockIdx.x];
  if (!wide_active(S)) return;
  const int lo_bit = (int)(S.wide >> 8);
  if (lo_bit <= 0) return;
  const int bits = lo_bit < 11 ? lo_bit : 11, shift = lo_bit - bits, nb = 1 << bits;
  uint32_t* gh = ghist + (size_t)blockIdx.x * 2048;
  for (int b = threadIdx.x; b < 2048; b += blockDim.x) { hist[b] = b < nb ? gh[b] : 0; gh[b] = 0; }
  __syncthreads();
  const uint32_t left = (uint32_t)S.rank_left;
  find_bin(hist, nb, left, &misc[0], &misc[1], scan);
  if (threadIdx.x == 0) {
    S.hist_prefix = (S.hist_prefix << bits) | misc[0];
    S.wide_above += misc[1];
    S.rank_left = left - misc[1];
    S.wide = 1u | ((uint32_t)shift << 8);
  }
}

// per work unit (item, chunk of kWideChunk candidates): (#key > T) << 32 | #key == T
__global__ void __launch_bounds__(256) k_topk_wide_count(const TopkItem* __restrict__ titems,
                                                         const TopkState* __restrict__ st, int nitems,
                                                         const uint2* __restrict__ cl,
                                                         unsigned long long* __restrict__ counts,
                                                         const uint32_t* total) {
  __shared__ unsigned long long s_w[8];
  const uint32_t nu = *total;
  for (uint32_t u = blockIdx.x; u < nu; u += gridDim.x) {
    const int i = wide_item_of(st, nitems, u);
    const TopkState& S = st[i];
    const TopkItem& ti = titems[i];
    const uint32_t T = S.hist_prefix, m = wide_m(ti, S), c = u - S.wchunk0;
    const uint2* cand = cl + ti.list_off;
    unsigned long long v = 0;
    const uint32_t lim = min(m, (c + 1) * kWideChunk);
#pragma unroll 4
    for (uint32_t x = c * kWideChunk + threadIdx.x; x < lim; x += blockDim.x) {
      const uint32_t key = cand[x].y & 0x7FFFFFFFu;
      v += ((unsigned long long)(key > T) << 32) | (unsigned long long)(key == T);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t = 0;
      for (int w = 0; w < 8; ++w) t += s_w[w];
      counts[ti.status_off + c] = t;
    }
    __syncthreads();
  }
}

// 1 CTA per item: exclusive scan of the chunk counts (in place into pref) and the final stats
__global__ void __launch_bounds__(kSelThreads) k_topk_wide_scan(const TopkItem* __restrict__ titems,
                                                                TopkState* __restrict__ st,
                                                                const unsigned long long* __restrict__ counts,
                                                                unsigned long long* __restrict__ pref) {
  __shared__ unsigned long long scan[32];
  const TopkItem ti = titems[blockIdx.x];
  TopkState& S = st[blockIdx.x];
  if (!wide_active(S)) return;
  const uint32_t nch = (wide_m(ti, S) + kWideChunk - 1) / kWideChunk;
  unsigned long long carry = 0;
  for (uint32_t j0 = 0; j0 < nch; j0 += kSelThreads) {
    const uint32_t j = j0 + threadIdx.x;
    const unsigned long long v = j < nch ? counts[ti.status_off + j] : 0ull;
    unsigned long long tot;
    const unsigned long long incl = block_incl_scan<kSelThreads>(v, scan, &tot);
    if (j < nch) pref[ti.status_off + j] = carry + incl - v;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    const uint64_t W = S.wcount;
    S.threshold = S.hist_prefix;
    S.count_above = W + S.wide_above;
    S.need = S.rank_left;
  }
}

// per work unit: stable positioned write of the selected candidates into clist2
__global__ void __launch_bounds__(256) k_topk_wide_write(const TopkItem* __restrict__ titems,
                                                         const TopkState* __restrict__ st, int nitems,
                                                         const uint2* __restrict__ cl, uint2* __restrict__ cl2,
                                                         const unsigned long long* __restrict__ pref,
                                                         const uint32_t* total) {
  __shared__ unsigned long long scan[32];
  const uint32_t nu = *total;
  for (uint32_t u = blockIdx.x; u < nu; u += gridDim.x) {
    const int i = wide_item_of(st, nitems, u);
    const TopkState& S = st[i];
    const TopkItem& ti = titems[i];
    const uint32_t T = S.hist_prefix, needT = (uint32_t)S.rank_left, m = wide_m(ti, S), c = u - S.wchunk0;
    const uint2* cand = cl + ti.list_off;
    uint2* outl = cl2 + ti.list_off;
    const unsigned long long pc = pref[ti.status_off + c];
    uint32_t gt_seen = (uint32_t)(pc >> 32), tie_seen = (uint32_t)(pc & 0xFFFFFFFFull);
    const uint32_t lim = min(m, (c + 1) * kWideChunk);
    // 4 entries per thread per round: the round's (gt, tie) prefix gives every entry's position
    for (uint32_t x0 = c * kWideChunk; x0 < lim; x0 += 4 * blockDim.x) {
      uint2 e[4];
      uint32_t ngt = 0, ntie = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t x = x0 + 4 * threadIdx.x + q;
        e[q] = x < lim ? cand[x] : make_uint2(0u, 0u);
        const uint32_t key = e[q].y & 0x7FFFFFFFu;
        ngt += (x < lim) && key > T;
        ntie += (x < lim) && key == T;
      }
      const unsigned long long v = ((unsigned long long)ngt << 32) | ntie;
      unsigned long long tot;
      const unsigned long long excl = block_incl_scan<256>(v, scan, &tot) - v;
      uint32_t gb = gt_seen + (uint32_t)(excl >> 32), tb = tie_seen + (uint32_t)(excl & 0xFFFFFFFFu);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t x = x0 + 4 * threadIdx.x + q;
        if (x >= lim) break;
        const uint32_t key = e[q].y & 0x7FFFFFFFu;
        if (key > T) {
          outl[gb + min(tb, needT)] = e[q];
          ++gb;
        } else if (key == T) {
          if (tb < needT) outl[gb + tb] = e[q];
          ++tb;
        }
      }
      gt_seen += (uint32_t)(tot >> 32);
      tie_seen += (uint32_t)(tot & 0xFFFFFFFFull);
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------- fallback: full radix histograms
template <bool VEC>
__global__ void __launch_bounds__(kThreads) k_topk_hist(const Item* __restrict__ aitems,
                                                        const TopkItem* __restrict__ titems,
                                                        const TopkState* __restrict__ st, int nitems, uint64_t chunks,
                                                        const float* __restrict__ pbase, bool p_in_r,
                                                        const float* __restrict__ gbase, uint32_t* __restrict__ ghist,
                                                        int d, const uint32_t* any_failed) {
  if (*((volatile const uint32_t*)any_failed) == 0) return;
  __shared__ uint32_t hist[2048];
  const Digit dg = digit_of(d);
  const int nb = 1 << dg.bits, hs = dg.shift + dg.bits;
  int hint = 0, cur = -1;
  for (int b = threadIdx.x; b < 2048; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  for (uint64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    const int i = find_item(aitems, nitems, c, hint);
    hint = i;
    if (st[i].failed != 1) continue;
    if (i != cur) {
      if (cur >= 0) {
        __syncthreads();
        for (int b = threadIdx.x; b < nb; b += blockDim.x)
          if (hist[b]) { atomicAdd(&ghist[(size_t)cur * 2048 + b], hist[b]); hist[b] = 0; }
        __syncthreads();
      }
      cur = i;
    }
    const Item it = aitems[i];
    const uint32_t prefix = st[i].t_lo;  // fallback keeps the running prefix in t_lo
    const uint64_t j = c - it.chunk0;
    const float* p = p_in_r ? pbase + it.r_off : gbase + it.g_off;
    for (int u = 0; u < 16; ++u) {
      const uint64_t e = j * kChunkElems + (uint64_t)u * kThreads + threadIdx.x;
      bool act = false;
      uint32_t bin = 0;
      if (e < it.n) {
        const uint32_t key = __float_as_uint(p[e]) & 0x7FFFFFFFu;
        act = (hs >= 31) || ((key >> hs) == prefix);
        bin = (key >> dg.shift) & (nb - 1);
      }
      hist_add(hist, act, bin);
    }
  }
  __syncthreads();
  if (cur >= 0)
    for (int b = threadIdx.x; b < nb; b += blockDim.x)
      if (hist[b]) atomicAdd(&ghist[(size_t)cur * 2048 + b], hist[b]);
}

__global__ void __launch_bounds__(kSelThreads) k_topk_hist_select(const TopkItem* __restrict__ titems,
                                                                  TopkState* __restrict__ st, uint32_t* ghist, int d,
                                                                  const uint32_t* any_failed) {
  if (*((volatile const uint32_t*)any_failed) == 0) return;
  __shared__ uint32_t hist[2048];
  __shared__ uint32_t misc[4];
  __shared__ unsigned long long scan[32];
  const TopkItem ti = titems[blockIdx.x];
  TopkState& S = st[blockIdx.x];
  if (S.failed != 1) return;
  const Digit dg = digit_of(d);
  const int nb = 1 << dg.bits;
  uint32_t* gh = ghist + (size_t)blockIdx.x * 2048;
  for (int b = threadIdx.x; b < 2048; b += blockDim.x) { hist[b] = b < nb ? gh[b] : 0; gh[b] = 0; }
  __syncthreads();
  const uint32_t left = d == 0 ? (uint32_t)ti.k : (uint32_t)S.rank_left;
  find_bin(hist, nb, left, &misc[0], &misc[1], scan);
  if (threadIdx.x == 0) {
    const uint32_t prefix = d == 0 ? 0u : S.t_lo;
    const uint32_t np = (prefix << dg.bits) | misc[0];
    const uint64_t above = (d == 0 ? 0ull : S.count_above) + misc[1];
    S.rank_left = left - misc[1];
    S.count_above = above;
    S.t_lo = np;
    if (d == 2) {  // exact T: rerun classify/resolve in exact mode
      S.t_hi = np;
      S.path = 1;
    }
  }
  if (d == 2) {
    __syncthreads();
    if (threadIdx.x == 0) S.failed = 0;   // mode stays 1: count / scan / write / resolve rerun
  }
}

// ---------------------------------------------------------------- F: merge -> payload + residual
__device__ __forceinline__ uint64_t merge_split(const uint2* A, uint64_t na, const uint2* B, uint64_t nb_, uint64_t d) {
  // number of A elements among the first d outputs of merge(A, B) (indices are distinct)
  uint64_t lo = d > nb_ ? d - nb_ : 0, hi = d < na ? d : na;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (A[mid].x < B[d - 1 - mid].x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Merge-path split points of every merge tile, computed by one thread each (all the
// latency-bound binary searches in flight at once instead of one per merge CTA).
__global__ void k_topk_splits(const TopkItem* __restrict__ titems, const TopkState* __restrict__ st, int nitems,
                              uint64_t tbase, uint64_t ntiles, const uint2* __restrict__ wl,
                              const uint2* __restrict__ cl, const uint2* __restrict__ cl2,
                              uint64_t* __restrict__ splits) {
  const uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= 2 * ntiles) return;
  const uint64_t t = tbase + x / 2;
  int lo = 0, hi = nitems - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (titems[mid].mt0 <= t) lo = mid; else hi = mid - 1;
  }
  const TopkItem& ti = titems[lo];
  const TopkState& S = st[lo];
  if (S.failed == 2 || ti.k == 0) return;
  const uint64_t k = ti.k, W = S.wcount, Ns = k - W;
  const uint64_t d0 = (t - ti.mt0) * kMergeTile;
  const uint64_t d = (x & 1) ? (d0 + kMergeTile < k ? d0 + kMergeTile : k) : d0;
  splits[x] = merge_split(wl + ti.list_off, W, (wide_active(S) ? cl2 : cl) + ti.list_off, Ns, d);
}

// Merge of one 2048-output tile (ModernGPU-style): the tile's ranges of the two ascending lists
// are staged in shared memory; each of the 256 threads finds its 8-output diagonal on the merge
// path (one binary search per thread, not per output) and merges its 8 outputs serially into a
// shared output buffer; the tile is then written with coalesced stores — index section,
// value section (f32 / RNE binary16 / int8 with the bucket scale), and the residual
// r = p - D(v) at the selected positions (ascending addresses within the tile).
template <bool EF>
__global__ void __launch_bounds__(kMergeThreads) k_topk_merge(const TopkItem* __restrict__ titems,
                                                           const TopkState* __restrict__ st, int nitems, uint64_t tbase,
                                                           const uint2* __restrict__ wl, const uint2* __restrict__ cl,
                                                           const uint2* __restrict__ cl2,
                                                           Dests dst, float* __restrict__ rbase, uint32_t* flags,
                                                           const uint64_t* __restrict__ splits) {
  __shared__ uint2 sab[kMergeTile], so[kMergeTile];   // sab: the A range, then the B range (na + nb = nout)
  __shared__ uint64_t s_split[2];
  const uint64_t t = tbase + blockIdx.x;
  int i = 0;
  {
    int lo = 0, hi = nitems - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (titems[mid].mt0 <= t) lo = mid; else hi = mid - 1;
    }
    i = lo;
  }
  const TopkItem ti = titems[i];
  const TopkState& S = st[i];
  if (S.failed == 2) return;
  const uint64_t so_off = ti.slot_off;
  if (ti.k == 0) {
    if (threadIdx.x == 0) {
      put_preamble(dst, so_off, M_TOPK, 0u, 1.0f, ti.value_type);
      if (dst.n > 1) __threadfence_system();
    }
    return;
  }
  const uint64_t k = ti.k;
  const uint64_t d0 = (t - ti.mt0) * kMergeTile, d1 = d0 + kMergeTile < k ? d0 + kMergeTile : k;
  const uint2* A = wl + ti.list_off;
  const uint2* B = (wide_active(S) ? cl2 : cl) + ti.list_off;
  if (threadIdx.x < 2) s_split[threadIdx.x] = splits[2 * blockIdx.x + threadIdx.x];
  __syncthreads();
  const uint64_t a0 = s_split[0], a1 = s_split[1], b0 = d0 - a0, b1 = d1 - a1;
  const uint32_t na = (uint32_t)(a1 - a0), nbb = (uint32_t)(b1 - b0), nout = (uint32_t)(d1 - d0);
  uint2* sa = sab;
  uint2* sb = sab + na;
  for (uint32_t x = threadIdx.x; x < na; x += kMergeThreads) sa[x] = A[a0 + x];
  for (uint32_t x = threadIdx.x; x < nbb; x += kMergeThreads) sb[x] = B[b0 + x];
  __syncthreads();
  {
    const uint32_t diag = threadIdx.x * kMergeVT;
    if (diag < nout) {
      // number of A entries among the first `diag` outputs of this tile (indices are distinct)
      uint32_t lo = diag > nbb ? diag - nbb : 0, hi = diag < na ? diag : na;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (sa[mid].x < sb[diag - 1 - mid].x) lo = mid + 1;
        else hi = mid;
      }
      uint32_t ia = lo, ib = diag - lo;
#pragma unroll
      for (int v = 0; v < kMergeVT; ++v) {
        if (diag + v < nout) {
          const bool takeA = ib >= nbb || (ia < na && sa[ia].x < sb[ib].x);
          so[diag + v] = takeA ? sa[ia] : sb[ib];
          ia += takeA;
          ib += !takeA;
        }
      }
    }
  }
  __syncthreads();
  const int vt = (int)ti.value_type;
  const float s = S.scale;
  const float sinv = int8_inv(s);
  if (d0 == 0 && threadIdx.x == 0) put_preamble(dst, so_off, M_TOPK, (uint32_t)k, s, (uint32_t)vt);
  const uint64_t io = so_off + 16, vo = so_off + 16 + pad16(4 * k);   // idx / value section offsets
  float* r = rbase + ti.r_off;
  bool ovf = false;
  for (uint32_t x = threadIdx.x; x < nout; x += kMergeThreads) {
    const uint2 e = so[x];
    const uint64_t o = d0 + x;
    const float pv = __uint_as_float(e.y);
    put(dst, io + 4 * o, e.x);
    float dv;
    if (vt == V_F32) {
      put(dst, vo + 4 * o, pv);
      dv = pv;
    } else if (vt == V_F16) {
      __half h = __float2half_rn(pv);
      const uint16_t hb = __half_as_ushort(h);
      ovf |= (hb & 0x7FFFu) == 0x7C00u;
      put(dst, vo + 2 * o, hb);
      dv = __half2float(h);
    } else {
      const int q = int8_qi(pv, s, sinv);
      put(dst, vo + o, (uint8_t)(q & 0xFF));
      dv = __fmul_rn((float)q, s);
    }
    if constexpr (EF) r[e.x] = __fsub_rn(pv, dv);
  }
  // zero the padding of the two sections (the tile that ends the item)
  if (d1 == k) {
    const uint64_t ib = 4 * k, ipad = pad16(ib), vb = (vt == V_F32 ? 4 : (vt == V_F16 ? 2 : 1)) * k, vpad = pad16(vb);
    for (uint64_t z = ib + threadIdx.x; z < ipad; z += blockDim.x) put(dst, io + z, (uint8_t)0);
    for (uint64_t z = vb + threadIdx.x; z < vpad; z += blockDim.x) put(dst, vo + z, (uint8_t)0);
  }
  if (__any_sync(0xFFFFFFFFu, ovf) && (threadIdx.x & 31) == 0) atomicOr(flags, kFlagOverflow);
  if (dst.n > 1) __threadfence_system();   // pushed payload visible system-wide before the flag
}

// ---------------------------------------------------------------- sparse reduce
template <class F>
__device__ __forceinline__ int find_by(const RItem* items, int nitems, uint64_t g, F field) {
  int lo = 0, hi = nitems - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (field(items[mid]) <= g) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <int P>
__device__ __forceinline__ float div_p_sparse(float x) {
  if constexpr ((P & (P - 1)) == 0) return __fmul_rn(x, 1.0f / (float)P);
  else return __fdiv_rn(x, (float)P);
}

__device__ __forceinline__ float topk_decode(const uint8_t* val, uint64_t e, int vt, float s) {
  if (vt == V_F32) return reinterpret_cast<const float*>(val)[e];
  if (vt == V_F16) return __half2float(reinterpret_cast<const __half*>(val)[e]);
  return __fmul_rn((float)(int8_t)val[e], s);
}

// Sparse average by output tiles (R16: out = fl(tree_sum(D_0..D_{P-1}) / P), +0.0 where a
// cluster did not select the index).  Persistent WARPS own contiguous ranges of 512-element
// output sub-tiles (4 per kRedTile tile).  Per sub-tile, the sub-tile's entries of every
// cluster are a contiguous run of its ascending index list: a running cursor per cluster (one
// binary search per warp per bucket, then it only advances).  Each lane loads U entries per
// cluster per round — index and value together (the value's position is the entry's), all P
// clusters in flight at once — and drops the in-range ones into the warp's zero-filled
// shared-memory tile [P][512]; then every output element is written once (float4 when
// aligned, 512 B per warp store).  No memset pass, no per-entry search, no CTA barrier.
constexpr int kDenThreads = 256, kDenSub = 512;

template <int P, int U, bool VEC>
__global__ void __launch_bounds__(kDenThreads) k_topk_densify(const RItem* __restrict__ items, int nitems,
                                                              uint64_t tiles, Dests src, float* __restrict__ obase,
                                                              int vt) {
  extern __shared__ __align__(16) float s_v[];   // per warp: [P][kDenSub]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* sw = s_v + (size_t)warp * P * kDenSub;
  const uint64_t nsub = tiles * (kRedTile / kDenSub);
  const uint64_t nw = (uint64_t)gridDim.x * (kDenThreads / 32), gw = (uint64_t)blockIdx.x * (kDenThreads / 32) + warp;
  const uint64_t per = (nsub + nw - 1) / nw;
  const uint64_t sa = gw * per, sb = min(nsub, sa + per);
  int i = -1;
  RItem it{};
  uint64_t it_end = 0;   // first sub-tile after the current item
  uint32_t cur[P];
  const uint8_t* sl[P];
  float scale[P];
  for (uint64_t q = sa; q < sb; ++q) {
    const uint64_t t = q / (kRedTile / kDenSub);
    if (i < 0 || q >= it_end) {
      i = find_by(items, nitems, t, [](const RItem& r) { return r.t0; });
      it = items[i];
      it_end = (it.t0 + (it.n + kRedTile - 1) / kRedTile) * (kRedTile / kDenSub);
      const uint32_t x0 = (uint32_t)((q - it.t0 * (kRedTile / kDenSub)) * kDenSub);
#pragma unroll
      for (int c = 0; c < P; ++c) {
        sl[c] = src.p[c] + it.slot_off + (uint64_t)c * it.pb;
        scale[c] = vt == V_I8 ? *reinterpret_cast<const float*>(sl[c] + 8) : 1.0f;
        const uint32_t* idx = reinterpret_cast<const uint32_t*>(sl[c] + 16);
        uint32_t lo = 0, hi = (uint32_t)it.k;   // lower_bound(x0), warp-uniform
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (idx[mid] < x0) lo = mid + 1; else hi = mid;
        }
        cur[c] = lo;
      }
    }
    const uint32_t e0 = (uint32_t)((q - it.t0 * (kRedTile / kDenSub)) * kDenSub);
    if (e0 >= it.n) continue;   // past the end of the item's last (partial) tile
    const uint32_t e1 = (uint32_t)min(it.n, (uint64_t)e0 + (uint64_t)kDenSub);
#pragma unroll
    for (int v = 0; v < P * kDenSub / 128; ++v)
      reinterpret_cast<float4*>(sw)[v * 32 + lane] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    __syncwarp();
    const uint64_t voff = 16 + pad16(4 * it.k);
    // round 1: U entries per lane of every cluster in flight at once (U sized from the density)
    uint32_t more_mask = 0;
    {
      uint32_t x[P][U];
      float val[P][U];
#pragma unroll
      for (int c = 0; c < P; ++c) {
        const uint32_t* idx = reinterpret_cast<const uint32_t*>(sl[c] + 16);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t e = cur[c] + (uint32_t)(u * 32 + lane);
          x[c][u] = 0xFFFFFFFFu;
          val[c][u] = 0.0f;
          if (e < it.k) {
            x[c][u] = idx[e];
            val[c][u] = topk_decode(sl[c] + voff, e, vt, scale[c]);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < P; ++c) {
        uint32_t nin = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool in = x[c][u] < e1;   // >= e0 holds: the cursor is the run's start
          if (in) sw[c * kDenSub + (x[c][u] - e0)] = val[c][u];
          nin += __popc(__ballot_sync(0xFFFFFFFFu, in));
        }
        cur[c] += nin;
        if (nin == 32u * U) more_mask |= 1u << c;
      }
    }
    // long runs (dense stretches, e.g. a tie run of zeros): 256 entries per round per cluster
#pragma unroll
    for (int c = 0; c < P; ++c) {
      if (!(more_mask >> c & 1u)) continue;
      const uint32_t* idx = reinterpret_cast<const uint32_t*>(sl[c] + 16);
      while (true) {
        uint32_t x[8];
        float val[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t e = cur[c] + (uint32_t)(u * 32 + lane);
          x[u] = 0xFFFFFFFFu;
          val[u] = 0.0f;
          if (e < it.k) {
            x[u] = idx[e];
            val[u] = topk_decode(sl[c] + voff, e, vt, scale[c]);
          }
        }
        uint32_t nin = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const bool in = x[u] < e1;
          if (in) sw[c * kDenSub + (x[u] - e0)] = val[u];
          nin += __popc(__ballot_sync(0xFFFFFFFFu, in));
        }
        cur[c] += nin;
        if (nin < 256u) break;
      }
    }
    __syncwarp();
    float* out = obase + it.out_off + e0;
    if (VEC && e1 - e0 == (uint32_t)kDenSub) {
#pragma unroll
      for (int v = 0; v < kDenSub / 128; ++v) {
        const int j = v * 32 + lane;
        float a[P], b[P], d[P], e[P];
#pragma unroll
        for (int c = 0; c < P; ++c) {
          const float4 w = reinterpret_cast<const float4*>(sw + c * kDenSub)[j];
          a[c] = w.x; b[c] = w.y; d[c] = w.z; e[c] = w.w;
        }
        st4(out + 4 * j, make_float4(div_p_sparse<P>(tree_sum<0, P>(a)), div_p_sparse<P>(tree_sum<0, P>(b)),
                                     div_p_sparse<P>(tree_sum<0, P>(d)), div_p_sparse<P>(tree_sum<0, P>(e))));
      }
    } else {
      for (uint32_t j = lane; j < e1 - e0; j += 32) {
        float v[P];
#pragma unroll
        for (int c = 0; c < P; ++c) v[c] = sw[c * kDenSub + j];
        out[j] = div_p_sparse<P>(tree_sum<0, P>(v));
      }
    }
    __syncwarp();   // the tile buffer is zeroed for the next sub-tile
  }
}

// Sparse variant (a sub-tile holds well under 32 entries per cluster, e.g. rho = 1 %): every
// lane keeps ONE entry of each cluster resident in registers — a 32-entry window per cluster,
// reloaded only when a sub-tile consumes all of it — so consecutive sub-tiles of a warp need no
// global load at all on their critical path (the window covers ~6 sub-tiles at 1 % density):
// zero the shared tile, drop the window's in-range entries in, store.  Same results as
// k_topk_densify (same tree order, +0.0 fill).
template <int P, bool VEC>
__global__ void __launch_bounds__(kDenThreads) k_topk_densify_w(const RItem* __restrict__ items, int nitems,
                                                                uint64_t tiles, Dests src, float* __restrict__ obase,
                                                                int vt) {
  extern __shared__ __align__(16) float s_v[];   // per warp: [P][kDenSub]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* sw = s_v + (size_t)warp * P * kDenSub;
  const uint64_t nsub = tiles * (kRedTile / kDenSub);
  const uint64_t nw = (uint64_t)gridDim.x * (kDenThreads / 32), gw = (uint64_t)blockIdx.x * (kDenThreads / 32) + warp;
  const uint64_t per = (nsub + nw - 1) / nw;
  const uint64_t sa = gw * per, sb = min(nsub, sa + per);
  int i = -1;
  RItem it{};
  uint64_t it_end = 0;
  uint32_t wb[P] = {};   // window base entry of each cluster
  uint32_t xw[P];        // this lane's entry (wb + lane): index, 0xFFFFFFFF past the end
  float vw[P];
  const uint8_t* sl[P];
  float scale[P];
  uint64_t voff = 0;
  auto load_window = [&](int c) {
    const uint32_t e = wb[c] + (uint32_t)lane;
    xw[c] = 0xFFFFFFFFu;
    vw[c] = 0.0f;
    if (e < it.k) {
      xw[c] = reinterpret_cast<const uint32_t*>(sl[c] + 16)[e];
      vw[c] = topk_decode(sl[c] + voff, e, vt, scale[c]);
    }
  };
  for (uint64_t q = sa; q < sb; ++q) {
    const uint64_t t = q / (kRedTile / kDenSub);
    if (i < 0 || q >= it_end) {
      i = find_by(items, nitems, t, [](const RItem& r) { return r.t0; });
      it = items[i];
      it_end = (it.t0 + (it.n + kRedTile - 1) / kRedTile) * (kRedTile / kDenSub);
      voff = 16 + pad16(4 * it.k);
      const uint32_t x0 = (uint32_t)((q - it.t0 * (kRedTile / kDenSub)) * kDenSub);
#pragma unroll
      for (int c = 0; c < P; ++c) {
        sl[c] = src.p[c] + it.slot_off + (uint64_t)c * it.pb;
        scale[c] = vt == V_I8 ? *reinterpret_cast<const float*>(sl[c] + 8) : 1.0f;
        const uint32_t* idx = reinterpret_cast<const uint32_t*>(sl[c] + 16);
        uint32_t lo = 0, hi = (uint32_t)it.k;   // lower_bound(x0), warp-uniform
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (idx[mid] < x0) lo = mid + 1; else hi = mid;
        }
        wb[c] = lo;
        load_window(c);
      }
    }
    const uint32_t e0 = (uint32_t)((q - it.t0 * (kRedTile / kDenSub)) * kDenSub);
    if (e0 >= it.n) continue;
    const uint32_t e1 = (uint32_t)min(it.n, (uint64_t)e0 + (uint64_t)kDenSub);
#pragma unroll
    for (int v = 0; v < P * kDenSub / 128; ++v)
      reinterpret_cast<float4*>(sw)[v * 32 + lane] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    __syncwarp();
#pragma unroll
    for (int c = 0; c < P; ++c) {
      while (true) {
        const bool in = xw[c] >= e0 && xw[c] < e1;
        if (in) sw[c * kDenSub + (xw[c] - e0)] = vw[c];
        // window exhausted inside this sub-tile (every lane's entry is < e1): slide by 32
        if (__ballot_sync(0xFFFFFFFFu, xw[c] < e1) != 0xFFFFFFFFu) break;
        wb[c] += 32;
        load_window(c);
      }
    }
    __syncwarp();
    float* out = obase + it.out_off + e0;
    if (VEC && e1 - e0 == (uint32_t)kDenSub) {
#pragma unroll
      for (int v = 0; v < kDenSub / 128; ++v) {
        const int j = v * 32 + lane;
        float a[P], b[P], d[P], e[P];
#pragma unroll
        for (int c = 0; c < P; ++c) {
          const float4 w = reinterpret_cast<const float4*>(sw + c * kDenSub)[j];
          a[c] = w.x; b[c] = w.y; d[c] = w.z; e[c] = w.w;
        }
        st4(out + 4 * j, make_float4(div_p_sparse<P>(tree_sum<0, P>(a)), div_p_sparse<P>(tree_sum<0, P>(b)),
                                     div_p_sparse<P>(tree_sum<0, P>(d)), div_p_sparse<P>(tree_sum<0, P>(e))));
      }
    } else {
      for (uint32_t j = lane; j < e1 - e0; j += 32) {
        float v[P];
#pragma unroll
        for (int c = 0; c < P; ++c) v[c] = sw[c * kDenSub + j];
        out[j] = div_p_sparse<P>(tree_sum<0, P>(v));
      }
    }
    __syncwarp();
  }
}

// Tile-interleaved variant (NEBULA_OPT_TOPK_REDUCE = 0; measured slower: 0.345 vs 0.30 ms at
// BASELINE config 2, the extra start-offset kernel and three CTA barriers per tile cost more
// than the write locality gains).  The contiguous per-warp ranges above leave every warp
// writing its own far-apart region of the output (~4700 concurrent write streams); here CTAs
// walk the 2048-element tiles grid-stride, so the active writes form one contiguous window, as
// in a fill.  A first kernel finds, massively in parallel, where every tile's run starts in
// every cluster's ascending index list (start[sbase + c (tiles + 1) + t], the last = k); the
// CTA then zero-fills a shared [P][2048] tile, scatters the run, tree-sums and stores float4.
__global__ void k_topk_starts(const RItem* __restrict__ items, int nitems, int P, Dests src, uint64_t total,
                              uint32_t* __restrict__ start) {
  const uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= total) return;
  const uint64_t s = items[0].sbase + x;
  const int i = find_by(items, nitems, s, [](const RItem& r) { return r.sbase; });
  const RItem it = items[i];
  const uint64_t nt = (it.n + kRedTile - 1) / kRedTile;
  const uint64_t local = s - it.sbase;
  const int c = (int)(local / (nt + 1));
  const uint64_t tt = local % (nt + 1);
  if (c >= P) return;
  uint32_t v = (uint32_t)it.k;
  if (tt < nt) {
    const uint32_t* idx = reinterpret_cast<const uint32_t*>(src.p[c] + it.slot_off + (uint64_t)c * it.pb + 16);
    const uint32_t x0 = (uint32_t)(tt * kRedTile);
    uint32_t lo = 0, hi = (uint32_t)it.k;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (idx[mid] < x0) lo = mid + 1; else hi = mid;
    }
    v = lo;
  }
  start[s] = v;
}

template <int P, bool VEC>
__global__ void __launch_bounds__(kDenThreads) k_topk_densify_t(const RItem* __restrict__ items, int nitems,
                                                                uint64_t tiles, Dests src,
                                                                const uint32_t* __restrict__ start,
                                                                float* __restrict__ obase, int vt) {
  extern __shared__ __align__(16) float s_t[];   // [P][kRedTile]
  int hint = 0;
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    int i = hint;
    while (i + 1 < nitems && items[i + 1].t0 <= t) ++i;
    hint = i;
    const RItem it = items[i];
    const uint64_t tt = t - it.t0, nt = (it.n + kRedTile - 1) / kRedTile;
    const uint32_t e0 = (uint32_t)(tt * kRedTile);
    const uint32_t e1 = (uint32_t)min(it.n, (uint64_t)e0 + kRedTile);
#pragma unroll
    for (int v = 0; v < P * kRedTile / 4 / kDenThreads; ++v)
      reinterpret_cast<float4*>(s_t)[v * kDenThreads + threadIdx.x] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    __syncthreads();
    const uint64_t voff = 16 + pad16(4 * it.k);
#pragma unroll
    for (int c = 0; c < P; ++c) {
      const uint8_t* sl = src.p[c] + it.slot_off + (uint64_t)c * it.pb;
      const uint32_t* idx = reinterpret_cast<const uint32_t*>(sl + 16);
      const float scale = vt == V_I8 ? *reinterpret_cast<const float*>(sl + 8) : 1.0f;
      const uint64_t sb = it.sbase + (uint64_t)c * (nt + 1) + tt;
      const uint32_t a = start[sb], b = start[sb + 1];
      for (uint32_t e = a + threadIdx.x; e < b; e += kDenThreads)
        s_t[c * kRedTile + (idx[e] - e0)] = topk_decode(sl + voff, e, vt, scale);
    }
    __syncthreads();
    float* out = obase + it.out_off + e0;
    if (VEC && e1 - e0 == (uint32_t)kRedTile) {
#pragma unroll
      for (int v = 0; v < kRedTile / 4 / kDenThreads; ++v) {
        const int j = v * kDenThreads + threadIdx.x;
        float a[P], b[P], d[P], e[P];
#pragma unroll
        for (int c = 0; c < P; ++c) {
          const float4 w = reinterpret_cast<const float4*>(s_t + c * kRedTile)[j];
          a[c] = w.x; b[c] = w.y; d[c] = w.z; e[c] = w.w;
        }
        st4(out + 4 * j, make_float4(div_p_sparse<P>(tree_sum<0, P>(a)), div_p_sparse<P>(tree_sum<0, P>(b)),
                                     div_p_sparse<P>(tree_sum<0, P>(d)), div_p_sparse<P>(tree_sum<0, P>(e))));
      }
    } else {
      for (uint32_t j = threadIdx.x; j < e1 - e0; j += kDenThreads) {
        float v[P];
#pragma unroll
        for (int c = 0; c < P; ++c) v[c] = s_t[c * kRedTile + j];
        out[j] = div_p_sparse<P>(tree_sum<0, P>(v));
      }
    }
    __syncthreads();   // the tile buffer is re-zeroed for the next tile
  }
}

// ---------------------------------------------------------------- launchers

template <bool EF, bool VEC>
static void topk_select_all(const Launch& L, const TopkBuffers& B, int item0, int nitems, uint64_t a_chunks,
                            const Item* aitems, const float* g, float* r, const Dests& slots, uint32_t* flags,
                            int value_type, uint64_t merge_tiles) {
  const TopkItem* ti = B.items + item0;
  TopkState* st = B.state + item0;
  uint32_t* anyf = B.ctrs + 2;
  // the TMA stage kernel for 16-B aligned calls (NEBULA_OPT_TOPK_STAGE = 1, the default)
  const bool tma = VEC && B.stage_tma;
  const void* kst = tma ? (const void*)k_topk_stage<EF, VEC, true> : (const void*)k_topk_stage<EF, VEC, false>;
  const size_t st_smem = tma ? sizeof(StageTile) * kStageNS : 0;
  if (tma) ensure_smem_attr(kst, st_smem);
  const unsigned ga = persistent_grid(L, a_chunks, kst, tma ? kThreads + 32 : kThreads, st_smem);
  // The fallback kernels run every step but exit at once unless a bracket failed (adversarial
  // inputs): one CTA per SM keeps those no-op launches at ~2 us instead of draining a full
  // occupancy grid each (measured 51 us per step for the eight of them at 8 CTAs / SM).
  const unsigned gsm = (unsigned)std::min<uint64_t>(a_chunks ? a_chunks : 1, (uint64_t)L.num_sms);
  const unsigned gp = gsm;
  const unsigned gw = persistent_grid(L, a_chunks, (const void*)k_topk_write<VEC>, kThreads);
  const unsigned gh = gsm;
  const uint64_t sbase = B.host_sample_off[item0];
  const uint64_t scount = B.host_sample_off[item0 + nitems] - sbase;
  {
    Mark mk(L, PH_MEMSET);
    cudaMemsetAsync(st, 0, sizeof(TopkState) * nitems, L.stream);
  }
  {
    Mark mk(L, PH_TOPK_BRACKET);
    k_topk_sample<EF><<<(unsigned)((scount + 255) / 256 ? (scount + 255) / 256 : 1), 256, 0, L.stream>>>(
        aitems, ti, nitems, sbase, scount, g, r, B.sample, B.ctrs);
    k_topk_bracket<<<nitems, kSelThreads, (size_t)B.bracket_smem_keys * 4, L.stream>>>(ti, st, B.sample,
                                                                                      B.bracket_smem_keys, B.ctrs + 4);
  }
  {
    Mark mk(L, PH_TOPK_A);
    if (tma)
      k_topk_stage<EF, VEC, true><<<ga, kThreads + 32, st_smem, L.stream>>>(aitems, ti, st, nitems, a_chunks, g, r,
                                                                           B.status, B.soff, B.stage,
                                                                           B.stage_entries / ga);
    else
      k_topk_stage<EF, VEC, false><<<ga, kThreads, 0, L.stream>>>(aitems, ti, st, nitems, a_chunks, g, r, B.status,
                                                                  B.soff, B.stage, B.stage_entries / ga);
  }
  {
    Mark mk(L, PH_TOPK_CLASSIFY);
    k_topk_scan<<<nitems, kSelThreads, 0, L.stream>>>(ti, st, B.status, B.pref, 0, flags, value_type, anyf);
    k_topk_move<<<(unsigned)((a_chunks * 32 + 255) / 256), 256, 0, L.stream>>>(aitems, ti, st, nitems, a_chunks,
                                                                             B.status, B.pref, B.soff, B.stage,
                                                                             B.wlist, B.clist);
    // exact-tie buckets: their first need_T ties in index order, at the scanned offsets
    k_topk_write<VEC><<<gw, kThreads, 0, L.stream>>>(aitems, ti, st, nitems, a_chunks, r, EF, g, B.wlist, B.clist,
                                                     B.pref, 2, B.ctrs + 4);
  }
  {
    Mark mk(L, PH_TOPK_RESOLVE);
    // test hook: NEBULA_DEBUG_WIDE_MIN lowers the threshold (more buckets on the multi-CTA path);
    // 32768 / 8192 measured the same speed at config 2 as the default
    static const uint32_t wide_min = [] { const char* e = getenv("NEBULA_DEBUG_WIDE_MIN"); return e ? (uint32_t)atoi(e) : kWideMin; }();
    k_topk_resolve<<<nitems, kSelThreads, 0, L.stream>>>(ti, st, B.clist, 0, anyf, wide_min);
    // long candidate lists: multi-CTA radix select + compaction (no-ops for the others; not
    // launched at all when no item's candidate capacity exceeds kWideMin, e.g. rho = 1 %)
    bool may_wide = false;
    for (int x = 0; x < nitems; ++x) may_wide |= B.host_ccap[item0 + x] > wide_min;
    if (B.wide_wait) cudaStreamWaitEvent(L.stream, B.wide_wait, 0);
    if (may_wide) {
    const unsigned gwide = (unsigned)L.num_sms * 8;
    uint32_t* wtotal = B.ctrs + 3;
    k_topk_wide_plan<<<1, kSelThreads, 0, L.stream>>>(ti, st, nitems, wtotal);
    for (int d = 0; d < 3; ++d) {
      k_topk_wide_hist<<<gwide, 256, 0, L.stream>>>(ti, st, nitems, B.clist, B.hist + (size_t)item0 * 2048, wtotal);
      k_topk_wide_pick<<<nitems, kSelThreads, 0, L.stream>>>(st, B.hist + (size_t)item0 * 2048);
    }
    k_topk_wide_count<<<gwide, 256, 0, L.stream>>>(ti, st, nitems, B.clist, B.status, wtotal);
    k_topk_wide_scan<<<nitems, kSelThreads, 0, L.stream>>>(ti, st, B.status, B.pref);
    k_topk_wide_write<<<gwide, 256, 0, L.stream>>>(ti, st, nitems, B.clist, B.clist2, B.pref, wtotal);
    *L.launches += 10;
    }
    if (B.wide_rec) cudaEventRecord(B.wide_rec, L.stream);
  }
  {
    // fallback for items whose bracket failed (every kernel exits at once otherwise)
    Mark mk(L, PH_TOPK_FALLBACK);
    for (int d = 0; d < 3; ++d) {
      k_topk_hist<VEC><<<gh, kThreads, 0, L.stream>>>(aitems, ti, st, nitems, a_chunks, r, EF, g,
                                                      B.hist + (size_t)item0 * 2048, d, anyf);
      k_topk_hist_select<<<nitems, kSelThreads, 0, L.stream>>>(ti, st, B.hist + (size_t)item0 * 2048, d, anyf);
    }
    k_topk_pass<true, EF, VEC><<<gp, kThreads, 0, L.stream>>>(aitems, ti, st, nitems, a_chunks, g, r, B.status, anyf);
    k_topk_scan<<<nitems, kSelThreads, 0, L.stream>>>(ti, st, B.status, B.pref, 1, flags, value_type, anyf);
    k_topk_write<VEC><<<gsm, kThreads, 0, L.stream>>>(aitems, ti, st, nitems, a_chunks, r, EF, g, B.wlist, B.clist,
                                                      B.pref, 1, anyf);
    k_topk_resolve<<<nitems, kSelThreads, 0, L.stream>>>(ti, st, B.clist, 1, anyf);
  }
  Mark mk(L, PH_TOPK_MERGE);
  const uint64_t tbase = B.host_mt0[item0];
  k_topk_splits<<<(unsigned)((2 * merge_tiles + 255) / 256), 256, 0, L.stream>>>(ti, st, nitems, tbase, merge_tiles,
                                                                                B.wlist, B.clist, B.clist2, B.splits);
  k_topk_merge<EF><<<(unsigned)merge_tiles, kMergeThreads, 0, L.stream>>>(ti, st, nitems, tbase, B.wlist, B.clist, B.clist2, slots,
                                                                      r, flags, B.splits);
  *L.launches += 19;
}

static void touch_t(const void* f) {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, f);
}
template <int P>
static void touch_densify() {
  touch_t((const void*)k_topk_densify<P, 1, true>); touch_t((const void*)k_topk_densify<P, 1, false>);
  touch_t((const void*)k_topk_densify<P, 2, true>); touch_t((const void*)k_topk_densify<P, 2, false>);
  touch_t((const void*)k_topk_densify<P, 4, true>); touch_t((const void*)k_topk_densify<P, 4, false>);
  touch_t((const void*)k_topk_densify_w<P, true>); touch_t((const void*)k_topk_densify_w<P, false>);
  touch_t((const void*)k_topk_densify_t<P, true>); touch_t((const void*)k_topk_densify_t<P, false>);
}
void preload_topk() {
  touch_t((const void*)k_topk_bracket);
  touch_t((const void*)k_topk_sample<true>); touch_t((const void*)k_topk_sample<false>);
  for (const void* f : {(const void*)k_topk_pass<true, true, true>, (const void*)k_topk_pass<true, true, false>,
                        (const void*)k_topk_pass<true, false, true>, (const void*)k_topk_pass<true, false, false>,
                        (const void*)k_topk_pass<false, true, true>, (const void*)k_topk_pass<false, true, false>,
                        (const void*)k_topk_pass<false, false, true>, (const void*)k_topk_pass<false, false, false>})
    touch_t(f);
  touch_t((const void*)k_topk_stage<true, true, false>); touch_t((const void*)k_topk_stage<true, false, false>);
  touch_t((const void*)k_topk_stage<false, true, false>); touch_t((const void*)k_topk_stage<false, false, false>);
  touch_t((const void*)k_topk_stage<true, true, true>); touch_t((const void*)k_topk_stage<false, true, true>);
  touch_t((const void*)k_topk_move); touch_t((const void*)k_topk_scan);
  touch_t((const void*)k_topk_wide_hist); touch_t((const void*)k_topk_wide_pick); touch_t((const void*)k_topk_wide_plan);
  touch_t((const void*)k_topk_wide_count); touch_t((const void*)k_topk_wide_scan);
  touch_t((const void*)k_topk_wide_write);
  touch_t((const void*)k_topk_write<true>); touch_t((const void*)k_topk_write<false>);
  touch_t((const void*)k_topk_resolve);
  touch_t((const void*)k_topk_hist<true>); touch_t((const void*)k_topk_hist<false>);
  touch_t((const void*)k_topk_hist_select); touch_t((const void*)k_topk_splits);
  touch_t((const void*)k_topk_merge<true>); touch_t((const void*)k_topk_merge<false>);
  touch_t((const void*)k_topk_starts);
  touch_densify<1>(); touch_densify<2>(); touch_densify<3>(); touch_densify<4>();
  touch_densify<5>(); touch_densify<6>(); touch_densify<7>(); touch_densify<8>();
}

void topk_prepare_bracket(uint32_t keys) { ensure_smem_attr((const void*)k_topk_bracket, (size_t)keys * 4); }

void launch_topk(const Launch& L, bool ef, bool vec, const TopkBuffers& B, int item0, int nitems, uint64_t a_chunks,
                 const Item* aitems, const float* g, float* r, const Dests& slots, uint32_t* flags, int value_type,
                 uint64_t merge_tiles) {
  if (nitems <= 0) return;
  if (ef && vec) topk_select_all<true, true>(L, B, item0, nitems, a_chunks, aitems, g, r, slots, flags, value_type, merge_tiles);
  else if (ef) topk_select_all<true, false>(L, B, item0, nitems, a_chunks, aitems, g, r, slots, flags, value_type, merge_tiles);
  else if (vec) topk_select_all<false, true>(L, B, item0, nitems, a_chunks, aitems, g, r, slots, flags, value_type, merge_tiles);
  else topk_select_all<false, false>(L, B, item0, nitems, a_chunks, aitems, g, r, slots, flags, value_type, merge_tiles);
}

template <int P, int U>
static void densify_pu(const Launch& L, int vt, bool vec, const RItem* items, int nitems, uint64_t tiles,
                       const Dests& slots, float* out) {
  const size_t smem = (size_t)(kDenThreads / 32) * P * kDenSub * sizeof(float);
  const void* f = vec ? (const void*)k_topk_densify<P, U, true> : (const void*)k_topk_densify<P, U, false>;
  ensure_smem_attr(f, smem);
  const unsigned grid = persistent_grid(L, tiles * (kRedTile / kDenSub) / (kDenThreads / 32) + 1, f, kDenThreads, smem);
  if (vec) k_topk_densify<P, U, true><<<grid, kDenThreads, smem, L.stream>>>(items, nitems, tiles, slots, out, vt);
  else k_topk_densify<P, U, false><<<grid, kDenThreads, smem, L.stream>>>(items, nitems, tiles, slots, out, vt);
}

template <int P>
static void densify_t(const Launch& L, int vt, bool vec, const RItem* items, int nitems, uint64_t tiles,
                      const Dests& slots, const uint32_t* start, float* out) {
  const size_t smem = (size_t)P * kRedTile * sizeof(float);
  const void* f = vec ? (const void*)k_topk_densify_t<P, true> : (const void*)k_topk_densify_t<P, false>;
  ensure_smem_attr(f, smem);
  const unsigned grid = persistent_grid(L, tiles, f, kDenThreads, smem);
  if (vec) k_topk_densify_t<P, true><<<grid, kDenThreads, smem, L.stream>>>(items, nitems, tiles, slots, start, out, vt);
  else k_topk_densify_t<P, false><<<grid, kDenThreads, smem, L.stream>>>(items, nitems, tiles, slots, start, out, vt);
}

template <int P>
static void densify_w(const Launch& L, int vt, bool vec, const RItem* items, int nitems, uint64_t tiles,
                      const Dests& slots, float* out) {
  const size_t smem = (size_t)(kDenThreads / 32) * P * kDenSub * sizeof(float);
  const void* f = vec ? (const void*)k_topk_densify_w<P, true> : (const void*)k_topk_densify_w<P, false>;
  ensure_smem_attr(f, smem);
  const unsigned grid = persistent_grid(L, tiles * (kRedTile / kDenSub) / (kDenThreads / 32) + 1, f, kDenThreads, smem);
  if (vec) k_topk_densify_w<P, true><<<grid, kDenThreads, smem, L.stream>>>(items, nitems, tiles, slots, out, vt);
  else k_topk_densify_w<P, false><<<grid, kDenThreads, smem, L.stream>>>(items, nitems, tiles, slots, out, vt);
}

// U = entries per lane per round: sized so a typical 512-element sub-tile's run fits one round
template <int P>
static void densify_p(const Launch& L, int vt, bool vec, const RItem* items, int nitems, uint64_t tiles,
                      uint64_t entries, const Dests& slots, float* out) {
  const double per_sub = (double)entries / (double)(tiles * (kRedTile / kDenSub));   // entries per sub-tile
  if (per_sub * 4.0 <= 32.0) densify_w<P>(L, vt, vec, items, nitems, tiles, slots, out);
  else if (per_sub * 1.25 <= 32.0 || P > 4) densify_pu<P, 1>(L, vt, vec, items, nitems, tiles, slots, out);
  else if (per_sub <= 64.0 || P > 2) densify_pu<P, 2>(L, vt, vec, items, nitems, tiles, slots, out);
  else densify_pu<P, 4>(L, vt, vec, items, nitems, tiles, slots, out);
}

void launch_reduce_topk(const Launch& L, int value_type, int P, bool vec, const RItem* items, int nitems,
                        uint64_t entries, uint64_t tiles, const Dests& slots, uint32_t* start, float* out,
                        float* zero_begin, uint64_t zero_count, uint64_t start_count, int variant) {
  (void)zero_begin; (void)zero_count;
  if (!tiles) return;
  Mark mk(L, PH_TOPK_REDUCE);
  if (variant == 0) {   // tile-interleaved
    k_topk_starts<<<(unsigned)((start_count + 255) / 256), 256, 0, L.stream>>>(items, nitems, P, slots, start_count, start);
    switch (P) {
      case 1: densify_t<1>(L, value_type, vec, items, nitems, tiles, slots, start, out); break;
      case 2: densify_t<2>(L, value_type, vec, items, nitems, tiles, slots, start, out); break;
      case 3: densify_t<3>(L, value_type, vec, items, nitems, tiles, slots, start, out); break;
      case 4: densify_t<4>(L, value_type, vec, items, nitems, tiles, slots, start, out); break;
      case 5: densify_t<5>(L, value_type, vec, items, nitems, tiles, slots, start, out); break;
      case 6: densify_t<6>(L, value_type, vec, items, nitems, tiles, slots, start, out); break;
      case 7: densify_t<7>(L, value_type, vec, items, nitems, tiles, slots, start, out); break;
      default: densify_t<8>(L, value_type, vec, items, nitems, tiles, slots, start, out); break;
    }
    *L.launches += 2;
    return;
  }
  switch (P) {
    case 1: densify_p<1>(L, value_type, vec, items, nitems, tiles, entries, slots, out); break;
    case 2: densify_p<2>(L, value_type, vec, items, nitems, tiles, entries, slots, out); break;
    case 3: densify_p<3>(L, value_type, vec, items, nitems, tiles, entries, slots, out); break;
    case 4: densify_p<4>(L, value_type, vec, items, nitems, tiles, entries, slots, out); break;
    case 5: densify_p<5>(L, value_type, vec, items, nitems, tiles, entries, slots, out); break;
    case 6: densify_p<6>(L, value_type, vec, items, nitems, tiles, entries, slots, out); break;
    case 7: densify_p<7>(L, value_type, vec, items, nitems, tiles, entries, slots, out); break;
    default: densify_p<8>(L, value_type, vec, items, nitems, tiles, entries, slots, out); break;
  }
  ++*L.launches;
}

}  // namespace nb
