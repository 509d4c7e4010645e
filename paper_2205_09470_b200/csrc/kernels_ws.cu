// kernels_ws.cu — sm_100a warp-specialised TMA kernels: the single-pass INT8 / FP8 / QSGD
// compressor (k_int8_ws), the fused step (compress + exchange + average in one cooperative
// kernel), the FP16 TMA-ring compressor and the P2P arrival-flag handshake.
// Paper passages: PAPER.md:101 / :418 (INT8 gradient compression), Eq. 5
// (FP16), PAPER.md:76 / :95 (aggregation across clusters).
#include <cuda_fp16.h>

#include <algorithm>
#include <mutex>
#include <set>

#include "kernels.h"
#include "dense_common.cuh"

namespace nb {


// ----------------------------------------------------------------------------- INT8 WS
// Warp-specialised TMA kernel (variant 10, the default for large buckets).  One CTA per SM:
//   warp 0          producer: one lane feeds two TMA (cp.async.bulk) rings —
//                   ring A: g and r tiles of bucket t; ring B: parked-p tiles of bucket t'
//   AW warps  "A":  p = g + r, bucket max, park p in r (L2 evict_last); per bucket they
//                   publish the CTA max (atomicMax) and ARRIVE on the grid-wide done[t]
//   BW warps  "B":  wait until done[t'] == grid (every CTA's max is in), quantise bucket t'
//                   from ring B, write the payload (+ NVLink pushes) and the residual
//   CW warps  "C":  (fused step only, CW > 0) wait until every cluster's payload of bucket b
//                   is complete — this GPU's B phase (grid counter bdone) and every peer's
//                   system-scope arrival flag — then decode the P payloads (peers' over
//                   NVLink in pull mode), tree-sum, divide and write the average of bucket b.
// A runs at most two buckets ahead of B (bounded L2 footprint); B-ring copies of bucket t' are
// issued only after this CTA's A warps parked all of p(t') and fenced it for the async proxy.
// No CTA-wide barrier sits on the streaming path: the grid-wide wait only stalls the B warps,
// while the producer and the A warps keep HBM busy; C drains bucket b while A/B stream b+1.
constexpr int kWsThreads = 1024;
constexpr int kWsTQ = 1024;
constexpr int kWsNA = 3, kWsNB = 4;

struct __align__(128) WsStageA {
  float4 g[kWsTQ];
  float4 r[kWsTQ];
};
struct __align__(128) WsStageB {
  float4 p[kWsTQ];
};

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred P1;\n mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n selp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(n) : "memory");
}

// ----------------------------------------------------------------------------- P2P flags
__device__ __forceinline__ uint4 ld16_cg(const void* p) {   // L2 (or the peer's L2), never a stale L1 line
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}

// The fused step's reduce side (unused when CW == 0).
struct StepArgs {
  const RItem* ritems;               // one per bucket of the call
  Dests src;                         // src.p[c]: buffer holding cluster c's payload (local or IPC-mapped)
  float* obase;
  unsigned* bdone;                   // per compress item: CTAs whose B phase finished it
  Peers pe;                          // pe.n > 1: P2P — signal / wait peers' arrival flags
  unsigned long long* local_arrive;  // this GPU's arrival flags [bucket * P + cluster]
  unsigned long long seq;
  int b0;                            // global index of the call's first bucket (flag index)
  int PL;                            // compress items per bucket (clusters computed on this GPU)
  SrArgs sr;                         // QSGD generator state (SR kernels only)
};

// Reduce role, TMA variant (LOOPBACK: every payload is local): warp 0 of the group is the
// producer — per bucket it waits until every cluster's payload is complete (grid counter
// bdone), then bulk-copies this CTA's quad slice of all P payloads into a 3-stage shared-memory
// ring; the other warps decode one quad per lane from shared memory, tree-sum, divide and store
// float4 (each warp store = 512 contiguous bytes).  The producer also writes the < 4 tail
// elements of the last slice.  A stage descriptor with nq = ~0 ends the consumers.  (For P2P
// pull, NVLink-latency bulk copies would sit in the TMA queue ahead of the A/B ring copies:
// measured slower there, so pull uses the register-load variant below.)
constexpr int kWsNC = 3;
constexpr uint32_t kWsCStage = 16384;   // payload bytes of all P clusters per C stage
struct WsCMeta {
  float* out;                           // output of the stage's first quad
  uint32_t nq;                          // quads in the stage (~0: stop)
  float sc[8];
};

// One payload byte -> its decoded value (INT8 / QSGD: q * s; FP8: E4M3(c) * s).
template <int F8>
__device__ __forceinline__ float dec_byte(uint32_t byte, float s) {
  if constexpr (F8) return __fmul_rn(fp8_val<F8>(byte), s);
  else return __fmul_rn((float)(int8_t)(byte & 0xFF), s);
}

template <int P, int F8 = 0>
__device__ __forceinline__ void ws_reduce_tma(const StepArgs& a, int nb, int ct, int nC, unsigned char* ringC,
                                              uint64_t* fullC, uint64_t* emptyC, WsCMeta* meta) {
  constexpr uint32_t TB = (kWsCStage / P) & ~15u;   // bytes per cluster per stage
  constexpr uint32_t TQ = TB / 4;                   // quads per stage
  const unsigned G = gridDim.x;
  const int lane = ct & 31;
  if (ct < 32) {
    // ------------------------------------------------------------------ C producer
    if (lane != 0) return;
    const uint64_t pol = l2_evict_first();
    uint32_t fc = 0;
    for (int b = 0; b < nb; ++b) {
      const RItem it = a.ritems[b];
      const uint64_t n4 = it.n >> 2;
      const Slice sl = slice_of(n4, G);
      const bool tail = blockIdx.x == G - 1 && (it.n & 3);
      if (sl.q1 <= sl.q0 && !tail) continue;
      for (int c = 0; c < a.PL; ++c) {
        const unsigned* w = a.bdone + b * a.PL + c;
        unsigned v;
        while (true) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(w) : "memory");
          if (v >= G) break;
          __nanosleep(64);
        }
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");   // generic-proxy payload writes -> TMA reads
      float sc[P];
#pragma unroll
      for (int k = 0; k < P; ++k)
        sc[k] = *reinterpret_cast<volatile const float*>(a.src.p[k] + it.slot_off + (uint64_t)k * it.pb + 8);
      float* out = a.obase + it.out_off;
      for (uint64_t q = sl.q0; q < sl.q1; q += TQ) {
        const uint32_t nq = (uint32_t)min((uint64_t)TQ, sl.q1 - q);
        const uint32_t st = fc % kWsNC, use = fc / kWsNC;
        if (use) mbar_wait(&emptyC[st], (use - 1) & 1u);
        meta[st].out = out + 4 * q;
        meta[st].nq = nq;
#pragma unroll
        for (int k = 0; k < P; ++k) meta[st].sc[k] = sc[k];
        const uint32_t bytes = (nq * 4 + 15) & ~15u;   // within the 16-B padded section
        mbar_expect_tx(&fullC[st], P * bytes);
#pragma unroll
        for (int k = 0; k < P; ++k)
          bulk_g2s(ringC + st * kWsCStage + k * TB, a.src.p[k] + it.slot_off + (uint64_t)k * it.pb + 16 + 4 * q, bytes,
                   &fullC[st], pol);
        ++fc;
      }
      if (tail) {
        for (uint64_t e = n4 * 4; e < it.n; ++e) {
          float v[P];
#pragma unroll
          for (int k = 0; k < P; ++k) {
            const uint8_t qv = *reinterpret_cast<volatile const uint8_t*>(a.src.p[k] + it.slot_off + (uint64_t)k * it.pb + 16 + e);
            v[k] = dec_byte<F8>(qv, sc[k]);
          }
          out[e] = div_p<P>(tree_sum<0, P>(v));
        }
      }
    }
    const uint32_t st = fc % kWsNC, use = fc / kWsNC;
    if (use) mbar_wait(&emptyC[st], (use - 1) & 1u);
    meta[st].nq = 0xFFFFFFFFu;
    mbar_arrive(&fullC[st]);
    return;
  }
  // -------------------------------------------------------------------- C consumers
  const int cc = ct - 32, ncons = nC - 32;
  const uint64_t pol = l2_evict_first();
  uint32_t fc = 0;
  while (true) {
    const uint32_t st = fc % kWsNC, use = fc / kWsNC;
    mbar_wait(&fullC[st], use & 1u);
    const uint32_t nq = meta[st].nq;
    if (nq == 0xFFFFFFFFu) break;
    float* out = meta[st].out;
    float sc[P];
#pragma unroll
    for (int k = 0; k < P; ++k) sc[k] = meta[st].sc[k];
    const uint32_t* pay = reinterpret_cast<const uint32_t*>(ringC + st * kWsCStage);
    for (uint32_t j = cc; j < nq; j += ncons) {
      float t[4][P];
#pragma unroll
      for (int k = 0; k < P; ++k) {
        const uint32_t w = pay[k * (TB / 4) + j];
#pragma unroll
        for (int e = 0; e < 4; ++e) t[e][k] = dec_byte<F8>(w >> (8 * e), sc[k]);
      }
      st4_hint(out + 4 * j,
               make_float4(div_p<P>(tree_sum<0, P>(t[0])), div_p<P>(tree_sum<0, P>(t[1])),
                           div_p<P>(tree_sum<0, P>(t[2])), div_p<P>(tree_sum<0, P>(t[3]))),
               pol);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&emptyC[st]);
    ++fc;
  }
}

// Reduce role, register-load variant (P2P pull): buckets in order; this CTA's share of bucket b is the same quad slice its B
// warps quantised, in 16-element groups (one 16-B load per cluster), staged through a per-warp
// shared-memory transpose so each store instruction writes 512 contiguous bytes.
template <int P, int F8 = 0>
__device__ __forceinline__ void ws_reduce_ld(const StepArgs& a, int nb, int ct, int nC, float* s_sc,
                                               volatile uint32_t* s_abort, float* s_out, uint32_t* flags) {
  // F8: 0 INT8 / QSGD bytes, 1 E4M3, 2 E5M2, 3 FP16 (2-byte codes, no scale).  E elements per
  // 16-byte group; a CTA's quad slice is 4-quad aligned, so groups never straddle two CTAs.
  constexpr int E = F8 == 3 ? 8 : 16, QPG = E / 4, SROW = E + 1, U = P <= 2 ? 2 : 1;
  const unsigned G = gridDim.x;
  const int lane = ct & 31, cw = ct >> 5, ncw = nC / 32;
  float* sw = s_out + cw * 32 * SROW;
  const uint64_t pol = l2_evict_first();
  for (int b = 0; b < nb; ++b) {
    const RItem it = a.ritems[b];
    float* scb = s_sc + (b & 1) * 8;   // double-buffered: rewritten only after the next barrier
    if (ct == 0) {
      for (int c = 0; c < a.PL; ++c) {
        const unsigned* w = a.bdone + b * a.PL + c;
        unsigned v;
        while (true) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(w) : "memory");
          if (v >= G) break;
          __nanosleep(128);
        }
      }
      if (a.pe.n > 1) {
        const unsigned long long t0 = globaltimer_ns_u64();
        for (int c = 0; c < P && !*s_abort; ++c) {
          if (c == a.pe.me) continue;
          while (ld_acquire_sys_u64(a.local_arrive + (size_t)(a.b0 + b) * P + c) < a.seq) {
            if (globaltimer_ns_u64() - t0 > 60ull * 1000000000ull) {
              atomicOr(flags, kFlagPeerTimeout);
              *s_abort = 1u;
              break;
            }
            __nanosleep(256);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < P; ++k)
        scb[k] = F8 == 3 ? 1.0f : *reinterpret_cast<volatile const float*>(a.src.p[k] + it.slot_off + (uint64_t)k * it.pb + 8);
    }
    named_sync(3, nC);
    if (*s_abort) return;
    float sc[P];
#pragma unroll
    for (int k = 0; k < P; ++k) sc[k] = scb[k];
    const uint64_t n4 = it.n >> 2;
    const Slice sl = slice_of(n4, G);
    const uint64_t g0 = sl.q0 / QPG, g1 = sl.q1 / QPG;   // whole E-element groups of this slice
    float* out = a.obase + it.out_off;
    auto slot = [&](int k, uint64_t gi) { return a.src.p[k] + it.slot_off + (uint64_t)k * it.pb + 16 + 16 * gi; };
    auto dec = [&](const uint4& x4, int e, float s) {
      if constexpr (F8 == 3) {
        const uint32_t x = (e >> 1) == 0 ? x4.x : (e >> 1) == 1 ? x4.y : (e >> 1) == 2 ? x4.z : x4.w;
        return __half2float(__ushort_as_half((unsigned short)((e & 1) ? (x >> 16) : (x & 0xFFFFu))));
      } else {
        const uint32_t x = (e >> 2) == 0 ? x4.x : (e >> 2) == 1 ? x4.y : (e >> 2) == 2 ? x4.z : x4.w;
        return dec_byte<F8>(x >> (8 * (e & 3)), s);
      }
    };
    auto store_groups = [&](uint64_t gw0, uint64_t gend) {   // the warp's 32 groups from the transpose buffer
#pragma unroll
      for (int v = 0; v < E / 4; ++v) {
        const int qq = v * 32 + lane, src_lane = qq / QPG, src_e = (qq % QPG) * 4;
        if (gw0 + src_lane < gend) {
          const float* r = sw + src_lane * SROW + src_e;
          st4_hint(out + 4 * (gw0 * QPG + qq), make_float4(r[0], r[1], r[2], r[3]), pol);
        }
      }
    };
    for (uint64_t gb = g0 + (uint64_t)cw * 32 * U; gb < g1; gb += (uint64_t)ncw * 32 * U) {
      if constexpr (P <= 4) {
        uint4 w[U][P];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t gi = gb + u * 32 + lane;
          if (gi < g1) {
#pragma unroll
            for (int k = 0; k < P; ++k) w[u][k] = ld16_cg(slot(k, gi));
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool ok = gb + u * 32 + lane < g1;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            float t[P];
#pragma unroll
            for (int k = 0; k < P; ++k) t[k] = ok ? dec(w[u][k], e, sc[k]) : 0.0f;
            sw[lane * SROW + e] = div_p<P>(tree_sum<0, P>(t));
          }
          __syncwarp();
          store_groups(gb + u * 32, g1);
          __syncwarp();
        }
      } else {
        // P > 4: the two subtrees of tree_sum<0, P> one after the other (register budget of a
        // 1024-thread CTA); the left subtree's sums wait in the transpose buffer
        constexpr int MID = (P + 1) / 2;
        const uint64_t gi = gb + lane;
        const bool ok = gi < g1;
        {
          uint4 w[MID];
#pragma unroll
          for (int k = 0; k < MID; ++k) w[k] = ok ? ld16_cg(slot(k, gi)) : make_uint4(0, 0, 0, 0);
#pragma unroll
          for (int e = 0; e < E; ++e) {
            float t[P];
#pragma unroll
            for (int k = 0; k < MID; ++k) t[k] = dec(w[k], e, sc[k]);
            sw[lane * SROW + e] = tree_sum<0, MID>(t);
          }
        }
        {
          uint4 w[P - MID];
#pragma unroll
          for (int k = MID; k < P; ++k) w[k - MID] = ok ? ld16_cg(slot(k, gi)) : make_uint4(0, 0, 0, 0);
#pragma unroll
          for (int e = 0; e < E; ++e) {
            float t[P];
#pragma unroll
            for (int k = MID; k < P; ++k) t[k] = dec(w[k - MID], e, sc[k]);
            sw[lane * SROW + e] = div_p<P>(__fadd_rn(sw[lane * SROW + e], tree_sum<MID, P>(t)));
          }
        }
        __syncwarp();
        store_groups(gb, g1);
        __syncwarp();
      }
    }
    // the < E elements after the last whole group of the bucket
    if (blockIdx.x == G - 1 && ct < E) {
      const uint64_t e = (uint64_t)E * (n4 / QPG) + ct;
      if (e < it.n) {
        float v[P];
#pragma unroll
        for (int k = 0; k < P; ++k) {
          const uint8_t* body = a.src.p[k] + it.slot_off + (uint64_t)k * it.pb + 16;
          if constexpr (F8 == 3) {
            const unsigned short hb = *reinterpret_cast<volatile const unsigned short*>(body + 2 * e);
            v[k] = __half2float(__ushort_as_half(hb));
          } else {
            const uint8_t q = *reinterpret_cast<volatile const uint8_t*>(body + e);
            v[k] = dec_byte<F8>(q, sc[k]);
          }
        }
        out[e] = div_p<P>(tree_sum<0, P>(v));
      }
    }
  }
}

// CM: reduce role — 0 none (compress only), 1 TMA variant (LOOPBACK), 2 register loads (P2P pull)
// F8: the same schedules for the FP8 E4M3 codec (NEXT-4, R27) — only the B warps' scale /
// quantise / dequantise and the C warps' byte decode differ.
template <bool EF, int AW, int BW, int CW, int CM, int F8 = 0, bool SR = false>
__global__ void __launch_bounds__(kWsThreads, 1)
    k_int8_ws(const Item* __restrict__ items, int nitems, const float* __restrict__ gbase, float* __restrict__ rbase,
              Dests dst, uint32_t* scratch, uint32_t* flags, unsigned* done, StepArgs sa) {
  static_assert(1 + AW + BW + CW == kWsThreads / 32, "warp roles must fill the CTA");
  constexpr int kA = AW * 32, kB = BW * 32, kC = CW * 32;
  extern __shared__ __align__(128) unsigned char ws_smem[];
  WsStageA* ringA = reinterpret_cast<WsStageA*>(ws_smem);
  WsStageB* ringB = reinterpret_cast<WsStageB*>(ws_smem + sizeof(WsStageA) * kWsNA);
  __shared__ __align__(8) uint64_t fullA[kWsNA], emptyA[kWsNA], fullB[kWsNB], emptyB[kWsNB];
  __shared__ volatile uint32_t s_pdone, s_bdone;   // buckets whose A (resp. B) phase this CTA finished
  __shared__ uint32_t s_amax[AW];
  __shared__ float s_scale[2];
  __shared__ float s_sc[16];
  __shared__ volatile uint32_t s_abort;
  __shared__ __align__(8) uint64_t fullC[kWsNC], emptyC[kWsNC];
  __shared__ WsCMeta s_cmeta[CM == 1 ? kWsNC : 1];
  const unsigned G = gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kWsNA; ++i) { mbar_init(&fullA[i], 1); mbar_init(&emptyA[i], AW); }
    for (int i = 0; i < kWsNB; ++i) { mbar_init(&fullB[i], 1); mbar_init(&emptyB[i], BW); }
    s_pdone = 0;
    s_bdone = 0;
    s_abort = 0;
    if (CM == 1)
      for (int i = 0; i < kWsNC; ++i) { mbar_init(&fullC[i], 1); mbar_init(&emptyC[i], CW > 1 ? CW - 1 : 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
  auto tiles_of = [&](int t, Slice& sl) {
    sl = slice_of(items[t].n >> 2, G);
    return (int)((sl.q1 - sl.q0 + kWsTQ - 1) / kWsTQ);
  };

  if (warp == 0) {
    // ------------------------------------------------------------------ producer
    if (lane != 0) return;
    int ia = 0, ka = 0, ib = 0, kb = 0;
    uint32_t fa = 0, fb = 0;   // fills issued per ring
    Slice sa_{}, sb{};
    int nta = nitems > 0 ? tiles_of(0, sa_) : 0, ntb = nitems > 0 ? tiles_of(0, sb) : 0;
    while (ia < nitems || ib < nitems) {
      bool progress = false;
      if (ia < nitems) {
        if (ka >= nta) {
          ++ia;
          ka = 0;
          if (ia < nitems) nta = tiles_of(ia, sa_);
          progress = true;
        } else if (ia <= ib + 2) {   // A leads B by at most two buckets
          const uint32_t st = fa % kWsNA, use = fa / kWsNA;
          if (use == 0 || mbar_test(&emptyA[st], (use - 1) & 1u)) {
            const Item it = items[ia];
            const uint64_t q = sa_.q0 + (uint64_t)ka * kWsTQ;
            const uint32_t nq = (uint32_t)min((uint64_t)kWsTQ, sa_.q1 - q);
            mbar_expect_tx(&fullA[st], nq * (EF ? 32u : 16u));
            // without EF the quantise warps re-read g (ring B): keep it in L2 (clean lines, no
            // write-back) so that re-read is an L2 hit — 5 B/elem of DRAM instead of 9
            bulk_g2s(ringA[st].g, gbase + it.g_off + 4 * q, nq * 16u, &fullA[st], EF ? pol_stream : pol_keep);
            if (EF) bulk_g2s(ringA[st].r, rbase + it.r_off + 4 * q, nq * 16u, &fullA[st], pol_stream);
            ++fa;
            ++ka;
            progress = true;
          }
        }
      }
      if (ib < nitems) {
        if (kb >= ntb) {
          ++ib;
          kb = 0;
          if (ib < nitems) ntb = tiles_of(ib, sb);
          progress = true;
        } else if (s_pdone > (uint32_t)ib) {   // p(ib) of this CTA is parked and fenced
          const uint32_t st = fb % kWsNB, use = fb / kWsNB;
          if (use == 0 || mbar_test(&emptyB[st], (use - 1) & 1u)) {
            __threadfence_block();
            asm volatile("fence.proxy.async.global;" ::: "memory");
            const Item it = items[ib];
            const uint64_t q = sb.q0 + (uint64_t)kb * kWsTQ;
            const uint32_t nq = (uint32_t)min((uint64_t)kWsTQ, sb.q1 - q);
            mbar_expect_tx(&fullB[st], nq * 16u);
            bulk_g2s(ringB[st].p, (EF ? rbase + it.r_off : gbase + it.g_off) + 4 * q, nq * 16u, &fullB[st], pol_stream);
            ++fb;
            ++kb;
            progress = true;
          }
        }
      }
      if (!progress) __nanosleep(32);
    }
    return;
  }

  if (warp <= AW) {
    // ------------------------------------------------------------------ A warps
    const int at = threadIdx.x - 32, aw = warp - 1;
    uint32_t fa = 0;
    for (int t = 0; t < nitems; ++t) {
      if (t >= 2)
        // B(t-2) finished: bounded L2 footprint.  (ncu r02: this spin is 13 % of the INT8
        // step's instructions, but a 2 us sleep made the step 4 % slower — A's late wake-up
        // costs more than the issue slots it takes; QSGD did not change either way)
        while (s_bdone < (uint32_t)(t - 1)) __nanosleep(64);
      Slice sl;
      const int nt = tiles_of(t, sl);
      const Item it = items[t];
      const float* g = gbase + it.g_off;
      float* r = rbase + it.r_off;
      uint32_t m = 0;
      for (int k = 0; k < nt; ++k) {
        const uint32_t st = fa % kWsNA, use = fa / kWsNA;
        mbar_wait(&fullA[st], use & 1u);
        const uint64_t q0 = sl.q0 + (uint64_t)k * kWsTQ;
        const uint32_t nq = (uint32_t)min((uint64_t)kWsTQ, sl.q1 - q0);
        const WsStageA& S = ringA[st];
#pragma unroll
        for (int u = 0; u < (kWsTQ + kA - 1) / kA; ++u) {
          const uint32_t j = u * kA + at;
          if (j < nq) {
            const float4 p = EF ? add4(S.g[j], S.r[j]) : S.g[j];
            m = max(m, max(max(abs_bits(p.x), abs_bits(p.y)), max(abs_bits(p.z), abs_bits(p.w))));
            if constexpr (EF) st4_hint(r + 4 * (q0 + j), p, pol_keep);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&emptyA[st]);
        ++fa;
      }
      if (blockIdx.x == G - 1 && at < (int)(it.n & 3)) {
        const uint64_t e = (it.n >> 2) * 4 + at;
        const float p = EF ? __fadd_rn(g[e], r[e]) : g[e];
        if constexpr (EF) r[e] = p;
        m = max(m, abs_bits(p));
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");   // parked p -> visible to ring-B copies
      m = __reduce_max_sync(0xFFFFFFFFu, m);
      if (lane == 0) s_amax[aw] = m;
      named_sync(1, kA);
      if (at == 0) {
        uint32_t w = 0;
        for (int i = 0; i < AW; ++i) w = max(w, s_amax[i]);
        if (w) atomicMax(&scratch[it.sidx], w);
        __threadfence();
        atomicAdd(&done[t], 1u);
        __threadfence_block();
        s_pdone = (uint32_t)(t + 1);
      }
      named_sync(1, kA);
    }
    return;
  }

  if (warp <= AW + BW) {
    // ------------------------------------------------------------------ B warps
    const int bt = threadIdx.x - 32 * (1 + AW);
    uint32_t fb = 0;
    for (int t = 0; t < nitems; ++t) {
      Slice sl;
      const int nt = tiles_of(t, sl);
      const Item it = items[t];
      if (bt == 0) {
        unsigned v;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&done[t]) : "memory");
        } while (v < G);
        const uint32_t mbits = *((volatile const uint32_t*)&scratch[it.sidx]);
        if (nonfinite_bits(mbits)) {
          s_scale[0] = 0.0f;
          if (blockIdx.x == 0) atomicOr(flags, kFlagNonfinite);
        } else {
          const float sc = F8 ? fp8_scale_from_bits<F8>(mbits) : int8_scale_from_bits(mbits);
          s_scale[0] = sc;
          s_scale[1] = int8_inv(sc);
          if (blockIdx.x == 0) put_preamble(dst, it.slot_off, F8 == 2 ? M_FP8_E5M2 : F8 ? M_FP8 : (SR ? M_QSGD : M_INT8), (uint32_t)it.n, sc, 0u);
        }
      }
      named_sync(2, kB);
      const float s = s_scale[0], sinv = s_scale[1];
      uint64_t srb = 0;
      if constexpr (SR)
        srb = qsgd_base(sa.sr.seed, sa.sr.step,
                        qsgd_key(sa.sr.cluster0 + it.sidx / sa.sr.num_buckets, sa.sr.shard, it.sidx % sa.sr.num_buckets));
      const bool ok = s != 0.0f;   // scale is never 0 (R4) except for the non-finite marker
      const float* g = gbase + it.g_off;
      float* r = rbase + it.r_off;
      const uint64_t bo = it.slot_off + 16;
      uint32_t* body = reinterpret_cast<uint32_t*>(dst.p[0] + bo);
      for (int k = 0; k < nt; ++k) {
        const uint32_t st = fb % kWsNB, use = fb / kWsNB;
        mbar_wait(&fullB[st], use & 1u);
        const uint64_t q0 = sl.q0 + (uint64_t)k * kWsTQ;
        const uint32_t nq = (uint32_t)min((uint64_t)kWsTQ, sl.q1 - q0);
        const WsStageB& S = ringB[st];
        for (uint32_t j0 = 0; j0 < (uint32_t)kWsTQ; j0 += kB) {
          const uint32_t j = j0 + bt;
          const bool valid = ok && j < nq;
          uint32_t w = 0u;
          if (valid) {
            const float4 p = S.p[j];
            float d0, d1, d2, d3;
            if constexpr (F8) {
              w = fp8x2_fast<F8>(p.x, p.y, s, sinv) | (fp8x2_fast<F8>(p.z, p.w, s, sinv) << 16);
              d0 = __fmul_rn(fp8_val<F8>(w), s); d1 = __fmul_rn(fp8_val<F8>(w >> 8), s);
              d2 = __fmul_rn(fp8_val<F8>(w >> 16), s); d3 = __fmul_rn(fp8_val<F8>(w >> 24), s);
            } else if constexpr (SR) {
              const uint64_t h0 = qsgd_h(srb, 2 * (q0 + j)), h1 = qsgd_h(srb, 2 * (q0 + j) + 1);
              const float a0 = qsgd_qf(p.x, s, sinv, qsgd_hi_f(h0)), a1 = qsgd_qf(p.y, s, sinv, qsgd_lo_f(h0)),
                          a2 = qsgd_qf(p.z, s, sinv, qsgd_hi_f(h1)), a3 = qsgd_qf(p.w, s, sinv, qsgd_lo_f(h1));
              w = byte_of_intf(a0) | (byte_of_intf(a1) << 8) | (byte_of_intf(a2) << 16) | (byte_of_intf(a3) << 24);
              d0 = __fmul_rn(a0, s); d1 = __fmul_rn(a1, s);
              d2 = __fmul_rn(a2, s); d3 = __fmul_rn(a3, s);
            } else {
              const int a0 = int8_qi(p.x, s, sinv), a1 = int8_qi(p.y, s, sinv), a2 = int8_qi(p.z, s, sinv),
                        a3 = int8_qi(p.w, s, sinv);
              w = pack_i8x4(a0, a1, a2, a3);
              d0 = __fmul_rn((float)a0, s); d1 = __fmul_rn((float)a1, s);
              d2 = __fmul_rn((float)a2, s); d3 = __fmul_rn((float)a3, s);
            }
            st_u32_hint(body + q0 + j, w, CW > 0 ? pol_keep : pol_stream);   // fused: C re-reads it from L2
            if constexpr (EF)
              st4_hint(r + 4 * (q0 + j),
                       make_float4(__fsub_rn(p.x, d0), __fsub_rn(p.y, d1), __fsub_rn(p.z, d2), __fsub_rn(p.w, d3)),
                       pol_stream);
          }
          push_u32(dst, bo + 4 * (q0 + j), w, valid);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&emptyB[st]);
        ++fb;
      }
      if (blockIdx.x == G - 1 && ok) {
        if (bt < (int)(it.n & 3)) {
          const uint64_t e = (it.n >> 2) * 4 + bt;
          const float p = EF ? r[e] : g[e];
          uint32_t ce;
          float de;
          if constexpr (F8) {
            ce = fp8x2_of<F8>(p, 0.0f, s) & 0xFF;
            de = __fmul_rn(fp8_val<F8>(ce), s);
          } else if constexpr (SR) {
            const int qe = qsgd_q(p, s, qsgd_u(srb, e));
            ce = (uint32_t)qe & 0xFF;
            de = __fmul_rn((float)qe, s);
          } else {
            const int qe = int8_qi(p, s, sinv);
            ce = (uint32_t)qe & 0xFF;
            de = __fmul_rn((float)qe, s);
          }
          put(dst, bo + e, (uint8_t)ce);
          if constexpr (EF) r[e] = __fsub_rn(p, de);
        }
        zero_padding_t(dst, bo, it.n, bt);
      }
      if constexpr (CW > 0) asm volatile("fence.proxy.async.global;" ::: "memory");   // payload -> C's TMA reads
      named_sync(2, kB);
      if (bt == 0) {
        if constexpr (CW > 0) {
          // publish this CTA's share of item t; the last CTA tells the peers (P2P)
          if (dst.n > 1) __threadfence_system();
          else __threadfence();
          const unsigned old = atomicAdd(&sa.bdone[t], 1u);
          if (old == G - 1 && sa.pe.n > 1) {
            __threadfence_system();
            for (int c = 0; c < sa.pe.n; ++c)
              if (c != sa.pe.me) st_release_sys_u64(sa.pe.arrive[c] + (size_t)(sa.b0 + t) * sa.pe.n + sa.pe.me, sa.seq);
          }
        }
        s_bdone = (uint32_t)(t + 1);
      }
    }
    if (dst.n > 1) __threadfence_system();
    return;
  }

  if constexpr (CW > 0) {
    // ------------------------------------------------------------------ C warps
    const int ct = threadIdx.x - 32 * (1 + AW + BW);
    const int nb = nitems / sa.PL;
    if constexpr (CM == 1) {
      static_assert(CW >= 2, "the TMA reduce role needs a producer warp and consumer warps");
      unsigned char* ringC = ws_smem + sizeof(WsStageA) * kWsNA + sizeof(WsStageB) * kWsNB;
#define NB_C(PP) ws_reduce_tma<PP, F8>(sa, nb, ct, kC, ringC, fullC, emptyC, s_cmeta)
      switch (sa.src.n) {
        case 1: NB_C(1); break;
        case 2: NB_C(2); break;
        case 3: NB_C(3); break;
        case 4: NB_C(4); break;
        case 5: NB_C(5); break;
        case 6: NB_C(6); break;
        case 7: NB_C(7); break;
        default: NB_C(8); break;
      }
#undef NB_C
    } else {
      __shared__ float s_out[CW * 32 * 17];
#define NB_C(PP) ws_reduce_ld<PP, F8>(sa, nb, ct, kC, s_sc, &s_abort, s_out, flags)
      switch (sa.src.n) {
        case 1: NB_C(1); break;
        case 2: NB_C(2); break;
        case 3: NB_C(3); break;
        case 4: NB_C(4); break;
        case 5: NB_C(5); break;
        case 6: NB_C(6); break;
        case 7: NB_C(7); break;
        default: NB_C(8); break;
      }
#undef NB_C
    }
  }
}


// ----------------------------------------------------------------------------- FP16 step
// FP16 compress + exchange + average in ONE cooperative kernel (LOOPBACK or P2P pull; the
// FP16 analogue of the fused INT8 step).  FP16 needs no bucket-wide scale, so the compress side
// streams without a grid barrier:
//   warp 0           producer: TMA ring of the g and r tiles of the CTA's slice of item t
//   warps 1..AW      p = g + r, h = RNE16(p) -> payload (8 B per quad), r <- p - h; when the CTA's
//                    slice of item t is done: fence, ARRIVE on bdone[t]; the last CTA to arrive
//                    publishes bucket t to the peers (system-scope release of the arrival word)
//   CW warps         reduce role (ws_reduce_ld<P, 3>): per bucket wait for bdone and, P2P, for
//                    every peer's arrival word, load the P payloads (peers' over NVLink, 16-B
//                    loads), tree-sum, divide, store — overlapping the NVLink-bound pull of bucket
//                    b with the HBM-bound compress of bucket b + 1.
template <bool EF, int AW, int CW>
__global__ void __launch_bounds__(kWsThreads, 1)
    k_fp16_step(const Item* __restrict__ items, int nitems, const float* __restrict__ gbase, float* __restrict__ rbase,
                Dests dst, uint32_t* flags, StepArgs sa) {
  static_assert(1 + AW + CW == kWsThreads / 32, "warp roles must fill the CTA");
  constexpr int kA = AW * 32, kC = CW * 32;
  extern __shared__ __align__(128) unsigned char f16s_smem[];
  WsStageA* ringA = reinterpret_cast<WsStageA*>(f16s_smem);
  __shared__ __align__(8) uint64_t fullA[kWsNA], emptyA[kWsNA];
  __shared__ float s_sc[16];
  __shared__ volatile uint32_t s_abort;
  __shared__ float s_out[CW * 32 * 9];
  const unsigned G = gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kWsNA; ++i) { mbar_init(&fullA[i], 1); mbar_init(&emptyA[i], AW); }
    s_abort = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
  auto tiles_of = [&](int t, Slice& sl) {
    sl = slice_of(items[t].n >> 2, G);
    return (int)((sl.q1 - sl.q0 + kWsTQ - 1) / kWsTQ);
  };
  if (warp == 0) {
    // ------------------------------------------------------------------ producer
    if (lane != 0) return;
    uint32_t fa = 0;
    for (int t = 0; t < nitems; ++t) {
      Slice sl;
      const int nt = tiles_of(t, sl);
      const Item it = items[t];
      for (int k = 0; k < nt; ++k) {
        const uint32_t st = fa % kWsNA, use = fa / kWsNA;
        if (use) mbar_wait(&emptyA[st], (use - 1) & 1u);
        const uint64_t q = sl.q0 + (uint64_t)k * kWsTQ;
        const uint32_t nq = (uint32_t)min((uint64_t)kWsTQ, sl.q1 - q);
        mbar_expect_tx(&fullA[st], nq * (EF ? 32u : 16u));
        bulk_g2s(ringA[st].g, gbase + it.g_off + 4 * q, nq * 16u, &fullA[st], pol_stream);
        if (EF) bulk_g2s(ringA[st].r, rbase + it.r_off + 4 * q, nq * 16u, &fullA[st], pol_stream);
        ++fa;
      }
    }
    return;
  }
  if (warp <= AW) {
    // ------------------------------------------------------------------ compress warps
    const int at = threadIdx.x - 32;
    bool bad = false, ovf = false;
    uint32_t fa = 0;
    for (int t = 0; t < nitems; ++t) {
      Slice sl;
      const int nt = tiles_of(t, sl);
      const Item it = items[t];
      const float* g = gbase + it.g_off;
      float* r = rbase + it.r_off;
      const uint64_t bo = it.slot_off + 16;
      if (blockIdx.x == 0 && at == 0) put_preamble(dst, it.slot_off, M_FP16, (uint32_t)it.n, 1.0f, 0u);
      for (int k = 0; k < nt; ++k) {
        const uint32_t st = fa % kWsNA, use = fa / kWsNA;
        mbar_wait(&fullA[st], use & 1u);
        const uint64_t q0 = sl.q0 + (uint64_t)k * kWsTQ;
        const uint32_t nq = (uint32_t)min((uint64_t)kWsTQ, sl.q1 - q0);
        const WsStageA& S = ringA[st];
        for (uint32_t j = at; j < nq; j += kA) {
          const float4 p = EF ? add4(S.g[j], S.r[j]) : S.g[j];
          uint16_t h0, h1, h2, h3;
          float4 d;
          d.x = fp16_one(p.x, h0, bad, ovf);
          d.y = fp16_one(p.y, h1, bad, ovf);
          d.z = fp16_one(p.z, h2, bad, ovf);
          d.w = fp16_one(p.w, h3, bad, ovf);
          // the reduce role re-reads this payload from L2 (local) or a peer pulls it (NVLink)
          const uint2 packed = make_uint2((uint32_t)h0 | ((uint32_t)h1 << 16), (uint32_t)h2 | ((uint32_t)h3 << 16));
          asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;" ::"l"(dst.p[0] + bo + 8 * (q0 + j)),
                       "r"(packed.x), "r"(packed.y), "l"(pol_keep) : "memory");
          if constexpr (EF)
            st4_hint(r + 4 * (q0 + j),
                     make_float4(__fsub_rn(p.x, d.x), __fsub_rn(p.y, d.y), __fsub_rn(p.z, d.z), __fsub_rn(p.w, d.w)),
                     pol_stream);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&emptyA[st]);
        ++fa;
      }
      if (blockIdx.x == G - 1) {   // tail elements (n % 4) and the 16-byte padding
        if (at < (int)(it.n & 3)) {
          const uint64_t e = (it.n >> 2) * 4 + at;
          const float p = EF ? __fadd_rn(g[e], r[e]) : g[e];
          uint16_t hb;
          const float d = fp16_one(p, hb, bad, ovf);
          put(dst, bo + 2 * e, hb);
          if constexpr (EF) r[e] = __fsub_rn(p, d);
        }
        zero_padding_t(dst, bo, 2 * it.n, at);
      }
      named_sync(1, kA);
      if (at == 0) {
        __threadfence_system();   // payload (incl. the peers' view of it) before the counter / flag
        const unsigned old = atomicAdd(&sa.bdone[t], 1u);
        if (old == G - 1 && sa.pe.n > 1) {
          __threadfence_system();
          for (int c = 0; c < sa.pe.n; ++c)
            if (c != sa.pe.me) st_release_sys_u64(sa.pe.arrive[c] + (size_t)(sa.b0 + t) * sa.pe.n + sa.pe.me, sa.seq);
        }
      }
    }
    raise_flags(flags, bad, ovf);
    return;
  }
  // -------------------------------------------------------------------- reduce warps
  const int ct = threadIdx.x - 32 * (1 + AW);
  const int nb = nitems / sa.PL;
#define NB_C(PP) ws_reduce_ld<PP, 3>(sa, nb, ct, kC, s_sc, &s_abort, s_out, flags)
  switch (sa.src.n) {
    case 1: NB_C(1); break;
    case 2: NB_C(2); break;
    case 3: NB_C(3); break;
    case 4: NB_C(4); break;
    case 5: NB_C(5); break;
    case 6: NB_C(6); break;
    case 7: NB_C(7); break;
    default: NB_C(8); break;
  }
#undef NB_C
}

// FP16 fused step launcher; config 0 = LOOPBACK split, 1 = P2P-pull split.
static const void* fp16_step_kernel(bool ef, int config) {
  if (config == 1) return ef ? (const void*)k_fp16_step<true, 19, 12> : (const void*)k_fp16_step<false, 19, 12>;
  return ef ? (const void*)k_fp16_step<true, 23, 8> : (const void*)k_fp16_step<false, 23, 8>;
}

void launch_fp16_step(const Launch& L, bool ef, const Item* items, int nitems, const float* g, float* r,
                      const Dests& dst_in, uint32_t* flags, uint32_t* bar_words, const RItem* ritems, int b0, int PL,
                      const Dests& src, float* obase, const Peers& pe, unsigned long long* local_arrive, uint64_t seq,
                      int config) {
  Mark mk(L, PH_FP16_STEP);
  cudaMemsetAsync(bar_words, 0, sizeof(unsigned) * (size_t)nitems, L.stream);
  Dests dst = dst_in;
  StepArgs sa{};
  sa.ritems = ritems;
  sa.src = src;
  sa.obase = obase;
  sa.bdone = bar_words;
  sa.pe = pe;
  sa.local_arrive = local_arrive;
  sa.seq = (unsigned long long)seq;
  sa.b0 = b0;
  sa.PL = PL;
  void* args[] = {(void*)&items, (void*)&nitems, (void*)&g, (void*)&r, (void*)&dst, (void*)&flags, (void*)&sa};
  const void* f = fp16_step_kernel(ef, config);
  const size_t smem = sizeof(WsStageA) * kWsNA;
  ensure_smem_attr(f, smem);
  cudaLaunchCooperativeKernel(f, dim3(L.num_sms), dim3(kWsThreads), args, smem, L.stream);
  ++*L.launches;
}

// ----------------------------------------------------------------------------- FP16 TMA
// FP16 + EF streaming with a TMA ring (default for 16-B aligned calls): one CTA per SM walks
// the same grid-stride chunk sequence as k_fp16; warp 0 bulk-loads the g and r tiles of each
// chunk into a 6-stage shared-memory ring (cp.async.bulk, mbarrier transaction counts), warps
// 1..31 convert and store the payload and the residual.  No grid-wide dependency.
constexpr int kF16Threads = 1024, kF16NS = 6;
struct __align__(128) F16Stage {
  float4 g[kChunkQuads];
  float4 r[kChunkQuads];
};

template <bool EF>
__global__ void __launch_bounds__(kF16Threads, 1)
    k_fp16_tma(const Item* __restrict__ items, int nitems, uint64_t chunks, const float* __restrict__ gbase,
               float* __restrict__ rbase, Dests dst, uint32_t* flags) {
  extern __shared__ __align__(128) unsigned char f16_smem[];
  F16Stage* ring = reinterpret_cast<F16Stage*>(f16_smem);
  __shared__ __align__(8) uint64_t full[kF16NS], empty[kF16NS];
  constexpr int kCons = kF16Threads - 32, kConsWarps = kCons / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kF16NS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], kConsWarps); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t pol = l2_evict_first();
  if (warp == 0) {   // ---------------- producer
    if (lane != 0) return;
    int hint = 0;
    uint32_t f = 0;
    for (uint64_t c = blockIdx.x; c < chunks; c += gridDim.x, ++f) {
      const int i = find_item(items, nitems, c, hint);
      hint = i;
      const Item it = items[i];
      const uint64_t j = c - it.chunk0, n4 = it.n >> 2, q0 = j * kChunkQuads;
      const uint32_t nq = q0 < n4 ? (uint32_t)min((uint64_t)kChunkQuads, n4 - q0) : 0u;
      const uint32_t st = f % kF16NS, use = f / kF16NS;
      if (use) mbar_wait(&empty[st], (use - 1) & 1u);
      if (nq) {
        mbar_expect_tx(&full[st], nq * (EF ? 32u : 16u));
        bulk_g2s(ring[st].g, gbase + it.g_off + 4 * q0, nq * 16u, &full[st], pol);
        if (EF) bulk_g2s(ring[st].r, rbase + it.r_off + 4 * q0, nq * 16u, &full[st], pol);
      } else {
        mbar_arrive(&full[st]);   // nothing to copy (tail-only / empty chunk): complete the phase
      }
    }
    return;
  }
  // ------------------------------------------------------------------ consumers
  const int ct = threadIdx.x - 32;
  bool bad = false, ovf = false;
  int hint = 0;
  uint32_t f = 0;
  for (uint64_t c = blockIdx.x; c < chunks; c += gridDim.x, ++f) {
    const int i = find_item(items, nitems, c, hint);
    hint = i;
    const Item it = items[i];
    const uint64_t j = c - it.chunk0, n4 = it.n >> 2, q0 = j * kChunkQuads;
    const uint32_t nq = q0 < n4 ? (uint32_t)min((uint64_t)kChunkQuads, n4 - q0) : 0u;
    const uint32_t st = f % kF16NS, use = f / kF16NS;
    mbar_wait(&full[st], use & 1u);
    float* r = rbase + it.r_off;
    const uint64_t bo = it.slot_off + 16;
    if (j == 0 && ct == 0) put_preamble(dst, it.slot_off, M_FP16, (uint32_t)it.n, 1.0f, 0u);
    const F16Stage& S = ring[st];
    for (uint32_t x0 = 0; x0 < (uint32_t)kChunkQuads; x0 += kCons) {
      const uint32_t x = x0 + ct;
      const uint64_t q = q0 + x;
      const bool valid = x < nq;
      uint2 packed = make_uint2(0u, 0u);
      if (valid) {
        const float4 p = EF ? add4(S.g[x], S.r[x]) : S.g[x];
        uint16_t h0, h1, h2, h3;
        float4 d;
        d.x = fp16_one(p.x, h0, bad, ovf);
        d.y = fp16_one(p.y, h1, bad, ovf);
        d.z = fp16_one(p.z, h2, bad, ovf);
        d.w = fp16_one(p.w, h3, bad, ovf);
        packed = make_uint2((uint32_t)h0 | ((uint32_t)h1 << 16), (uint32_t)h2 | ((uint32_t)h3 << 16));
        *reinterpret_cast<uint2*>(dst.p[0] + bo + 8 * q) = packed;
        if constexpr (EF)
          st4(r + 4 * q, make_float4(__fsub_rn(p.x, d.x), __fsub_rn(p.y, d.y), __fsub_rn(p.z, d.z), __fsub_rn(p.w, d.w)));
      }
      if (x0 < (uint32_t)kChunkQuads) push_u64(dst, bo + 8 * q, packed, valid);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (j == n4 / kChunkQuads) {   // tail elements (n % 4) and the 16-byte padding
      const float* g = gbase + it.g_off;
      if (ct < (int)(it.n & 3)) {
        const uint64_t e = n4 * 4 + ct;
        const float p = EF ? __fadd_rn(g[e], r[e]) : g[e];
        uint16_t hb;
        const float d = fp16_one(p, hb, bad, ovf);
        put(dst, bo + 2 * e, hb);
        if constexpr (EF) r[e] = __fsub_rn(p, d);
      }
      zero_padding_t(dst, bo, 2 * it.n, ct);
    }
  }
  raise_flags(flags, bad, ovf);
  if (dst.n > 1) __threadfence_system();
}

bool launch_fp16_tma(const Launch& L, bool ef, const Item* items, int nitems, uint64_t chunks, const float* g,
                     float* r, const Dests& slots, uint32_t* flags) {
  const size_t smem = sizeof(F16Stage) * kF16NS;
  ensure_smem_attr(ef ? (const void*)k_fp16_tma<true> : (const void*)k_fp16_tma<false>, smem);
  Mark mk(L, PH_FP16);
  const unsigned grid = (unsigned)std::min<uint64_t>(chunks, (uint64_t)L.num_sms);
  if (ef) k_fp16_tma<true><<<grid, kF16Threads, smem, L.stream>>>(items, nitems, chunks, g, r, slots, flags);
  else k_fp16_tma<false><<<grid, kF16Threads, smem, L.stream>>>(items, nitems, chunks, g, r, slots, flags);
  ++*L.launches;
  return true;
}

// The single-pass kernels need a cooperative launch of one 1024-thread CTA per SM with the two
// TMA rings in dynamic shared memory; false when the device cannot host that grid.
bool int8_onchip_capacity(int device, uint64_t* max_items, int* grid, size_t* smem) {
  int sms = 0, coop = 0, optin = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  const size_t need = sizeof(WsStageA) * kWsNA + sizeof(WsStageB) * kWsNB + (size_t)kWsNC * kWsCStage;
  cudaGetLastError();
  *grid = sms;
  *max_items = 0;
  *smem = sizeof(WsStageA) * kWsNA + sizeof(WsStageB) * kWsNB;
  return coop && sms > 0 && (size_t)optin >= need;
}

// kind: 0 INT8, 1 FP8 E4M3, 2 QSGD (compress only: no reduce warps)
static const void* ws_compress_kernel(bool ef, int kind) {
  if (kind == 3) return ef ? (const void*)k_int8_ws<true, 8, 23, 0, 0, 2> : (const void*)k_int8_ws<false, 8, 23, 0, 0, 2>;
  if (kind == 2) return ef ? (const void*)k_int8_ws<true, 8, 23, 0, 0, 0, true>
                           : (const void*)k_int8_ws<false, 8, 23, 0, 0, 0, true>;
  if (kind == 1) return ef ? (const void*)k_int8_ws<true, 8, 23, 0, 0, 1>
                           : (const void*)k_int8_ws<false, 8, 23, 0, 0, 1>;
  return ef ? (const void*)k_int8_ws<true, 8, 23, 0, 0> : (const void*)k_int8_ws<false, 8, 23, 0, 0>;
}

template <bool EF>
static const void* step_kernel(int config, int kind);
static const void* fp16_step_kernel(bool ef, int config);
__global__ void k_exchange_flags(Peers pe, unsigned long long* local, int lo, int hi, unsigned long long seq,
                                 uint32_t* flags);

void preload_ws() {
  cudaFuncAttributes a;
  for (int kind = 0; kind < 4; ++kind)
    for (int ef = 0; ef < 2; ++ef) {
      cudaFuncGetAttributes(&a, ws_compress_kernel(ef != 0, kind));
      for (int config = 0; config <= 10; ++config) {
        cudaFuncGetAttributes(&a, step_kernel<true>(config, kind));
        cudaFuncGetAttributes(&a, step_kernel<false>(config, kind));
      }
    }
  for (int c = 0; c < 2; ++c) {
    cudaFuncGetAttributes(&a, fp16_step_kernel(true, c));
    cudaFuncGetAttributes(&a, fp16_step_kernel(false, c));
  }
  cudaFuncGetAttributes(&a, (const void*)k_fp16_tma<true>);
  cudaFuncGetAttributes(&a, (const void*)k_fp16_tma<false>);
  cudaFuncGetAttributes(&a, (const void*)k_exchange_flags);
}

void launch_ws_compress(const Launch& L, bool ef, int kind, const Item* items, int nitems, const float* g, float* r,
                        const Dests& slots_in, uint32_t* scratch, uint32_t* flags, uint32_t* done_words,
                        const SrArgs& srargs) {
  Dests slots = slots_in;
  Mark mk(L, kind == 2 ? PH_QSGD_QUANT : (kind == 1 || kind == 3 ? PH_FP8_QUANT : PH_INT8_ONCHIP));
  cudaMemsetAsync(done_words, 0, sizeof(unsigned) * (size_t)nitems, L.stream);
  unsigned* done = done_words;
  StepArgs sa{};
  sa.sr = srargs;
  void* args[] = {(void*)&items, (void*)&nitems, (void*)&g, (void*)&r, (void*)&slots, (void*)&scratch,
                  (void*)&flags, (void*)&done, (void*)&sa};
  const void* f = ws_compress_kernel(ef, kind);
  const size_t smem = sizeof(WsStageA) * kWsNA + sizeof(WsStageB) * kWsNB;
  ensure_smem_attr(f, smem);
  cudaLaunchCooperativeKernel(f, dim3(L.num_sms), dim3(kWsThreads), args, smem, L.stream);
  ++*L.launches;
}

// ----------------------------------------------------------------------------- INT8 step
// compress + exchange + decompress/average of an INT8 call in ONE cooperative kernel (the
// warp-specialised kernel with reduce warps).  bar_words: 2 * nitems words (done, bdone).
// Warp splits (A, B, C) of the fused step; config 0 is the default, the rest a tuning sweep.
template <bool EF>
static const void* step_kernel(int config, int kind) {
  if (kind == 1) return config == 4 ? (const void*)k_int8_ws<EF, 4, 16, 11, 2, 1> : (const void*)k_int8_ws<EF, 8, 19, 4, 1, 1>;
  if (kind == 3) return config == 4 ? (const void*)k_int8_ws<EF, 4, 16, 11, 2, 2> : (const void*)k_int8_ws<EF, 8, 19, 4, 1, 2>;
  if (kind == 2) {   // QSGD: the quantise warps are instruction-bound, config 1 gives them more warps
    if (config == 4) return (const void*)k_int8_ws<EF, 4, 16, 11, 2, 0, true>;
    if (config == 1) return (const void*)k_int8_ws<EF, 5, 22, 4, 1, 0, true>;
    return (const void*)k_int8_ws<EF, 8, 19, 4, 1, 0, true>;
  }
  switch (config) {
    // LOOPBACK (TMA reduce role)
    case 1: return (const void*)k_int8_ws<EF, 5, 20, 6, 1>;
    case 2: return (const void*)k_int8_ws<EF, 6, 22, 3, 1>;
    case 3: return (const void*)k_int8_ws<EF, 6, 20, 5, 1>;
    // P2P pull (register-load reduce role); 4 is the pull default
    case 4: return (const void*)k_int8_ws<EF, 4, 16, 11, 2>;
    case 5: return (const void*)k_int8_ws<EF, 5, 16, 10, 2>;
    case 6: return (const void*)k_int8_ws<EF, 4, 15, 12, 2>;
    case 7: return (const void*)k_int8_ws<EF, 3, 16, 12, 2>;
    case 8: return (const void*)k_int8_ws<EF, 4, 17, 10, 2>;
    case 9: return (const void*)k_int8_ws<EF, 5, 18, 8, 2>;
    case 10: return (const void*)k_int8_ws<EF, 3, 17, 11, 2>;
    default: return (const void*)k_int8_ws<EF, 8, 19, 4, 1>;   // LOOPBACK default
  }
}

void launch_int8_step(const Launch& L, bool ef, const Item* items, int nitems, const float* g, float* r,
                      const Dests& dst_in, uint32_t* scratch, uint32_t* flags, uint32_t* bar_words, const RItem* ritems,
                      int b0, int PL, const Dests& src, float* obase, const Peers& pe, unsigned long long* local_arrive,
                      uint64_t seq, int config, int kind, const SrArgs& srargs) {
  Mark mk(L, PH_INT8_STEP);
  cudaMemsetAsync(bar_words, 0, sizeof(unsigned) * 2 * (size_t)nitems, L.stream);
  Dests dst = dst_in;
  unsigned* done = bar_words;
  StepArgs sa{};
  sa.ritems = ritems;
  sa.src = src;
  sa.obase = obase;
  sa.bdone = bar_words + nitems;
  sa.pe = pe;
  sa.local_arrive = local_arrive;
  sa.seq = (unsigned long long)seq;
  sa.b0 = b0;
  sa.PL = PL;
  sa.sr = srargs;
  void* args[] = {(void*)&items, (void*)&nitems, (void*)&g, (void*)&r, (void*)&dst, (void*)&scratch,
                  (void*)&flags, (void*)&done, (void*)&sa};
  if (kind != 0 && config != 4 && !(kind == 2 && config == 1)) config = 0;   // FP8 / QSGD: few splits
  const void* f = ef ? step_kernel<true>(config, kind) : step_kernel<false>(config, kind);
  // the TMA reduce role (LOOPBACK configs) adds its ring; the register-load role uses static smem
  const bool tma_c = config <= 3 || config > 10;
  const size_t smem = sizeof(WsStageA) * kWsNA + sizeof(WsStageB) * kWsNB + (tma_c ? (size_t)kWsNC * kWsCStage : 0);
  ensure_smem_attr(f, smem);
  cudaLaunchCooperativeKernel(f, dim3(L.num_sms), dim3(kWsThreads), args, smem, L.stream);
  ++*L.launches;
}

// ----------------------------------------------------------------------------- P2P flags
// Signal every peer that our payloads of exchange `seq` sit in its slots, then wait for every
// peer's signal.  The compress kernels ended with a system-scope fence after their pushes, and
// stream order puts them before this kernel; the release store publishes them.  A peer that
// never signals (dead rank) sets kFlagPeerTimeout after 60 s instead of hanging the GPU.
__global__ void k_exchange_flags(Peers pe, unsigned long long* local, int lo, int hi, unsigned long long seq,
                                 uint32_t* flags) {
  const int P = pe.n, me = pe.me, total = (hi - lo) * P;
  __threadfence_system();
  for (int x = threadIdx.x; x < total; x += blockDim.x) {
    const int b = lo + x / P, c = x % P;
    if (c != me) st_release_sys_u64(pe.arrive[c] + (size_t)b * P + me, seq);
  }
  const unsigned long long t0 = globaltimer_ns_u64();
  for (int x = threadIdx.x; x < total; x += blockDim.x) {
    const int b = lo + x / P, c = x % P;
    if (c == me) continue;
    while (ld_acquire_sys_u64(local + (size_t)b * P + c) < seq) {
      if (globaltimer_ns_u64() - t0 > 60ull * 1000000000ull) {
        atomicOr(flags, kFlagPeerTimeout);
        return;
      }
    }
  }
}

void launch_exchange_flags(const Launch& L, const Peers& pe, unsigned long long* local_arrive, int lo, int hi,
                           uint64_t seq, uint32_t* flags, int phase) {
  Mark mk(L, phase);
  k_exchange_flags<<<1, 256, 0, L.stream>>>(pe, local_arrive, lo, hi, (unsigned long long)seq, flags);
  ++*L.launches;
}

}  // namespace nb
