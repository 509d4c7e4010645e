// kernels_dense.cu — sm_100a streaming kernels for the dense codecs and the dense reducer.
//
//   K1 k_fp16        : p = g + r; h = RNE16(p); r <- p - h                     (one pass, 14 B/elem)
//   K2 k_absmax      : m = max |g + r| (bit max; NaN/Inf detected as bits >= 0x7F800000)
//   K3 k_int8_quant  : s = fl(m/127); q = clamp(rint(p/s)); r <- p - q*s      (8+4+1 B/elem)
//   K0 k_identity    : payload <- g                                            (non-finite check)
//   K8 k_reduce_dense: out = tree_sum_c D(slot_c) / P                          (P*b + 4 B/elem)
//
// Layout: every kernel walks a table of Items (one per (cluster, bucket)); the global
// chunk space (4096 elements per chunk) is the concatenation of all items' chunks, walked
// grid-stride by a persistent grid of ~8 CTAs x 148 SMs.  Each thread moves 4 quads
// (16 B each of g and r) per chunk with 128-bit loads; payload bytes are written with
// 32/64/128-bit stores.  Paper passages: PAPER.md:101 / :418 (INT8 gradient compression),
// PAPER.md:125-130 Eq. 5 (FP16), PAPER.md:76 (aggregation).
#include <cuda_fp16.h>

#include <algorithm>
#include <mutex>
#include <map>
#include <set>
#include <tuple>
#include <utility>

#include "kernels.h"
#include "dense_common.cuh"

namespace nb {

template <bool VEC>
__device__ __forceinline__ float4 ldq(const float* base, uint64_t q) {
  if constexpr (VEC) {
    return ld4_stream(base + 4 * q);
  } else {
    const float* p = base + 4 * q;
    return make_float4(p[0], p[1], p[2], p[3]);
  }
}
template <bool VEC>
__device__ __forceinline__ void stq(float* base, uint64_t q, float4 v) {
  if constexpr (VEC) {
    st4(base + 4 * q, v);
  } else {
    float* p = base + 4 * q;
    p[0] = v.x; p[1] = v.y; p[2] = v.z; p[3] = v.w;
  }
}

// R18: sections are zero-padded to 16 bytes (slots are reused across methods/steps, so the
// padding is rewritten every time; threads 16.. of the tail chunk, disjoint from the tail
// element writers 0..3).
__device__ __forceinline__ void zero_padding(const Dests& d, uint64_t body_off, uint64_t nbytes) {
  const uint64_t end = pad16(nbytes);
  const uint64_t z = nbytes + (threadIdx.x >= 16 ? threadIdx.x - 16 : end);
  if (z < end) put<uint8_t>(d, body_off + z, (uint8_t)0);
}


// ----------------------------------------------------------------------------- IDENTITY
template <bool VEC>
__global__ void __launch_bounds__(kThreads) k_identity(const Item* __restrict__ items, int nitems, uint64_t chunks,
                                                       const float* __restrict__ gbase, Dests dst,
                                                       uint32_t* flags) {
  int hint = 0;
  bool bad = false;
  for (uint64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    const int i = find_item(items, nitems, c, hint);
    hint = i;
    const Item it = items[i];
    const uint64_t j = c - it.chunk0, n4 = it.n >> 2;
    const float* g = gbase + it.g_off;
    const uint64_t bo = it.slot_off + 16;   // body offset inside every destination
    if (j == 0 && threadIdx.x == 0) put_preamble(dst, it.slot_off, M_IDENTITY, (uint32_t)it.n, 1.0f, 0u);
#pragma unroll
    for (int u = 0; u < kQuadsPerThread; ++u) {
      const uint64_t q = j * kChunkQuads + (uint64_t)u * kThreads + threadIdx.x;
      if (q < n4) {
        float4 v = ldq<VEC>(g, q);
        bad |= nonfinite_bits(abs_bits(v.x)) | nonfinite_bits(abs_bits(v.y)) | nonfinite_bits(abs_bits(v.z)) |
               nonfinite_bits(abs_bits(v.w));
        put(dst, bo + 16 * q, v);
      }
    }
    if (j == n4 / kChunkQuads) {
      if (threadIdx.x < (it.n & 3)) {
        const uint64_t e = n4 * 4 + threadIdx.x;
        float v = g[e];
        bad |= nonfinite_bits(abs_bits(v));
        put(dst, bo + 4 * e, v);
      }
      zero_padding(dst, bo, 4 * it.n);
    }
  }
  raise_flags(flags, bad, false);
  if (dst.n > 1) __threadfence_system();   // pushed payload visible system-wide before the flag
}

// ----------------------------------------------------------------------------- FP16 + EF

template <bool EF, bool VEC>
__global__ void __launch_bounds__(kThreads) k_fp16(const Item* __restrict__ items, int nitems, uint64_t chunks,
                                                   const float* __restrict__ gbase, float* __restrict__ rbase,
                                                   Dests dst, uint32_t* flags) {
  int hint = 0;
  bool bad = false, ovf = false;
  for (uint64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    const int i = find_item(items, nitems, c, hint);
    hint = i;
    const Item it = items[i];
    const uint64_t j = c - it.chunk0, n4 = it.n >> 2;
    const float* g = gbase + it.g_off;
    float* r = rbase + it.r_off;
    const uint64_t bo = it.slot_off + 16;
    if (j == 0 && threadIdx.x == 0) put_preamble(dst, it.slot_off, M_FP16, (uint32_t)it.n, 1.0f, 0u);
    float4 gv[kQuadsPerThread], rv[kQuadsPerThread];
#pragma unroll
    for (int u = 0; u < kQuadsPerThread; ++u) {
      const uint64_t q = j * kChunkQuads + (uint64_t)u * kThreads + threadIdx.x;
      if (q < n4) {
        gv[u] = ldq<VEC>(g, q);
        if constexpr (EF) rv[u] = ld4_stream(r + 4 * q);
      }
    }
#pragma unroll
    for (int u = 0; u < kQuadsPerThread; ++u) {
      const uint64_t q = j * kChunkQuads + (uint64_t)u * kThreads + threadIdx.x;
      uint2 packed = make_uint2(0u, 0u);
      if (q < n4) {
        float4 p = EF ? add4(gv[u], rv[u]) : gv[u];
        uint16_t h0, h1, h2, h3;
        float4 d;
        d.x = fp16_one(p.x, h0, bad, ovf);
        d.y = fp16_one(p.y, h1, bad, ovf);
        d.z = fp16_one(p.z, h2, bad, ovf);
        d.w = fp16_one(p.w, h3, bad, ovf);
        packed = make_uint2((uint32_t)h0 | ((uint32_t)h1 << 16), (uint32_t)h2 | ((uint32_t)h3 << 16));
        *reinterpret_cast<uint2*>(dst.p[0] + bo + 8 * q) = packed;
        if constexpr (EF)
          st4(r + 4 * q, make_float4(__fsub_rn(p.x, d.x), __fsub_rn(p.y, d.y), __fsub_rn(p.z, d.z),
                                     __fsub_rn(p.w, d.w)));
      }
      push_u64(dst, bo + 8 * q, packed, q < n4);   // q % 2 == lane % 2: pairs are 16-B aligned
    }
    if (j == n4 / kChunkQuads) {
      if (threadIdx.x < (it.n & 3)) {
        const uint64_t e = n4 * 4 + threadIdx.x;
        float p = EF ? __fadd_rn(g[e], r[e]) : g[e];
        uint16_t hb;
        float d = fp16_one(p, hb, bad, ovf);
        put(dst, bo + 2 * e, hb);
        if constexpr (EF) r[e] = __fsub_rn(p, d);
      }
      zero_padding(dst, bo, 2 * it.n);
    }
  }
  raise_flags(flags, bad, ovf);
  if (dst.n > 1) __threadfence_system();
}

// ----------------------------------------------------------------------------- INT8 pass 1
template <bool EF, bool VEC>
__global__ void __launch_bounds__(kThreads) k_absmax(const Item* __restrict__ items, int nitems, uint64_t chunks,
                                                     const float* __restrict__ gbase, const float* __restrict__ rbase,
                                                     uint32_t* __restrict__ scratch) {
  int hint = 0, cur = -1;
  uint32_t m = 0;
  for (uint64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    const int i = find_item(items, nitems, c, hint);
    hint = i;
    if (i != cur) {  // block-uniform: flush the running max of the previous item
      if (cur >= 0) {
        uint32_t w = __reduce_max_sync(0xFFFFFFFFu, m);
        if ((threadIdx.x & 31) == 0 && w) atomicMax(&scratch[items[cur].sidx], w);
      }
      cur = i;
      m = 0;
    }
    const Item it = items[i];
    const uint64_t j = c - it.chunk0, n4 = it.n >> 2;
    const float* g = gbase + it.g_off;
    const float* r = rbase + it.r_off;
    float4 gv[kQuadsPerThread], rv[kQuadsPerThread];
#pragma unroll
    for (int u = 0; u < kQuadsPerThread; ++u) {
      const uint64_t q = j * kChunkQuads + (uint64_t)u * kThreads + threadIdx.x;
      if (q < n4) {
        gv[u] = ldq<VEC>(g, q);
        if constexpr (EF) rv[u] = ld4_stream(r + 4 * q);
      }
    }
#pragma unroll
    for (int u = 0; u < kQuadsPerThread; ++u) {
      const uint64_t q = j * kChunkQuads + (uint64_t)u * kThreads + threadIdx.x;
      if (q < n4) {
        float4 p = EF ? add4(gv[u], rv[u]) : gv[u];
        m = max(m, max(max(abs_bits(p.x), abs_bits(p.y)), max(abs_bits(p.z), abs_bits(p.w))));
      }
    }
    if (j == n4 / kChunkQuads && threadIdx.x < (it.n & 3)) {
      const uint64_t e = n4 * 4 + threadIdx.x;
      float p = EF ? __fadd_rn(g[e], r[e]) : g[e];
      m = max(m, abs_bits(p));
    }
  }
  if (cur >= 0) {
    uint32_t w = __reduce_max_sync(0xFFFFFFFFu, m);
    if ((threadIdx.x & 31) == 0 && w) atomicMax(&scratch[items[cur].sidx], w);
  }
}

// ----------------------------------------------------------------------------- INT8 pass 2
template <bool EF, bool VEC, int FP8 = 0, bool SR = false>
__global__ void __launch_bounds__(kThreads) k_int8_quant(const Item* __restrict__ items, int nitems, uint64_t chunks,
                                                         const float* __restrict__ gbase, float* __restrict__ rbase,
                                                         Dests dst,
                                                         const uint32_t* __restrict__ scratch, uint32_t* flags,
                                                         SrArgs sr = SrArgs{}) {
  int hint = 0;
  for (uint64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    const int i = find_item(items, nitems, c, hint);
    hint = i;
    const Item it = items[i];
    const uint64_t j = c - it.chunk0, n4 = it.n >> 2;
    const uint32_t mbits = scratch[it.sidx];
    if (nonfinite_bits(mbits)) {  // all-or-nothing: nothing of this bucket is written
      if (j == 0 && threadIdx.x == 0) atomicOr(flags, kFlagNonfinite);
      continue;
    }
    const float s = FP8 ? fp8_scale_from_bits<FP8>(mbits) : int8_scale_from_bits(mbits);
    const float sinv = int8_inv(s);   // fl(1/s) if normal, else 0 (both fast paths then divide)
    const float* g = gbase + it.g_off;
    float* r = rbase + it.r_off;
    const uint64_t bo = it.slot_off + 16;
    if (j == 0 && threadIdx.x == 0) put_preamble(dst, it.slot_off, FP8 == 2 ? M_FP8_E5M2 : FP8 ? M_FP8 : (SR ? M_QSGD : M_INT8), (uint32_t)it.n, s, 0u);
    uint64_t srb = 0;
    if constexpr (SR)
      srb = qsgd_base(sr.seed, sr.step, qsgd_key(sr.cluster0 + it.sidx / sr.num_buckets, sr.shard, it.sidx % sr.num_buckets));
    float4 gv[kQuadsPerThread], rv[kQuadsPerThread];
#pragma unroll
    for (int u = 0; u < kQuadsPerThread; ++u) {
      const uint64_t q = j * kChunkQuads + (uint64_t)u * kThreads + threadIdx.x;
      if (q < n4) {
        gv[u] = ldq<VEC>(g, q);
        if constexpr (EF) rv[u] = ld4_stream(r + 4 * q);
      }
    }
#pragma unroll
    for (int u = 0; u < kQuadsPerThread; ++u) {
      const uint64_t q = j * kChunkQuads + (uint64_t)u * kThreads + threadIdx.x;
      uint32_t wv = 0u;
      if (q < n4) {
        float4 p = EF ? add4(gv[u], rv[u]) : gv[u];
        float d0, d1, d2, d3;
        if constexpr (FP8) {
          wv = fp8x2_fast<FP8>(p.x, p.y, s, sinv) | (fp8x2_fast<FP8>(p.z, p.w, s, sinv) << 16);
          d0 = __fmul_rn(fp8_val<FP8>(wv), s); d1 = __fmul_rn(fp8_val<FP8>(wv >> 8), s);
          d2 = __fmul_rn(fp8_val<FP8>(wv >> 16), s); d3 = __fmul_rn(fp8_val<FP8>(wv >> 24), s);
        } else if constexpr (SR) {
          const uint64_t h0 = qsgd_h(srb, 2 * q), h1 = qsgd_h(srb, 2 * q + 1);   // elements 4q .. 4q+3
          const float q0 = qsgd_qf(p.x, s, sinv, qsgd_hi_f(h0)), q1 = qsgd_qf(p.y, s, sinv, qsgd_lo_f(h0)),
                      q2 = qsgd_qf(p.z, s, sinv, qsgd_hi_f(h1)), q3 = qsgd_qf(p.w, s, sinv, qsgd_lo_f(h1));
          wv = byte_of_intf(q0) | (byte_of_intf(q1) << 8) | (byte_of_intf(q2) << 16) | (byte_of_intf(q3) << 24);
          d0 = __fmul_rn(q0, s); d1 = __fmul_rn(q1, s); d2 = __fmul_rn(q2, s); d3 = __fmul_rn(q3, s);
        } else {
          int q0 = int8_qi(p.x, s, sinv), q1 = int8_qi(p.y, s, sinv), q2 = int8_qi(p.z, s, sinv), q3 = int8_qi(p.w, s, sinv);
          wv = pack_i8x4(q0, q1, q2, q3);
          d0 = __fmul_rn((float)q0, s); d1 = __fmul_rn((float)q1, s); d2 = __fmul_rn((float)q2, s); d3 = __fmul_rn((float)q3, s);
        }
        *reinterpret_cast<uint32_t*>(dst.p[0] + bo + 4 * q) = wv;
        if constexpr (EF)
          st4(r + 4 * q, make_float4(__fsub_rn(p.x, d0), __fsub_rn(p.y, d1), __fsub_rn(p.z, d2), __fsub_rn(p.w, d3)));
      }
      push_u32(dst, bo + 4 * q, wv, q < n4);   // q % 4 == lane % 4: groups are 16-B aligned
    }
    if (j == n4 / kChunkQuads) {
      if (threadIdx.x < (it.n & 3)) {
        const uint64_t e = n4 * 4 + threadIdx.x;
        float p = EF ? __fadd_rn(g[e], r[e]) : g[e];
        uint32_t ce;
        float de;
        if constexpr (FP8) {
          ce = fp8x2_of<FP8>(p, 0.0f, s) & 0xFF;
          de = __fmul_rn(fp8_val<FP8>(ce), s);
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
      zero_padding(dst, bo, it.n);
    }
  }
  if (dst.n > 1) __threadfence_system();
}

// ----------------------------------------------------------------------------- reduce
template <int METHOD>
__device__ __forceinline__ float decode_one(const uint8_t* slot, uint64_t e, float s) {
  const uint8_t* body = slot + 16;
  if constexpr (METHOD == M_IDENTITY) return reinterpret_cast<const float*>(body)[e];
  else if constexpr (METHOD == M_FP16) return __half2float(reinterpret_cast<const __half*>(body)[e]);
  else if constexpr (METHOD == M_FP8) return __fmul_rn(fp8_val<1>(body[e]), s);
  else if constexpr (METHOD == M_FP8_E5M2) return __fmul_rn(fp8_val<2>(body[e]), s);
  else return __fmul_rn((float)(int8_t)body[e], s);
}

// Element e (compile-time after unrolling) of the 16 payload bytes w.
template <int METHOD>
__device__ __forceinline__ float decode_at(const uint4& w, int e, float s) {
  const uint32_t x = (e * (METHOD == M_IDENTITY ? 4 : (METHOD == M_FP16 ? 2 : 1)) / 4) == 0 ? w.x
                   : (e * (METHOD == M_IDENTITY ? 4 : (METHOD == M_FP16 ? 2 : 1)) / 4) == 1 ? w.y
                   : (e * (METHOD == M_IDENTITY ? 4 : (METHOD == M_FP16 ? 2 : 1)) / 4) == 2 ? w.z : w.w;
  if constexpr (METHOD == M_IDENTITY) {
    return __uint_as_float(x);
  } else if constexpr (METHOD == M_FP16) {
    return __half2float(__ushort_as_half((unsigned short)((e & 1) ? (x >> 16) : (x & 0xFFFF))));
  } else if constexpr (METHOD == M_FP8) {
    return __fmul_rn(fp8_val<1>(x >> (8 * (e & 3))), s);
  } else if constexpr (METHOD == M_FP8_E5M2) {
    return __fmul_rn(fp8_val<2>(x >> (8 * (e & 3))), s);
  } else {
    return __fmul_rn((float)(int8_t)((x >> (8 * (e & 3))) & 0xFF), s);
  }
}


// Every lane loads 16 contiguous payload bytes per cluster (one 128-bit load: 16 INT8, 8 FP16
// or 4 FP32 elements — wide loads are what NVLink pulls and HBM both want), decodes, tree-sums
// and stores the E fp32 results as E/4 float4.  A chunk (4096 elements) is 256 lanes x E x
// (4096 / (256 E)) groups.  src.p[c] = the slot buffer holding cluster c's payload: the local
// buffer (LOOPBACK / NCCL / push) or cluster c's own IPC-mapped buffer (P2P pull, over NVLink).
template <int METHOD, int P, bool VEC>
__global__ void __launch_bounds__(kThreads) k_reduce_dense(const RItem* __restrict__ items, int nitems, uint64_t chunks,
                                                           Dests src, float* __restrict__ obase) {
  constexpr int B = METHOD == M_IDENTITY ? 4 : (METHOD == M_FP16 ? 2 : 1);
  constexpr int E = 16 / B;                       // elements per 16-byte load
  constexpr int NG = (int)(kChunkElems / (kThreads * E));   // groups per lane per chunk
  constexpr int UG = (P * NG <= 8) ? NG : (8 / P > 0 ? 8 / P : 1);   // groups in flight
  // E > 4: a lane's E results are contiguous; stage them through shared memory (row stride E+1,
  // conflict-free) so each warp store instruction writes 512 contiguous bytes
  constexpr int SROW = E + 1;
  __shared__ float s_out[(E > 4) ? (kThreads / 32) * 32 * SROW : 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int hint = 0, cur = -1;
  RItem it{};
  float sc[P];
  for (uint64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    const int i = find_item(items, nitems, c, hint);
    hint = i;
    if (i != cur) {   // per-bucket constants loaded once, not per chunk (block-uniform branch)
      it = items[i];
      cur = i;
#pragma unroll
      for (int k = 0; k < P; ++k)
        sc[k] = (METHOD == M_INT8 || METHOD == M_FP8 || METHOD == M_FP8_E5M2) ? *reinterpret_cast<const float*>(src.p[k] + it.slot_off + k * it.pb + 8) : 1.0f;
    }
    const uint64_t j = c - it.chunk0, nfull = it.n / E;   // groups entirely inside the bucket
    float* out = obase + it.out_off;
#pragma unroll
    for (int h0 = 0; h0 < NG; h0 += UG) {
      uint4 w[UG][P];
#pragma unroll
      for (int u = 0; u < UG; ++u) {
        const uint64_t gidx = j * (kChunkElems / E) + (uint64_t)(h0 + u) * kThreads + threadIdx.x;
        if (gidx < nfull) {
#pragma unroll
          for (int k = 0; k < P; ++k)
            w[u][k] = *reinterpret_cast<const uint4*>(src.p[k] + it.slot_off + k * it.pb + 16 + 16 * gidx);
        }
      }
#pragma unroll
      for (int u = 0; u < UG; ++u) {
        const uint64_t gidx = j * (kChunkElems / E) + (uint64_t)(h0 + u) * kThreads + threadIdx.x;
        const bool ok = gidx < nfull;
        float o[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
          float t[P];
#pragma unroll
          for (int k = 0; k < P; ++k) t[k] = ok ? decode_at<METHOD>(w[u][k], e, sc[k]) : 0.0f;
          o[e] = div_p<P>(tree_sum<0, P>(t));
        }
        if constexpr (E == 4) {
          if (ok) stq<VEC>(out, gidx, make_float4(o[0], o[1], o[2], o[3]));
        } else {
          float* sw = s_out + warp * 32 * SROW;
#pragma unroll
          for (int e = 0; e < E; ++e) sw[lane * SROW + e] = o[e];
          __syncwarp();
          // warp region: groups gw0 .. gw0+31 = elements [gw0*E, gw0*E + 32E); instruction v writes
          // quad v*32 + lane of it
          const uint64_t gw0 = gidx - lane;
#pragma unroll
          for (int v = 0; v < E / 4; ++v) {
            const int qq = v * 32 + lane;                 // quad inside the warp region
            const int src_lane = (4 * qq) / E, src_e = (4 * qq) % E;
            if (gw0 + src_lane < nfull) {
              const float* r = sw + src_lane * SROW + src_e;
              stq<VEC>(out, gw0 * (E / 4) + qq, make_float4(r[0], r[1], r[2], r[3]));
            }
          }
          __syncwarp();
        }
      }
    }
    // elements after the last full group (< E of them) in the bucket's last chunk
    if (j == (nfull * E) / kChunkElems) {
      const uint64_t e = nfull * E + threadIdx.x;
      if (e < it.n && threadIdx.x < E) {
        float v[P];
#pragma unroll
        for (int k = 0; k < P; ++k) v[k] = decode_one<METHOD>(src.p[k] + it.slot_off + k * it.pb, e, sc[k]);
        out[e] = div_p<P>(tree_sum<0, P>(v));
      }
    }
  }
}

// ----------------------------------------------------------------------------- INT8 fused
// Single HBM pass for INT8 + EF (13 B/elem instead of 21).  A cooperative persistent grid
// walks the buckets; iteration t of every CTA interleaves, in ONE loop over its slice,
//
//   A(t)   : p = g + r for bucket t, parked back into r (L2 evict_last), running max, then
//            ARRIVE on done[t] (atomicMax of the bucket max before it)
//   B(t-2) : s = fl(max/127) of bucket t-2, re-read p from r (an L2 hit), quantise, write
//            the payload and the residual r = p - q*s (L2 evict_first)
//
// B(t-2) WAITS until all CTAs arrived on done[t-2], which they did one whole iteration ago,
// so in steady state nobody stalls (a split arrive/wait barrier with a lag of two), and the
// loads of both phases are in flight together.  The same CTA owns the same slice of a bucket
// in A and B, so the only cross-CTA datum is the max.  L2 holds p of two buckets (~52 MB at
// 25 MiB buckets) next to the streamed traffic; if it did not, the cost degrades to the
// two-pass traffic, never to a wrong result.  Without EF, B re-reads g.

// ----------------------------------------------------------------------------- launchers
int occupancy_per_sm(const void* kernel, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, int, size_t>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_tuple(dev, kernel, threads, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int per = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem) != cudaSuccess || per < 1) per = 1;
  cache[key] = per;
  return per;
}

void ensure_smem_attr(const void* kernel, size_t bytes) {
  // the attribute is an upper bound: keep the largest value set per (device, kernel) — setting a
  // smaller one for a later call would break the earlier size (e.g. the bracket kernel's
  // sample capacity differs between contexts)
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = done.find({dev, kernel});
  if (it != done.end() && it->second >= bytes) return;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess)
    done[{dev, kernel}] = bytes;
}

static void touch(const void* f) {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, f);
}
template <int M, int... Ps>
static void touch_reduce(std::integer_sequence<int, Ps...>) {
  (touch((const void*)k_reduce_dense<M, Ps + 1, true>), ...);
  (touch((const void*)k_reduce_dense<M, Ps + 1, false>), ...);
}
void preload_dense() {
  touch((const void*)k_identity<true>); touch((const void*)k_identity<false>);
  touch((const void*)k_fp16<true, true>); touch((const void*)k_fp16<true, false>);
  touch((const void*)k_fp16<false, true>); touch((const void*)k_fp16<false, false>);
  touch((const void*)k_absmax<true, true>); touch((const void*)k_absmax<true, false>);
  touch((const void*)k_absmax<false, true>); touch((const void*)k_absmax<false, false>);
#define NB_Q(F, SR)                                                                                   \
  touch((const void*)k_int8_quant<true, true, F, SR>); touch((const void*)k_int8_quant<true, false, F, SR>); \
  touch((const void*)k_int8_quant<false, true, F, SR>); touch((const void*)k_int8_quant<false, false, F, SR>)
  NB_Q(0, false); NB_Q(1, false); NB_Q(2, false); NB_Q(0, true);
#undef NB_Q
  touch_reduce<M_IDENTITY>(std::make_integer_sequence<int, 8>{});
  touch_reduce<M_FP16>(std::make_integer_sequence<int, 8>{});
  touch_reduce<M_INT8>(std::make_integer_sequence<int, 8>{});
  touch_reduce<M_FP8>(std::make_integer_sequence<int, 8>{});
  touch_reduce<M_FP8_E5M2>(std::make_integer_sequence<int, 8>{});
}

void preload_kernels() {
  static std::mutex mu;
  static std::set<int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(dev)) return;
  preload_dense();
  preload_ws();
  preload_intra();
  preload_topk();
  cudaGetLastError();
  done.insert(dev);
}

#define GRID(kernel) persistent_grid(L, chunks, (const void*)(kernel), kThreads)

void launch_identity(const Launch& L, bool vec, const Item* items, int nitems, uint64_t chunks, const float* g,
                     const Dests& slots, uint32_t* flags) {
  if (!chunks) return;
  Mark mk(L, PH_IDENTITY);
  if (vec) k_identity<true><<<GRID(k_identity<true>), kThreads, 0, L.stream>>>(items, nitems, chunks, g, slots, flags);
  else k_identity<false><<<GRID(k_identity<false>), kThreads, 0, L.stream>>>(items, nitems, chunks, g, slots, flags);
  ++*L.launches;
}

void launch_fp16(const Launch& L, bool ef, bool vec, const Item* items, int nitems, uint64_t chunks, const float* g,
                 float* r, const Dests& slots, uint32_t* flags) {
  if (!chunks) return;
  Mark mk(L, PH_FP16);
  if (ef && vec) k_fp16<true, true><<<GRID((k_fp16<true, true>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, slots, flags);
  else if (ef) k_fp16<true, false><<<GRID((k_fp16<true, false>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, slots, flags);
  else if (vec) k_fp16<false, true><<<GRID((k_fp16<false, true>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, slots, flags);
  else k_fp16<false, false><<<GRID((k_fp16<false, false>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, slots, flags);
  ++*L.launches;
}

void launch_absmax(const Launch& L, bool ef, bool vec, const Item* items, int nitems, uint64_t chunks,
                   const float* g, const float* r, uint32_t* scratch) {
  if (!chunks) return;
  Mark mk(L, PH_ABSMAX);
  if (ef && vec) k_absmax<true, true><<<GRID((k_absmax<true, true>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, scratch);
  else if (ef) k_absmax<true, false><<<GRID((k_absmax<true, false>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, scratch);
  else if (vec) k_absmax<false, true><<<GRID((k_absmax<false, true>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, scratch);
  else k_absmax<false, false><<<GRID((k_absmax<false, false>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, scratch);
  ++*L.launches;
}

void launch_int8_quant(const Launch& L, bool ef, bool vec, const Item* items, int nitems, uint64_t chunks,
                       const float* g, float* r, const Dests& slots, const uint32_t* scratch, uint32_t* flags) {
  if (!chunks) return;
  Mark mk(L, PH_INT8_QUANT);
  if (ef && vec) k_int8_quant<true, true><<<GRID((k_int8_quant<true, true>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, slots, scratch, flags);
  else if (ef) k_int8_quant<true, false><<<GRID((k_int8_quant<true, false>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, slots, scratch, flags);
  else if (vec) k_int8_quant<false, true><<<GRID((k_int8_quant<false, true>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, slots, scratch, flags);
  else k_int8_quant<false, false><<<GRID((k_int8_quant<false, false>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, slots, scratch, flags);
  ++*L.launches;
}

template <int F>
static void fp8_quant_f(const Launch& L, bool ef, bool vec, const Item* items, int nitems, uint64_t chunks,
                        const float* g, float* r, const Dests& slots, const uint32_t* scratch, uint32_t* flags) {
  if (ef && vec) k_int8_quant<true, true, F><<<GRID((k_int8_quant<true, true, F>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, slots, scratch, flags);
  else if (ef) k_int8_quant<true, false, F><<<GRID((k_int8_quant<true, false, F>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, slots, scratch, flags);
  else if (vec) k_int8_quant<false, true, F><<<GRID((k_int8_quant<false, true, F>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, slots, scratch, flags);
  else k_int8_quant<false, false, F><<<GRID((k_int8_quant<false, false, F>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, slots, scratch, flags);
}

void launch_fp8_quant(const Launch& L, bool ef, bool vec, const Item* items, int nitems, uint64_t chunks,
                      const float* g, float* r, const Dests& slots, const uint32_t* scratch, uint32_t* flags, int fmt) {
  if (!chunks) return;
  Mark mk(L, PH_FP8_QUANT);
  if (fmt == 2) fp8_quant_f<2>(L, ef, vec, items, nitems, chunks, g, r, slots, scratch, flags);
  else fp8_quant_f<1>(L, ef, vec, items, nitems, chunks, g, r, slots, scratch, flags);
  ++*L.launches;
}

void launch_qsgd_quant(const Launch& L, bool ef, bool vec, const Item* items, int nitems, uint64_t chunks,
                       const float* g, float* r, const Dests& slots, const uint32_t* scratch, uint32_t* flags,
                       const SrArgs& sr) {
  if (!chunks) return;
  Mark mk(L, PH_QSGD_QUANT);
  if (ef && vec) k_int8_quant<true, true, false, true><<<GRID((k_int8_quant<true, true, false, true>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, slots, scratch, flags, sr);
  else if (ef) k_int8_quant<true, false, false, true><<<GRID((k_int8_quant<true, false, false, true>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, slots, scratch, flags, sr);
  else if (vec) k_int8_quant<false, true, false, true><<<GRID((k_int8_quant<false, true, false, true>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, slots, scratch, flags, sr);
  else k_int8_quant<false, false, false, true><<<GRID((k_int8_quant<false, false, false, true>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, slots, scratch, flags, sr);
  ++*L.launches;
}

template <int METHOD, int P>
static void reduce_p(const Launch& L, bool vec, const RItem* items, int nitems, uint64_t chunks, const Dests& slots,
                     float* out) {
  if (vec) k_reduce_dense<METHOD, P, true><<<GRID((k_reduce_dense<METHOD, P, true>)), kThreads, 0, L.stream>>>(items, nitems, chunks, slots, out);
  else k_reduce_dense<METHOD, P, false><<<GRID((k_reduce_dense<METHOD, P, false>)), kThreads, 0, L.stream>>>(items, nitems, chunks, slots, out);
}
template <int METHOD>
static void reduce_m(const Launch& L, int P, bool vec, const RItem* items, int nitems, uint64_t chunks,
                     const Dests& slots, float* out) {
  switch (P) {
    case 1: reduce_p<METHOD, 1>(L, vec, items, nitems, chunks, slots, out); break;
    case 2: reduce_p<METHOD, 2>(L, vec, items, nitems, chunks, slots, out); break;
    case 3: reduce_p<METHOD, 3>(L, vec, items, nitems, chunks, slots, out); break;
    case 4: reduce_p<METHOD, 4>(L, vec, items, nitems, chunks, slots, out); break;
    case 5: reduce_p<METHOD, 5>(L, vec, items, nitems, chunks, slots, out); break;
    case 6: reduce_p<METHOD, 6>(L, vec, items, nitems, chunks, slots, out); break;
    case 7: reduce_p<METHOD, 7>(L, vec, items, nitems, chunks, slots, out); break;
    default: reduce_p<METHOD, 8>(L, vec, items, nitems, chunks, slots, out); break;
  }
}
void launch_reduce_dense(const Launch& L, int method, int P, bool vec, const RItem* items, int nitems, uint64_t chunks,
                         const Dests& slots, float* out) {
  if (!chunks) return;
  Mark mk(L, PH_REDUCE_DENSE);
  if (method == M_IDENTITY) reduce_m<M_IDENTITY>(L, P, vec, items, nitems, chunks, slots, out);
  else if (method == M_FP16) reduce_m<M_FP16>(L, P, vec, items, nitems, chunks, slots, out);
  else if (method == M_FP8) reduce_m<M_FP8>(L, P, vec, items, nitems, chunks, slots, out);
  else if (method == M_FP8_E5M2) reduce_m<M_FP8_E5M2>(L, P, vec, items, nitems, chunks, slots, out);
  else reduce_m<M_INT8>(L, P, vec, items, nitems, chunks, slots, out);   // INT8 and QSGD: same decode
  ++*L.launches;
}

}  // namespace nb
