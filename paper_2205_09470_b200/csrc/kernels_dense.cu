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
#include <unordered_map>

#include "kernels.h"

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
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}

// R18: sections are zero-padded to 16 bytes (slots are reused across methods/steps, so the
// padding is rewritten every time; threads 16.. of the tail chunk, disjoint from the tail
// element writers 0..3).
__device__ __forceinline__ void zero_padding(const Dests& d, uint64_t body_off, uint64_t nbytes) {
  const uint64_t end = pad16(nbytes);
  const uint64_t z = nbytes + (threadIdx.x >= 16 ? threadIdx.x - 16 : end);
  if (z < end) put<uint8_t>(d, body_off + z, (uint8_t)0);
}

__device__ __forceinline__ void zero_padding_t(const Dests& d, uint64_t body_off, uint64_t nbytes, int tid) {
  const uint64_t end = pad16(nbytes);
  const uint64_t z = nbytes + (tid >= 16 ? tid - 16 : end);
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
__device__ __forceinline__ float fp16_one(float p, uint16_t& hb, bool& bad, bool& ovf) {
  __half h = __float2half_rn(p);              // IEEE binary32 -> binary16, RNE, subnormals kept
  hb = __half_as_ushort(h);
  const uint32_t ab = abs_bits(p);
  bad |= nonfinite_bits(ab);
  ovf |= ((hb & 0x7FFFu) == 0x7C00u) && !nonfinite_bits(ab);   // finite p rounded to +-inf (R10)
  return __half2float(h);
}

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
template <bool EF, bool VEC, bool FP8 = false, bool SR = false>
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
    const float s = FP8 ? fp8_scale_from_bits(mbits) : int8_scale_from_bits(mbits);
    const float sinv = int8_inv(s);   // fl(1/s) if normal, else 0 (both fast paths then divide)
    const float* g = gbase + it.g_off;
    float* r = rbase + it.r_off;
    const uint64_t bo = it.slot_off + 16;
    if (j == 0 && threadIdx.x == 0) put_preamble(dst, it.slot_off, FP8 ? M_FP8 : (SR ? M_QSGD : M_INT8), (uint32_t)it.n, s, 0u);
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
          wv = fp8x2_fast(p.x, p.y, s, sinv) | (fp8x2_fast(p.z, p.w, s, sinv) << 16);
          d0 = __fmul_rn(fp8_val(wv), s); d1 = __fmul_rn(fp8_val(wv >> 8), s);
          d2 = __fmul_rn(fp8_val(wv >> 16), s); d3 = __fmul_rn(fp8_val(wv >> 24), s);
        } else if constexpr (SR) {
          const uint64_t h0 = qsgd_h(srb, 2 * q), h1 = qsgd_h(srb, 2 * q + 1);   // elements 4q .. 4q+3
          int q0 = qsgd_q(p.x, s, qsgd_hi(h0)), q1 = qsgd_q(p.y, s, qsgd_lo(h0)),
              q2 = qsgd_q(p.z, s, qsgd_hi(h1)), q3 = qsgd_q(p.w, s, qsgd_lo(h1));
          wv = pack_i8x4(q0, q1, q2, q3);
          d0 = __fmul_rn((float)q0, s); d1 = __fmul_rn((float)q1, s); d2 = __fmul_rn((float)q2, s); d3 = __fmul_rn((float)q3, s);
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
          ce = fp8x2_of(p, 0.0f, s) & 0xFF;
          de = __fmul_rn(fp8_val(ce), s);
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
  else if constexpr (METHOD == M_FP8) return __fmul_rn(fp8_val(body[e]), s);
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
    return __fmul_rn(fp8_val(x >> (8 * (e & 3))), s);
  } else {
    return __fmul_rn((float)(int8_t)((x >> (8 * (e & 3))) & 0xFF), s);
  }
}

// out = fl(tree_sum / P).  For P a power of two, x * (1/P) is the same correctly rounded
// value as x / P (1/P is exact), so the multiply is used; otherwise IEEE division.
template <int P>
__device__ __forceinline__ float div_p(float x) {
  if constexpr ((P & (P - 1)) == 0) return __fmul_rn(x, 1.0f / (float)P);
  else return __fdiv_rn(x, (float)P);
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
        sc[k] = (METHOD == M_INT8 || METHOD == M_FP8) ? *reinterpret_cast<const float*>(src.p[k] + it.slot_off + k * it.pb + 8) : 1.0f;
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
constexpr int kFusedThreads = 512;
constexpr int kFusedUnroll = 2;   // (lag 2 is the default LAG template argument of the variants below)

__device__ __forceinline__ void arrive(unsigned* done) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(done, 1u);
  }
}
__device__ __forceinline__ void wait_all(const unsigned* done, unsigned target) {
  if (threadIdx.x == 0) {
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(done) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

struct Slice {
  uint64_t q0, q1;
};
__device__ __forceinline__ Slice slice_of(uint64_t n4, unsigned G) {
  const uint64_t per = ((n4 + G - 1) / G + 3) & ~uint64_t(3);   // 4-quad aligned (16-B pushes)
  const uint64_t q0 = min(n4, (uint64_t)blockIdx.x * per);
  return Slice{q0, min(n4, q0 + per)};
}

// PARK: phase A stores p into r and B re-reads p (4 B); otherwise A only reads g and r with
// L2 evict_last and B re-reads both and recomputes p = g + r (same binary32 addition, so
// bit-identical) — clean lines, nothing to write back.  LAG: B(t - LAG) runs with A(t).
template <bool EF, bool VEC, bool PARK, int LAG, int NT = kFusedThreads, int UNR = kFusedUnroll, int MINB = 2>
__global__ void __launch_bounds__(NT, MINB)
    k_int8_fused(const Item* __restrict__ items, int nitems, const float* __restrict__ gbase,
                 float* __restrict__ rbase, Dests dst, uint32_t* scratch, uint32_t* flags,
                 unsigned* done) {
  __shared__ uint32_t s_red[NT / 32];
  const unsigned G = gridDim.x;
  const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
  for (int t = 0; t < nitems + LAG; ++t) {
    const int ia = t, ib = t - LAG;
    const bool doA = ia < nitems;
    bool doB = ib >= 0;
    // ---- B setup (wait for everyone's A(ib), finished an iteration ago)
    Item itB{};
    Slice sb{0, 0};
    float s = 1.0f, sinv = 1.0f;
    if (doB) {
      itB = items[ib];
      wait_all(&done[ib], G);
      const uint32_t mbits = *((volatile const uint32_t*)&scratch[itB.sidx]);
      if (nonfinite_bits(mbits)) {   // all-or-nothing: no payload for this bucket
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(flags, kFlagNonfinite);
        doB = false;
      } else {
        s = int8_scale_from_bits(mbits);
        sinv = int8_inv(s);
        sb = slice_of(itB.n >> 2, G);
        if (blockIdx.x == 0 && threadIdx.x == 0) put_preamble(dst, itB.slot_off, M_INT8, (uint32_t)itB.n, s, 0u);
      }
    }
    // ---- A setup
    Item itA{};
    Slice sa{0, 0};
    if (doA) {
      itA = items[ia];
      sa = slice_of(itA.n >> 2, G);
    }
    const float* gA = gbase + itA.g_off;
    float* rA = rbase + itA.r_off;
    const float* gB = gbase + itB.g_off;
    float* rB = rbase + itB.r_off;
    const uint64_t boB = itB.slot_off + 16;
    uint32_t* bodyB = reinterpret_cast<uint32_t*>(dst.p[0] + boB);
    const uint64_t lenA = sa.q1 - sa.q0, lenB = doB ? sb.q1 - sb.q0 : 0;
    const uint64_t len = max(lenA, lenB);
    uint32_t m = 0;
    // block-uniform trip count (the lane-group pushes below use full-warp shuffles)
    for (uint64_t kb0 = 0; kb0 < len; kb0 += (uint64_t)NT * UNR) {
      const uint64_t kb = kb0 + threadIdx.x;
      float4 ga[UNR], ra[UNR], pb[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const uint64_t k = kb + (uint64_t)u * NT;
        if (k < lenA) {
          const uint64_t q = sa.q0 + k;
          const uint64_t polA = PARK ? pol_stream : pol_keep;
          if constexpr (VEC) ga[u] = ld4_hint(gA + 4 * q, polA);
          else ga[u] = ldq<false>(gA, q);
          if constexpr (EF) ra[u] = ld4_hint(rA + 4 * q, polA);
        }
        if (k < lenB) {
          const uint64_t q = sb.q0 + k;
          if constexpr (EF && PARK) {
            pb[u] = ld4_hint(rB + 4 * q, pol_stream);
          } else if constexpr (EF) {
            const float4 gg = VEC ? ld4_hint(gB + 4 * q, pol_stream) : ldq<false>(gB, q);
            pb[u] = add4(gg, ld4_hint(rB + 4 * q, pol_stream));
          } else {
            pb[u] = ldq<VEC>(gB, q);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const uint64_t k = kb + (uint64_t)u * NT;
        if (k < lenA) {
          const uint64_t q = sa.q0 + k;
          const float4 p = EF ? add4(ga[u], ra[u]) : ga[u];
          m = max(m, max(max(abs_bits(p.x), abs_bits(p.y)), max(abs_bits(p.z), abs_bits(p.w))));
          if constexpr (EF && PARK) st4_hint(rA + 4 * q, p, pol_keep);   // parked for B(t + LAG)
        }
        uint32_t w = 0u;
        if (k < lenB) {
          const uint64_t q = sb.q0 + k;
          const float4 p = pb[u];
          const int a0 = int8_qi(p.x, s, sinv), a1 = int8_qi(p.y, s, sinv), a2 = int8_qi(p.z, s, sinv), a3 = int8_qi(p.w, s, sinv);
          w = pack_i8x4(a0, a1, a2, a3);
          st_u32_hint(bodyB + q, w, pol_stream);
          if constexpr (EF)
            st4_hint(rB + 4 * q,
                     make_float4(__fsub_rn(p.x, __fmul_rn((float)a0, s)), __fsub_rn(p.y, __fmul_rn((float)a1, s)),
                                 __fsub_rn(p.z, __fmul_rn((float)a2, s)), __fsub_rn(p.w, __fmul_rn((float)a3, s))),
                     pol_stream);
        }
        push_u32(dst, boB + 4 * (sb.q0 + k), w, k < lenB);   // NVLink push, 16 B per lane group
      }
    }
    // ---- tails (n % 4 elements after the last quad) on the last CTA
    if (blockIdx.x == G - 1) {
      if (doA && threadIdx.x < (itA.n & 3)) {
        const uint64_t e = (itA.n >> 2) * 4 + threadIdx.x;
        const float p = EF ? __fadd_rn(gA[e], rA[e]) : gA[e];
        if constexpr (EF && PARK) rA[e] = p;
        m = max(m, abs_bits(p));
      }
      if (doB) {
        if (threadIdx.x < (itB.n & 3)) {
          const uint64_t e = (itB.n >> 2) * 4 + threadIdx.x;
          const float p = EF ? (PARK ? rB[e] : __fadd_rn(gB[e], rB[e])) : gB[e];
          const int qe = int8_qi(p, s, sinv);
          put(dst, boB + e, (uint8_t)(qe & 0xFF));
          if constexpr (EF) rB[e] = __fsub_rn(p, __fmul_rn((float)qe, s));
        }
        zero_padding(dst, boB, itB.n);
      }
    }
    // ---- A epilogue: bucket max, arrive
    if (doA) {
      m = __reduce_max_sync(0xFFFFFFFFu, m);
      if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = m;
      __syncthreads();
      if (threadIdx.x < 32) {
        uint32_t w = threadIdx.x < NT / 32 ? s_red[threadIdx.x] : 0u;
        w = __reduce_max_sync(0xFFFFFFFFu, w);
        if (threadIdx.x == 0 && w) atomicMax(&scratch[itA.sidx], w);
      }
      arrive(&done[ia]);
    }
    __syncthreads();
  }
  if (dst.n > 1) __threadfence_system();
}

// ----------------------------------------------------------------------------- launchers
int occupancy_per_sm(const void* kernel, int threads, size_t smem) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(kernel);
  if (it != cache.end()) return it->second;
  int per = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem) != cudaSuccess || per < 1) per = 1;
  cache[kernel] = per;
  return per;
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

void launch_fp8_quant(const Launch& L, bool ef, bool vec, const Item* items, int nitems, uint64_t chunks,
                      const float* g, float* r, const Dests& slots, const uint32_t* scratch, uint32_t* flags) {
  if (!chunks) return;
  Mark mk(L, PH_FP8_QUANT);
  if (ef && vec) k_int8_quant<true, true, true><<<GRID((k_int8_quant<true, true, true>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, slots, scratch, flags);
  else if (ef) k_int8_quant<true, false, true><<<GRID((k_int8_quant<true, false, true>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, slots, scratch, flags);
  else if (vec) k_int8_quant<false, true, true><<<GRID((k_int8_quant<false, true, true>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, slots, scratch, flags);
  else k_int8_quant<false, false, true><<<GRID((k_int8_quant<false, false, true>)), kThreads, 0, L.stream>>>(items, nitems, chunks, g, r, slots, scratch, flags);
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
  else reduce_m<M_INT8>(L, P, vec, items, nitems, chunks, slots, out);   // INT8 and QSGD: same decode
  ++*L.launches;
}

// Split schedule (default): each iteration runs A(t) over the CTA's slice, ARRIVES, then runs
// B(t-1).  B(t-1) waits for everyone's A(t-1), which they finished before their own B(t-2),
// i.e. a whole B phase ago — the wait rarely stalls, yet only two buckets of p are ever parked
// in L2 (measured: DRAM traffic equals the algorithmic 13 B/elem, no dirty write-back).
template <bool EF, bool VEC>
__global__ void __launch_bounds__(kFusedThreads, 2)
    k_int8_fused_split(const Item* __restrict__ items, int nitems, const float* __restrict__ gbase,
                       float* __restrict__ rbase, Dests dst, uint32_t* scratch, uint32_t* flags, unsigned* done) {
  constexpr int U = 4;
  __shared__ uint32_t s_red[kFusedThreads / 32];
  const unsigned G = gridDim.x;
  const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
  for (int t = 0; t <= nitems; ++t) {
    if (t < nitems) {   // ---------------- A(t): p = g + r -> parked in r, bucket max, arrive
      const Item it = items[t];
      const Slice sa = slice_of(it.n >> 2, G);
      const uint64_t len = sa.q1 - sa.q0;
      const float* g = gbase + it.g_off;
      float* r = rbase + it.r_off;
      uint32_t m = 0;
      for (uint64_t k0 = 0; k0 < len; k0 += (uint64_t)kFusedThreads * U) {
        float4 gv[U], rv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t k = k0 + (uint64_t)u * kFusedThreads + threadIdx.x;
          if (k < len) {
            const uint64_t q = sa.q0 + k;
            if constexpr (VEC) gv[u] = ld4_hint(g + 4 * q, pol_stream);
            else gv[u] = ldq<false>(g, q);
            if constexpr (EF) rv[u] = ld4_hint(r + 4 * q, pol_stream);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t k = k0 + (uint64_t)u * kFusedThreads + threadIdx.x;
          if (k < len) {
            const uint64_t q = sa.q0 + k;
            const float4 p = EF ? add4(gv[u], rv[u]) : gv[u];
            m = max(m, max(max(abs_bits(p.x), abs_bits(p.y)), max(abs_bits(p.z), abs_bits(p.w))));
            if constexpr (EF) st4_hint(r + 4 * q, p, pol_keep);
          }
        }
      }
      if (blockIdx.x == G - 1 && threadIdx.x < (it.n & 3)) {
        const uint64_t e = (it.n >> 2) * 4 + threadIdx.x;
        const float p = EF ? __fadd_rn(g[e], r[e]) : g[e];
        if constexpr (EF) r[e] = p;
        m = max(m, abs_bits(p));
      }
      m = __reduce_max_sync(0xFFFFFFFFu, m);
      if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = m;
      __syncthreads();
      if (threadIdx.x < 32) {
        uint32_t w = threadIdx.x < kFusedThreads / 32 ? s_red[threadIdx.x] : 0u;
        w = __reduce_max_sync(0xFFFFFFFFu, w);
        if (threadIdx.x == 0 && w) atomicMax(&scratch[it.sidx], w);
      }
      arrive(&done[t]);
    }
    if (t >= 1) {       // ---------------- B(t-1): quantise from the parked p
      const Item it = items[t - 1];
      wait_all(&done[t - 1], G);
      const uint32_t mbits = *((volatile const uint32_t*)&scratch[it.sidx]);
      if (nonfinite_bits(mbits)) {   // all-or-nothing: no payload for this bucket
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(flags, kFlagNonfinite);
        continue;
      }
      const float s = int8_scale_from_bits(mbits);
      const float sinv = int8_inv(s);
      const Slice sb = slice_of(it.n >> 2, G);
      const uint64_t len = sb.q1 - sb.q0;
      const float* g = gbase + it.g_off;
      float* r = rbase + it.r_off;
      const uint64_t bo = it.slot_off + 16;
      uint32_t* body = reinterpret_cast<uint32_t*>(dst.p[0] + bo);
      if (blockIdx.x == 0 && threadIdx.x == 0) put_preamble(dst, it.slot_off, M_INT8, (uint32_t)it.n, s, 0u);
      for (uint64_t k0 = 0; k0 < len; k0 += (uint64_t)kFusedThreads * U) {
        float4 pv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t k = k0 + (uint64_t)u * kFusedThreads + threadIdx.x;
          if (k < len) {
            const uint64_t q = sb.q0 + k;
            pv[u] = EF ? ld4_hint(r + 4 * q, pol_stream) : ldq<VEC>(g, q);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t k = k0 + (uint64_t)u * kFusedThreads + threadIdx.x;
          uint32_t w = 0u;
          if (k < len) {
            const uint64_t q = sb.q0 + k;
            const float4 p = pv[u];
            const int a0 = int8_qi(p.x, s, sinv), a1 = int8_qi(p.y, s, sinv), a2 = int8_qi(p.z, s, sinv), a3 = int8_qi(p.w, s, sinv);
            w = pack_i8x4(a0, a1, a2, a3);
            st_u32_hint(body + q, w, pol_stream);
            if constexpr (EF)
              st4_hint(r + 4 * q,
                       make_float4(__fsub_rn(p.x, __fmul_rn((float)a0, s)), __fsub_rn(p.y, __fmul_rn((float)a1, s)),
                                   __fsub_rn(p.z, __fmul_rn((float)a2, s)), __fsub_rn(p.w, __fmul_rn((float)a3, s))),
                       pol_stream);
          }
          push_u32(dst, bo + 4 * (sb.q0 + k), w, k < len);   // P2P push (no-op otherwise)
        }
      }
      if (blockIdx.x == G - 1) {
        if (threadIdx.x < (it.n & 3)) {
          const uint64_t e = (it.n >> 2) * 4 + threadIdx.x;
          const float p = EF ? r[e] : g[e];
          const int qe = int8_qi(p, s, sinv);
          put(dst, bo + e, (uint8_t)(qe & 0xFF));
          if constexpr (EF) r[e] = __fsub_rn(p, __fmul_rn((float)qe, s));
        }
        zero_padding(dst, bo, it.n);
      }
      __syncthreads();
    }
  }
  if (dst.n > 1) __threadfence_system();
}

// Lag-2 interleave with alternating parking (variant 5): even buckets park p in SHARED MEMORY
// (the first cap4 quads of the CTA's slice; B(t-2) reads slot k and A(t) overwrites it in the
// same thread, same loop trip), odd buckets park p in r / L2.  So at most one bucket's p sits
// in L2 at a time (the footprint that kept DRAM traffic at the algorithmic 13 B/elem) while
// the lag of two removes the per-bucket grid stall.  Slice overflow beyond cap4 parks in r.
template <bool EF, bool VEC>
__global__ void __launch_bounds__(kFusedThreads, 2)
    k_int8_fused_smem(const Item* __restrict__ items, int nitems, const float* __restrict__ gbase,
                      float* __restrict__ rbase, Dests dst, uint32_t* scratch, uint32_t* flags, unsigned* done,
                      uint32_t cap4) {
  constexpr int U = 2;
  extern __shared__ float4 sp[];
  __shared__ uint32_t s_red[kFusedThreads / 32];
  const unsigned G = gridDim.x;
  const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
  for (int t = 0; t < nitems + 2; ++t) {
    const int ia = t, ib = t - 2;
    const bool doA = ia < nitems;
    bool doB = ib >= 0;
    Item itB{};
    Slice sb{0, 0};
    float s = 1.0f, sinv = 1.0f;
    if (doB) {
      itB = items[ib];
      wait_all(&done[ib], G);
      const uint32_t mbits = *((volatile const uint32_t*)&scratch[itB.sidx]);
      if (nonfinite_bits(mbits)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(flags, kFlagNonfinite);
        doB = false;
      } else {
        s = int8_scale_from_bits(mbits);
        sinv = int8_inv(s);
        sb = slice_of(itB.n >> 2, G);
        if (blockIdx.x == 0 && threadIdx.x == 0) put_preamble(dst, itB.slot_off, M_INT8, (uint32_t)itB.n, s, 0u);
      }
    }
    Item itA{};
    Slice sa{0, 0};
    if (doA) {
      itA = items[ia];
      sa = slice_of(itA.n >> 2, G);
    }
    const bool a_smem = EF && ((ia & 1) == 0), b_smem = EF && ((ib & 1) == 0);
    const float* gA = gbase + itA.g_off;
    float* rA = rbase + itA.r_off;
    const float* gB = gbase + itB.g_off;
    float* rB = rbase + itB.r_off;
    const uint64_t boB = itB.slot_off + 16;
    uint32_t* bodyB = reinterpret_cast<uint32_t*>(dst.p[0] + boB);
    const uint64_t lenA = sa.q1 - sa.q0, lenB = doB ? sb.q1 - sb.q0 : 0;
    const uint64_t len = max(lenA, lenB);
    uint32_t m = 0;
    for (uint64_t kb0 = 0; kb0 < len; kb0 += (uint64_t)kFusedThreads * U) {
      float4 ga[U], ra[U], pb[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t k = kb0 + (uint64_t)u * kFusedThreads + threadIdx.x;
        if (k < lenB) {   // B's p first: its shared-memory slot is overwritten by A below
          const uint64_t q = sb.q0 + k;
          if constexpr (EF) pb[u] = (b_smem && k < cap4) ? sp[k] : ld4_hint(rB + 4 * q, pol_stream);
          else pb[u] = ldq<VEC>(gB, q);
        }
        if (k < lenA) {
          const uint64_t q = sa.q0 + k;
          if constexpr (VEC) ga[u] = ld4_hint(gA + 4 * q, pol_stream);
          else ga[u] = ldq<false>(gA, q);
          if constexpr (EF) ra[u] = ld4_hint(rA + 4 * q, pol_stream);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t k = kb0 + (uint64_t)u * kFusedThreads + threadIdx.x;
        if (k < lenA) {
          const uint64_t q = sa.q0 + k;
          const float4 p = EF ? add4(ga[u], ra[u]) : ga[u];
          m = max(m, max(max(abs_bits(p.x), abs_bits(p.y)), max(abs_bits(p.z), abs_bits(p.w))));
          if constexpr (EF) {
            if (a_smem && k < cap4) sp[k] = p;
            else st4_hint(rA + 4 * q, p, pol_keep);
          }
        }
        uint32_t w = 0u;
        if (k < lenB) {
          const uint64_t q = sb.q0 + k;
          const float4 p = pb[u];
          const int a0 = int8_qi(p.x, s, sinv), a1 = int8_qi(p.y, s, sinv), a2 = int8_qi(p.z, s, sinv), a3 = int8_qi(p.w, s, sinv);
          w = pack_i8x4(a0, a1, a2, a3);
          st_u32_hint(bodyB + q, w, pol_stream);
          if constexpr (EF)
            st4_hint(rB + 4 * q,
                     make_float4(__fsub_rn(p.x, __fmul_rn((float)a0, s)), __fsub_rn(p.y, __fmul_rn((float)a1, s)),
                                 __fsub_rn(p.z, __fmul_rn((float)a2, s)), __fsub_rn(p.w, __fmul_rn((float)a3, s))),
                     pol_stream);
        }
        push_u32(dst, boB + 4 * (sb.q0 + k), w, k < lenB);
      }
    }
    if (blockIdx.x == G - 1) {
      if (doA && threadIdx.x < (itA.n & 3)) {   // tail elements park in r (never in smem)
        const uint64_t e = (itA.n >> 2) * 4 + threadIdx.x;
        const float p = EF ? __fadd_rn(gA[e], rA[e]) : gA[e];
        if constexpr (EF) rA[e] = p;
        m = max(m, abs_bits(p));
      }
      if (doB) {
        if (threadIdx.x < (itB.n & 3)) {
          const uint64_t e = (itB.n >> 2) * 4 + threadIdx.x;
          const float p = EF ? rB[e] : gB[e];
          const int qe = int8_qi(p, s, sinv);
          put(dst, boB + e, (uint8_t)(qe & 0xFF));
          if constexpr (EF) rB[e] = __fsub_rn(p, __fmul_rn((float)qe, s));
        }
        zero_padding(dst, boB, itB.n);
      }
    }
    if (doA) {
      m = __reduce_max_sync(0xFFFFFFFFu, m);
      if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = m;
      __syncthreads();
      if (threadIdx.x < 32) {
        uint32_t w = threadIdx.x < kFusedThreads / 32 ? s_red[threadIdx.x] : 0u;
        w = __reduce_max_sync(0xFFFFFFFFu, w);
        if (threadIdx.x == 0 && w) atomicMax(&scratch[itA.sidx], w);
      }
      arrive(&done[ia]);
    }
    __syncthreads();
  }
  if (dst.n > 1) __threadfence_system();
}

// ----------------------------------------------------------------------------- INT8 TMA
// Fused INT8 with TMA staging (variant 9, the default): one CTA per SM streams its slice of
// every bucket through a 4-stage shared-memory ring filled by cp.async.bulk (TMA bulk copies
// completing on an mbarrier transaction count).  A ring stage holds, for tile k of the
// iteration, the g and r tiles of bucket t (phase A) and the parked-p tile of bucket t-1
// (phase B); up to 4 tiles (192 KB) are in flight per SM no matter what the warps are doing.
// Same lag-1 split barrier as k_int8_fused: A(t) parks p in r (L2 evict_last), B(t-1)
// quantises from it; the wait for bucket t-1's max is taken after the first tiles' copies
// were issued.  Stores stay ordinary st.global (they are posted).
constexpr int kTmaThreads = 1024;
constexpr int kTmaTQ = 1024;   // quads per tile: 16 KB per stream
constexpr int kTmaNS = 4;      // ring stages

struct __align__(128) TmaStage {
  float4 g[kTmaTQ];
  float4 r[kTmaTQ];
  float4 p[kTmaTQ];
};

__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n}\n" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      :: "r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}

struct TmaTiles {          // tile geometry of one iteration (identical in every thread)
  uint64_t qa0, lenA, qb0, lenB;
  int ntA, ntB, nt;
};

template <bool EF>
__device__ __forceinline__ void tma_issue(TmaStage* stg, uint64_t* bar, int k, const TmaTiles& T, const float* gA,
                                          const float* rA, const float* srcB, uint64_t pol_stream, uint64_t pol_keep) {
  const int sidx = k % kTmaNS;
  uint32_t bytes = 0;
  uint32_t nqa = 0, nqb = 0;
  if (k < T.ntA) nqa = (uint32_t)min((uint64_t)kTmaTQ, T.lenA - (uint64_t)k * kTmaTQ);
  if (k < T.ntB) nqb = (uint32_t)min((uint64_t)kTmaTQ, T.lenB - (uint64_t)k * kTmaTQ);
  bytes = nqa * (EF ? 32u : 16u) + nqb * 16u;
  if (!bytes) return;
  mbar_expect_tx(&bar[sidx], bytes);
  if (nqa) {
    const uint64_t q = T.qa0 + (uint64_t)k * kTmaTQ;
    bulk_g2s(stg[sidx].g, gA + 4 * q, nqa * 16u, &bar[sidx], pol_stream);
    if (EF) bulk_g2s(stg[sidx].r, rA + 4 * q, nqa * 16u, &bar[sidx], pol_stream);
  }
  if (nqb) {
    const uint64_t q = T.qb0 + (uint64_t)k * kTmaTQ;
    bulk_g2s(stg[sidx].p, srcB + 4 * q, nqb * 16u, &bar[sidx], pol_stream);
  }
}

template <bool EF>
__global__ void __launch_bounds__(kTmaThreads, 1)
    k_int8_tma(const Item* __restrict__ items, int nitems, const float* __restrict__ gbase, float* __restrict__ rbase,
               Dests dst, uint32_t* scratch, uint32_t* flags, unsigned* done) {
  extern __shared__ __align__(128) unsigned char tma_smem[];
  TmaStage* stg = reinterpret_cast<TmaStage*>(tma_smem);
  __shared__ __align__(8) uint64_t bar[kTmaNS];     // full: TMA bytes landed
  __shared__ __align__(8) uint64_t empty[kTmaNS];   // empty: every warp finished reading the stage
  __shared__ uint32_t s_red[kTmaThreads / 32];
  const unsigned G = gridDim.x;
  const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
  if (threadIdx.x == 0) {
    for (int i = 0; i < kTmaNS; ++i) {
      mbar_init(&bar[i], 1);
      mbar_init(&empty[i], kTmaThreads / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase = 0;                 // full-barrier parity per ring stage (every thread)
  uint32_t ephase = 0, filled = 0;    // producer (thread 0): empty parity, stages holding an unreleased fill
  // producer: (re)fill the stage of tile k once its previous contents were released
  auto refill = [&](int k, const TmaTiles& T, const float* gA, const float* rA, const float* srcB) {
    const int sidx = k % kTmaNS;
    if (filled & (1u << sidx)) {
      mbar_wait(&empty[sidx], (ephase >> sidx) & 1u);
      ephase ^= 1u << sidx;
    }
    filled |= 1u << sidx;
    tma_issue<EF>(stg, bar, k, T, gA, rA, srcB, pol_stream, pol_keep);
  };
  for (int t = 0; t <= nitems; ++t) {
    const bool doA = t < nitems;
    bool doB = t >= 1;
    Item itA{}, itB{};
    TmaTiles T{};
    if (doA) {
      itA = items[t];
      const Slice sa = slice_of(itA.n >> 2, G);
      T.qa0 = sa.q0;
      T.lenA = sa.q1 - sa.q0;
    }
    if (doB) {
      itB = items[t - 1];
      const Slice sb = slice_of(itB.n >> 2, G);
      T.qb0 = sb.q0;
      T.lenB = sb.q1 - sb.q0;
    }
    T.ntA = (int)((T.lenA + kTmaTQ - 1) / kTmaTQ);
    T.ntB = (int)((T.lenB + kTmaTQ - 1) / kTmaTQ);
    T.nt = max(T.ntA, T.ntB);
    const float* gA = gbase + itA.g_off;
    float* rA = rbase + itA.r_off;
    const float* gB = gbase + itB.g_off;
    float* rB = rbase + itB.r_off;
    const float* srcB = EF ? rB : gB;
    // prologue: the first ring-full of tiles is in flight before the barrier wait below
    if (threadIdx.x == 0)
      for (int k = 0; k < min(T.nt, kTmaNS); ++k) refill(k, T, gA, rA, srcB);
    float s = 1.0f, sinv = 1.0f;
    const uint64_t boB = itB.slot_off + 16;
    uint32_t* bodyB = reinterpret_cast<uint32_t*>(dst.p[0] + boB);
    if (doB) {
      wait_all(&done[t - 1], G);
      const uint32_t mbits = *((volatile const uint32_t*)&scratch[itB.sidx]);
      if (nonfinite_bits(mbits)) {   // all-or-nothing: no payload for this bucket
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(flags, kFlagNonfinite);
        doB = false;
      } else {
        s = int8_scale_from_bits(mbits);
        sinv = int8_inv(s);
        if (blockIdx.x == 0 && threadIdx.x == 0) put_preamble(dst, itB.slot_off, M_INT8, (uint32_t)itB.n, s, 0u);
      }
    }
    uint32_t m = 0;
    for (int k = 0; k < T.nt; ++k) {
      const int sidx = k % kTmaNS;
      mbar_wait(&bar[sidx], (phase >> sidx) & 1u);
      phase ^= 1u << sidx;
      const TmaStage& S = stg[sidx];
      const uint32_t nqa = k < T.ntA ? (uint32_t)min((uint64_t)kTmaTQ, T.lenA - (uint64_t)k * kTmaTQ) : 0u;
      const uint32_t nqb = k < T.ntB ? (uint32_t)min((uint64_t)kTmaTQ, T.lenB - (uint64_t)k * kTmaTQ) : 0u;
#pragma unroll
      for (int u = 0; u < kTmaTQ / kTmaThreads; ++u) {
        const uint32_t j = u * kTmaThreads + threadIdx.x;
        if (j < nqa) {
          const uint64_t q = T.qa0 + (uint64_t)k * kTmaTQ + j;
          const float4 p = EF ? add4(S.g[j], S.r[j]) : S.g[j];
          m = max(m, max(max(abs_bits(p.x), abs_bits(p.y)), max(abs_bits(p.z), abs_bits(p.w))));
          if constexpr (EF) st4_hint(rA + 4 * q, p, pol_keep);   // parked for B(t) next iteration
        }
        uint32_t w = 0u;
        const uint64_t qb = T.qb0 + (uint64_t)k * kTmaTQ + j;
        if (doB && j < nqb) {
          const float4 p = S.p[j];
          const int a0 = int8_qi(p.x, s, sinv), a1 = int8_qi(p.y, s, sinv), a2 = int8_qi(p.z, s, sinv),
                    a3 = int8_qi(p.w, s, sinv);
          w = pack_i8x4(a0, a1, a2, a3);
          st_u32_hint(bodyB + qb, w, pol_stream);
          if constexpr (EF)
            st4_hint(rB + 4 * qb,
                     make_float4(__fsub_rn(p.x, __fmul_rn((float)a0, s)), __fsub_rn(p.y, __fmul_rn((float)a1, s)),
                                 __fsub_rn(p.z, __fmul_rn((float)a2, s)), __fsub_rn(p.w, __fmul_rn((float)a3, s))),
                     pol_stream);
        }
        push_u32(dst, boB + 4 * qb, w, doB && j < nqb);
      }
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[sidx]);   // this warp is done with the stage
      if (threadIdx.x == 0 && k + kTmaNS < T.nt) refill(k + kTmaNS, T, gA, rA, srcB);
    }
    // tails (n % 4 elements after the last quad) on the last CTA
    if (blockIdx.x == G - 1) {
      if (doA && threadIdx.x < (itA.n & 3)) {
        const uint64_t e = (itA.n >> 2) * 4 + threadIdx.x;
        const float p = EF ? __fadd_rn(gA[e], rA[e]) : gA[e];
        if constexpr (EF) rA[e] = p;
        m = max(m, abs_bits(p));
      }
      if (doB) {
        if (threadIdx.x < (itB.n & 3)) {
          const uint64_t e = (itB.n >> 2) * 4 + threadIdx.x;
          const float p = EF ? rB[e] : gB[e];
          const int qe = int8_qi(p, s, sinv);
          put(dst, boB + e, (uint8_t)(qe & 0xFF));
          if constexpr (EF) rB[e] = __fsub_rn(p, __fmul_rn((float)qe, s));
        }
        zero_padding(dst, boB, itB.n);
      }
    }
    // the parked p must be visible to next iteration's bulk copies (async proxy)
    asm volatile("fence.proxy.async.global;" ::: "memory");
    if (doA) {
      m = __reduce_max_sync(0xFFFFFFFFu, m);
      if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = m;
      __syncthreads();
      if (threadIdx.x < 32) {
        uint32_t w = threadIdx.x < kTmaThreads / 32 ? s_red[threadIdx.x] : 0u;
        w = __reduce_max_sync(0xFFFFFFFFu, w);
        if (threadIdx.x == 0 && w) atomicMax(&scratch[itA.sidx], w);
      }
      arrive(&done[t]);
    }
    __syncthreads();
  }
  if (dst.n > 1) __threadfence_system();
}

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
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
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
template <bool F8>
__device__ __forceinline__ float dec_byte(uint32_t byte, float s) {
  if constexpr (F8) return __fmul_rn(fp8_val(byte), s);
  else return __fmul_rn((float)(int8_t)(byte & 0xFF), s);
}

template <int P, bool F8 = false>
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
template <int P, bool F8 = false>
__device__ __forceinline__ void ws_reduce_ld(const StepArgs& a, int nb, int ct, int nC, float* s_sc,
                                               volatile uint32_t* s_abort, float* s_out, uint32_t* flags) {
  constexpr int E = 16, SROW = E + 1, U = P <= 2 ? 2 : 1;
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
        const unsigned long long t0 = globaltimer_ns();
        for (int c = 0; c < P && !*s_abort; ++c) {
          if (c == a.pe.me) continue;
          while (ld_acquire_sys(a.local_arrive + (size_t)(a.b0 + b) * P + c) < a.seq) {
            if (globaltimer_ns() - t0 > 60ull * 1000000000ull) {
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
        scb[k] = *reinterpret_cast<volatile const float*>(a.src.p[k] + it.slot_off + (uint64_t)k * it.pb + 8);
    }
    named_sync(3, nC);
    if (*s_abort) return;
    float sc[P];
#pragma unroll
    for (int k = 0; k < P; ++k) sc[k] = scb[k];
    const uint64_t n4 = it.n >> 2;
    const Slice sl = slice_of(n4, G);
    const uint64_t g0 = sl.q0 >> 2, g1 = sl.q1 >> 2;   // whole 16-element groups of this slice
    float* out = a.obase + it.out_off;
    auto slot = [&](int k, uint64_t gi) { return a.src.p[k] + it.slot_off + (uint64_t)k * it.pb + 16 + 16 * gi; };
    auto dec = [&](const uint4& x4, int e, float s) {
      const uint32_t x = (e >> 2) == 0 ? x4.x : (e >> 2) == 1 ? x4.y : (e >> 2) == 2 ? x4.z : x4.w;
      return dec_byte<F8>(x >> (8 * (e & 3)), s);
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
          const uint64_t gw0 = gb + u * 32;
#pragma unroll
          for (int v = 0; v < E / 4; ++v) {
            const int qq = v * 32 + lane, src_lane = qq >> 2, src_e = (qq & 3) * 4;
            if (gw0 + src_lane < g1) {
              const float* r = sw + src_lane * SROW + src_e;
              st4_hint(out + 4 * (gw0 * 4 + qq), make_float4(r[0], r[1], r[2], r[3]), pol);
            }
          }
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
#pragma unroll
        for (int v = 0; v < E / 4; ++v) {
          const int qq = v * 32 + lane, src_lane = qq >> 2, src_e = (qq & 3) * 4;
          if (gb + src_lane < g1) {
            const float* r = sw + src_lane * SROW + src_e;
            st4_hint(out + 4 * (gb * 4 + qq), make_float4(r[0], r[1], r[2], r[3]), pol);
          }
        }
        __syncwarp();
      }
    }
    // the < 16 elements after the last whole group of the bucket
    if (blockIdx.x == G - 1 && ct < 16) {
      const uint64_t e = 16 * (n4 >> 2) + ct;
      if (e < it.n) {
        float v[P];
#pragma unroll
        for (int k = 0; k < P; ++k) {
          const uint8_t q = *reinterpret_cast<volatile const uint8_t*>(a.src.p[k] + it.slot_off + (uint64_t)k * it.pb + 16 + e);
          v[k] = dec_byte<F8>(q, sc[k]);
        }
        out[e] = div_p<P>(tree_sum<0, P>(v));
      }
    }
  }
}

// CM: reduce role — 0 none (compress only), 1 TMA variant (LOOPBACK), 2 register loads (P2P pull)
// F8: the same schedules for the FP8 E4M3 codec (NEXT-4, R27) — only the B warps' scale /
// quantise / dequantise and the C warps' byte decode differ.
template <bool EF, int AW, int BW, int CW, int CM, bool F8 = false, bool SR = false>
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
            bulk_g2s(ringA[st].g, gbase + it.g_off + 4 * q, nq * 16u, &fullA[st], pol_stream);
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
        while (s_bdone < (uint32_t)(t - 1)) __nanosleep(64);   // B(t-2) finished: bounded L2 footprint
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
          const float sc = F8 ? fp8_scale_from_bits(mbits) : int8_scale_from_bits(mbits);
          s_scale[0] = sc;
          s_scale[1] = int8_inv(sc);
          if (blockIdx.x == 0) put_preamble(dst, it.slot_off, F8 ? M_FP8 : (SR ? M_QSGD : M_INT8), (uint32_t)it.n, sc, 0u);
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
              w = fp8x2_fast(p.x, p.y, s, sinv) | (fp8x2_fast(p.z, p.w, s, sinv) << 16);
              d0 = __fmul_rn(fp8_val(w), s); d1 = __fmul_rn(fp8_val(w >> 8), s);
              d2 = __fmul_rn(fp8_val(w >> 16), s); d3 = __fmul_rn(fp8_val(w >> 24), s);
            } else if constexpr (SR) {
              const uint64_t h0 = qsgd_h(srb, 2 * (q0 + j)), h1 = qsgd_h(srb, 2 * (q0 + j) + 1);
              const int a0 = qsgd_q(p.x, s, qsgd_hi(h0)), a1 = qsgd_q(p.y, s, qsgd_lo(h0)),
                        a2 = qsgd_q(p.z, s, qsgd_hi(h1)), a3 = qsgd_q(p.w, s, qsgd_lo(h1));
              w = pack_i8x4(a0, a1, a2, a3);
              d0 = __fmul_rn((float)a0, s); d1 = __fmul_rn((float)a1, s);
              d2 = __fmul_rn((float)a2, s); d3 = __fmul_rn((float)a3, s);
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
            ce = fp8x2_of(p, 0.0f, s) & 0xFF;
            de = __fmul_rn(fp8_val(ce), s);
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
              if (c != sa.pe.me) st_release_sys(sa.pe.arrive[c] + (size_t)(sa.b0 + t) * sa.pe.n + sa.pe.me, sa.seq);
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
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fp16_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_fp16_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  Mark mk(L, PH_FP16);
  const unsigned grid = (unsigned)std::min<uint64_t>(chunks, (uint64_t)L.num_sms);
  if (ef) k_fp16_tma<true><<<grid, kF16Threads, smem, L.stream>>>(items, nitems, chunks, g, r, slots, flags);
  else k_fp16_tma<false><<<grid, kF16Threads, smem, L.stream>>>(items, nitems, chunks, g, r, slots, flags);
  ++*L.launches;
  return true;
}

bool int8_onchip_capacity(int device, uint64_t* max_items, int* grid, size_t* smem) {
  int sms = 0, per_sm = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_int8_fused<true, true, true, 2>, kFusedThreads, 0) !=
          cudaSuccess || per_sm < 1)
    return false;
  const void* all[] = {(const void*)k_int8_fused<true, true, true, 2>, (const void*)k_int8_fused<true, false, true, 2>,
                       (const void*)k_int8_fused<false, true, true, 2>, (const void*)k_int8_fused<false, false, true, 2>,
                       (const void*)k_int8_fused<true, true, false, 2>, (const void*)k_int8_fused<true, true, true, 1>,
                       (const void*)k_int8_fused<true, true, false, 1>, (const void*)k_int8_fused_split<true, true>,
                       (const void*)k_int8_fused_split<true, false>, (const void*)k_int8_fused_split<false, true>,
                       (const void*)k_int8_fused_split<false, false>};
  // (the NT/UNR sweep variants 6..8 size their own grids at launch)
  for (const void* f : all) {
    int p2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p2, f, kFusedThreads, 0);
    per_sm = std::min(per_sm, std::max(1, p2));
  }
  *grid = sms * std::min(per_sm, 2);
  *max_items = 0;
  // shared-memory parking for variant 5: as much as two CTAs per SM can hold
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  size_t bytes = std::min<size_t>((size_t)optin, 100 * 1024);
  const void* sk[] = {(const void*)k_int8_fused_smem<true, true>, (const void*)k_int8_fused_smem<true, false>,
                      (const void*)k_int8_fused_smem<false, true>, (const void*)k_int8_fused_smem<false, false>};
  for (;;) {
    bool ok = true;
    for (const void* f : sk) ok &= cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess;
    int occ = 0;
    if (ok) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_int8_fused_smem<true, true>, kFusedThreads, bytes);
    if (ok && occ >= std::min(per_sm, 2)) break;
    if (bytes <= 16 * 1024) { bytes = 0; break; }
    bytes -= 8 * 1024;
  }
  cudaGetLastError();
  *smem = bytes;
  return true;
}

void launch_ws_compress(const Launch& L, bool ef, int kind, const Item* items, int nitems, const float* g, float* r,
                        const Dests& slots_in, uint32_t* scratch, uint32_t* flags, uint32_t* done_words,
                        const SrArgs& srargs) {
  Dests slots = slots_in;
  Mark mk(L, kind == 2 ? PH_QSGD_QUANT : PH_FP8_QUANT);
  cudaMemsetAsync(done_words, 0, sizeof(unsigned) * (size_t)nitems, L.stream);
  unsigned* done = done_words;
  StepArgs sa{};
  sa.sr = srargs;
  void* args[] = {(void*)&items, (void*)&nitems, (void*)&g, (void*)&r, (void*)&slots, (void*)&scratch,
                  (void*)&flags, (void*)&done, (void*)&sa};
  const void* f = kind == 2 ? (ef ? (const void*)k_int8_ws<true, 8, 23, 0, 0, false, true>
                                  : (const void*)k_int8_ws<false, 8, 23, 0, 0, false, true>)
                            : (ef ? (const void*)k_int8_ws<true, 8, 23, 0, 0, true>
                                  : (const void*)k_int8_ws<false, 8, 23, 0, 0, true>);
  const size_t smem = sizeof(WsStageA) * kWsNA + sizeof(WsStageB) * kWsNB;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_int8_ws<true, 8, 23, 0, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_int8_ws<false, 8, 23, 0, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_int8_ws<true, 8, 23, 0, 0, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_int8_ws<false, 8, 23, 0, 0, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaLaunchCooperativeKernel(f, dim3(sms), dim3(kWsThreads), args, smem, L.stream);
  ++*L.launches;
}

void launch_int8_onchip(const Launch& L, bool ef, bool vec, const Item* items, int nitems, const float* g, float* r,
                        const Dests& slots_in, uint32_t* scratch, uint32_t* flags, uint32_t* done_words, int grid,
                        size_t smem_bytes, int variant) {
  Dests slots = slots_in;
  if (variant == 5 && smem_bytes >= 16 * 1024) {
    Mark mk(L, PH_INT8_ONCHIP);
    cudaMemsetAsync(done_words, 0, sizeof(unsigned) * (size_t)nitems, L.stream);
    unsigned* done = done_words;
    uint32_t cap4 = (uint32_t)(smem_bytes / 16);
    void* args[] = {(void*)&items, (void*)&nitems, (void*)&g, (void*)&r, (void*)&slots, (void*)&scratch,
                    (void*)&flags, (void*)&done, (void*)&cap4};
    const void* f = ef ? (vec ? (const void*)k_int8_fused_smem<true, true> : (const void*)k_int8_fused_smem<true, false>)
                       : (vec ? (const void*)k_int8_fused_smem<false, true> : (const void*)k_int8_fused_smem<false, false>);
    cudaLaunchCooperativeKernel(f, dim3(grid), dim3(kFusedThreads), args, smem_bytes, L.stream);
    ++*L.launches;
    return;
  }
  if (variant == 10 && vec) {   // warp-specialised TMA kernel: one CTA per SM
    Mark mk(L, PH_INT8_ONCHIP);
    cudaMemsetAsync(done_words, 0, sizeof(unsigned) * (size_t)nitems, L.stream);
    unsigned* done = done_words;
    StepArgs sa{};
    void* args[] = {(void*)&items, (void*)&nitems, (void*)&g, (void*)&r, (void*)&slots, (void*)&scratch,
                    (void*)&flags, (void*)&done, (void*)&sa};
    const void* f = ef ? (const void*)k_int8_ws<true, 8, 23, 0, 0> : (const void*)k_int8_ws<false, 8, 23, 0, 0>;
    const size_t smem = sizeof(WsStageA) * kWsNA + sizeof(WsStageB) * kWsNB;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_int8_ws<true, 8, 23, 0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(k_int8_ws<false, 8, 23, 0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaLaunchCooperativeKernel(f, dim3(sms), dim3(kWsThreads), args, smem, L.stream);
    ++*L.launches;
    return;
  }
  if (variant == 10) variant = 2;
  if (variant == 9 && vec) {   // TMA-staged fused kernel: one CTA per SM
    Mark mk(L, PH_INT8_ONCHIP);
    cudaMemsetAsync(done_words, 0, sizeof(unsigned) * (size_t)nitems, L.stream);
    unsigned* done = done_words;
    void* args[] = {(void*)&items, (void*)&nitems, (void*)&g, (void*)&r, (void*)&slots, (void*)&scratch,
                    (void*)&flags, (void*)&done};
    const void* f = ef ? (const void*)k_int8_tma<true> : (const void*)k_int8_tma<false>;
    const size_t smem = sizeof(TmaStage) * kTmaNS;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_int8_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(k_int8_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaLaunchCooperativeKernel(f, dim3(sms), dim3(kTmaThreads), args, smem, L.stream);
    ++*L.launches;
    return;
  }
  if (variant == 9) variant = 2;
  if (variant == 5) variant = 2;
  if (variant >= 6 && variant <= 8 && ef && vec) {   // shape sweep of the lag-1 park kernel
    Mark mk(L, PH_INT8_ONCHIP);
    cudaMemsetAsync(done_words, 0, sizeof(unsigned) * (size_t)nitems, L.stream);
    unsigned* done = done_words;
    void* args[] = {(void*)&items, (void*)&nitems, (void*)&g, (void*)&r, (void*)&slots, (void*)&scratch,
                    (void*)&flags, (void*)&done};
    const void* f = variant == 6 ? (const void*)k_int8_fused<true, true, true, 1, 256, 2, 4>
                  : variant == 7 ? (const void*)k_int8_fused<true, true, true, 1, 256, 4, 3>
                                 : (const void*)k_int8_fused<true, true, true, 1, 1024, 2, 1>;
    const int nt = variant == 8 ? 1024 : 256;
    int per = 0, sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, f, nt, 0);
    cudaLaunchCooperativeKernel(f, dim3(sms * std::max(1, per)), dim3(nt), args, 0, L.stream);
    ++*L.launches;
    return;
  }
  if (variant > 5) variant = 2;
  Mark mk(L, PH_INT8_ONCHIP);
  cudaMemsetAsync(done_words, 0, sizeof(unsigned) * (size_t)nitems, L.stream);
  unsigned* done = done_words;
  void* args[] = {(void*)&items, (void*)&nitems, (void*)&g, (void*)&r, (void*)&slots, (void*)&scratch,
                  (void*)&flags, (void*)&done};
  // variant: 0 park p / lag 2, 1 recompute / lag 2, 2 park / lag 1, 3 recompute / lag 1,
  // 4 split schedule (A(t), arrive, B(t-1)) — the default
  const void* f = ef ? (vec ? (const void*)k_int8_fused<true, true, true, 2> : (const void*)k_int8_fused<true, false, true, 2>)
                     : (vec ? (const void*)k_int8_fused<false, true, true, 2> : (const void*)k_int8_fused<false, false, true, 2>);
  if (ef && vec && variant == 1) f = (const void*)k_int8_fused<true, true, false, 2>;
  if (ef && vec && variant == 2) f = (const void*)k_int8_fused<true, true, true, 1>;
  if (ef && vec && variant == 3) f = (const void*)k_int8_fused<true, true, false, 1>;
  if (variant == 4)
    f = ef ? (vec ? (const void*)k_int8_fused_split<true, true> : (const void*)k_int8_fused_split<true, false>)
           : (vec ? (const void*)k_int8_fused_split<false, true> : (const void*)k_int8_fused_split<false, false>);
  cudaLaunchCooperativeKernel(f, dim3(grid), dim3(kFusedThreads), args, 0, L.stream);
  ++*L.launches;
}

// ----------------------------------------------------------------------------- INT8 step
// compress + exchange + decompress/average of an INT8 call in ONE cooperative kernel (the
// warp-specialised kernel with reduce warps).  bar_words: 2 * nitems words (done, bdone).
// Warp splits (A, B, C) of the fused step; config 0 is the default, the rest a tuning sweep.
template <bool EF>
static const void* step_kernel(int config, int kind) {
  if (kind == 1) return config == 4 ? (const void*)k_int8_ws<EF, 4, 16, 11, 2, true> : (const void*)k_int8_ws<EF, 8, 19, 4, 1, true>;
  if (kind == 2) {   // QSGD: the quantise warps are instruction-bound, config 1 gives them more warps
    if (config == 4) return (const void*)k_int8_ws<EF, 4, 16, 11, 2, false, true>;
    if (config == 1) return (const void*)k_int8_ws<EF, 5, 22, 4, 1, false, true>;
    return (const void*)k_int8_ws<EF, 8, 19, 4, 1, false, true>;
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
  static bool attr[3][2][11] = {};
  if (!attr[kind][ef][config < 0 || config > 10 ? 0 : config]) {
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr[kind][ef][config < 0 || config > 10 ? 0 : config] = true;
  }
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaLaunchCooperativeKernel(f, dim3(sms), dim3(kWsThreads), args, smem, L.stream);
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
    if (c != me) st_release_sys(pe.arrive[c] + (size_t)b * P + me, seq);
  }
  const unsigned long long t0 = globaltimer_ns();
  for (int x = threadIdx.x; x < total; x += blockDim.x) {
    const int b = lo + x / P, c = x % P;
    if (c == me) continue;
    while (ld_acquire_sys(local + (size_t)b * P + c) < seq) {
      if (globaltimer_ns() - t0 > 60ull * 1000000000ull) {
        atomicOr(flags, kFlagPeerTimeout);
        return;
      }
    }
  }
}

void launch_exchange_flags(const Launch& L, const Peers& pe, unsigned long long* local_arrive, int lo, int hi,
                           uint64_t seq, uint32_t* flags) {
  Mark mk(L, PH_P2P_FLAGS);
  k_exchange_flags<<<1, 256, 0, L.stream>>>(pe, local_arrive, lo, hi, (unsigned long long)seq, flags);
  ++*L.launches;
}

}  // namespace nb
