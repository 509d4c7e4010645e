// nebula_internal.cuh — types and device helpers shared by the library's kernels.
//
// Everything here is B200 (sm_100a) device code or plain host bookkeeping.  The CPU oracle
// (oracle/) shares nothing with this file.  Arithmetic rules:
// every fp32 operation on the codec path is an explicitly rounded intrinsic
// (__fadd_rn/__fsub_rn/__fmul_rn/__fdiv_rn), so no FMA contraction can change a bit
// (contraction breaks the residual identity on ~5% of elements), and
// the library is compiled without --use_fast_math, with -ftz=false -prec-div=true -fmad=false.
#pragma once

#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace nb {

constexpr int kThreads = 256;               // CTA size of the streaming kernels
constexpr int kQuadsPerThread = 4;          // 4 x float4 per thread per chunk (64 B of g, 64 B of r in flight)
constexpr int kChunkQuads = kThreads * kQuadsPerThread;
constexpr uint64_t kChunkElems = (uint64_t)kChunkQuads * 4;   // 4096 elements per chunk

enum : uint32_t { kFlagNonfinite = 1u, kFlagOverflow = 2u, kFlagPeerTimeout = 4u };
enum : int { M_IDENTITY = 0, M_FP16 = 1, M_INT8 = 2, M_TOPK = 3, M_FP8 = 4, M_QSGD = 6, M_FP8_E5M2 = 7 };
enum : int { V_F32 = 0, V_F16 = 1, V_I8 = 2 };

// One (cluster, bucket) unit of codec work.  Offsets are relative to per-call base
// pointers so the same table serves every step.
struct Item {
  uint64_t g_off;     // element offset of this item's gradient from the grad base
  uint64_t r_off;     // element offset of its residual from the residual base (16-B aligned)
  uint64_t slot_off;  // byte offset of its payload (preamble start) from the slot base
  uint64_t n;         // coded elements
  uint64_t chunk0;    // first global chunk index of this item in the launch
  uint32_t sidx;      // scratch index (cluster * num_buckets + bucket)
  uint32_t pad;
};

// One bucket of decompress-reduce work.
struct RItem {
  uint64_t slot_off;  // byte offset of slot 0 (cluster 0's payload) of this bucket
  uint64_t pb;        // bytes per slot (stride between clusters' payloads)
  uint64_t out_off;   // element offset of the output from the out base
  uint64_t n;         // elements
  uint64_t chunk0;    // dense: first chunk of this bucket in the launch
  uint64_t k;         // TOPK: entries per payload
  uint64_t e0;        // TOPK: prefix of (k + 1) over the launch's buckets (offsets pass)
  uint64_t t0;        // TOPK: prefix of sparse-reduce tiles
  uint64_t sbase;     // TOPK: base of this bucket's [P][tiles + 1] start offsets
};

__host__ __device__ inline uint64_t pad16(uint64_t b) { return (b + 15) & ~uint64_t(15); }

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ uint32_t abs_bits(float x) { return __float_as_uint(x) & 0x7FFFFFFFu; }
__device__ __forceinline__ bool nonfinite_bits(uint32_t ab) { return ab >= 0x7F800000u; }

// Locate the item owning global chunk c.  Items are sorted by chunk0 and a CTA visits
// chunks in increasing order, so a forward scan from the previous hit is amortised O(1).
template <class T>
__device__ __forceinline__ int find_item(const T* items, int nitems, uint64_t c, int hint) {
  int i = hint;
  while (i + 1 < nitems && items[i + 1].chunk0 <= c) ++i;
  return i;
}

__device__ __forceinline__ float4 ld4_stream(const float* p) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st4(float* p, float4 v) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// L2 eviction-priority hints (createpolicy + .L2::cache_hint): streamed-once data is marked
// evict_first so that lines meant to be re-read (the fused INT8 kernel parks p in r) stay.
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_unchanged() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ld4_hint(const float* ptr, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ void st4_hint(float* ptr, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
               :: "l"(ptr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_u32_hint(uint32_t* ptr, uint32_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" :: "l"(ptr), "r"(v), "l"(pol) : "memory");
}

__device__ __forceinline__ void raise_flags(uint32_t* flags, bool bad, bool ovf) {
  unsigned m = __activemask();
  unsigned b = __ballot_sync(m, bad), o = __ballot_sync(m, ovf);
  if ((threadIdx.x & 31) == (__ffs(m) - 1)) {
    uint32_t f = (b ? kFlagNonfinite : 0u) | (o ? kFlagOverflow : 0u);
    if (f) atomicOr(flags, f);
  }
}

// INT8 scale from the bucket's max-abs bits (readings R3/R4):
// s = fl(m / 127); s := 1 when m == 0 or when fl(m/127) underflows to 0.
__device__ __forceinline__ float int8_scale_from_bits(uint32_t mbits) {
  float m = __uint_as_float(mbits);
  float s = __fdiv_rn(m, 127.0f);
  if (m == 0.0f || s == 0.0f) s = 1.0f;
  return s;
}

// q = clamp(rint(fl(p / s)), -127, 127)  (R5 ties-to-even, R6 IEEE division, R7 clamp)
__device__ __forceinline__ int int8_q(float p, float s) {
  int q = __float2int_rn(__fdiv_rn(p, s));
  return max(-127, min(127, q));
}

// Same result, cheaper: x = fl(p * fl(1/s)) is within 3 * 2^-24 * |x| of y = fl(p/s) (two
// roundings of 2^-24 each plus y's own), i.e. < 2.3e-5 while |x| <= 128.  If x is farther than
// 4e-5 from every half-integer, x and y round to the same integer (ties-to-even included:
// neither sits on a tie), and any |x| >= 128 + 4e-5 clamps either way.  Otherwise — and
// whenever 1/s is not a normal number — the IEEE division decides.  inv = fl(1/s) per bucket.
__device__ __forceinline__ int int8_q_fast(float p, float s, float inv) {
  const float x = __fmul_rn(p, inv);
  const float ax = fabsf(x);
  if (ax >= 128.0f + 4e-5f) return x > 0.0f ? 127 : -127;
  const float f = ax - floorf(ax);                 // exact for |x| < 2^23
  if (fabsf(f - 0.5f) > 4e-5f) {
    const int q = __float2int_rn(x);
    return max(-127, min(127, q));
  }
  return int8_q(p, s);
}
// fl(1/s) when it is a usable normal number, else 0 (then callers must use int8_q).
__device__ __forceinline__ float int8_inv(float s) {
  const float inv = __fdiv_rn(1.0f, s);
  return (inv < 3.0e38f && s >= 1.17549435e-38f) ? inv : 0.0f;
}
__device__ __forceinline__ int int8_qi(float p, float s, float inv) {
  return inv != 0.0f ? int8_q_fast(p, s, inv) : int8_q(p, s);
}

// FP8 (NEXT-4; "8-bit floating point"), format F: 1 = OCP E4M3 (R27: max 448, 3
// mantissa bits, smallest normal exponent -6), 2 = OCP E5M2 (R33: max 57344, 2 mantissa bits,
// smallest normal exponent -14).  s = fl(m / max) with the R4 degenerate rules; code = RNE of
// fl(p / s) to the format, saturating to +-max (cvt.rn.satfinite.{e4m3,e5m2}x2.f32);
// D = fl(FP8(code) * s).
template <int F>
__device__ __forceinline__ constexpr float fp8_max() { return F == 2 ? 57344.0f : 448.0f; }
template <int F>
__device__ __forceinline__ __nv_fp8_interpretation_t fp8_kind() { return F == 2 ? __NV_E5M2 : __NV_E4M3; }
template <int F = 1>
__device__ __forceinline__ float fp8_scale_from_bits(uint32_t mbits) {
  float m = __uint_as_float(mbits);
  float s = __fdiv_rn(m, fp8_max<F>());
  if (m == 0.0f || s == 0.0f) s = 1.0f;
  return s;
}
// two quotients -> two FP8 bytes (a in the low byte)
template <int F = 1>
__device__ __forceinline__ uint32_t fp8x2_of(float pa, float pb, float s) {
  return (uint32_t)__nv_cvt_float2_to_fp8x2(make_float2(__fdiv_rn(pa, s), __fdiv_rn(pb, s)), __NV_SATFINITE, fp8_kind<F>());
}
// Same bytes, cheaper (the INT8 argument of int8_q_fast, for the FP8 grid): x = fl(p * fl(1/s))
// is within 3 * 2^-24 |x| of y = fl(p / s).  In the binade of |x| (exponent e >= emin, the
// subnormal quantum below) the format rounds t = |x| 2^(MB-e) (exact scaling, t < 2^(MB+1)) to
// an integer, so x and y round alike unless frac(t) is within 3 * 2^-24 * 16 < 4e-6 of one half
// (binade edges are representable; the saturation boundary is such a midpoint).  Otherwise — or
// when inv = fl(1/s) is not a usable normal number (inv == 0) — the IEEE division decides.
template <int F = 1>
__device__ __forceinline__ float fp8_quotient(float p, float s, float inv) {
  constexpr int MB = F == 2 ? 2 : 3, EMIN = F == 2 ? -14 : -6, ESAT = F == 2 ? 17 : 20;
  if (inv == 0.0f) return __fdiv_rn(p, s);
  const float x = __fmul_rn(p, inv);
  const uint32_t b = __float_as_uint(x) & 0x7FFFFFFFu;
  const int e = max((int)(b >> 23) - 127, EMIN);
  if (e > ESAT) return x;                                 // saturates to +-max either way
  const float t = __fmul_rn(__uint_as_float(b), __uint_as_float((uint32_t)(127 + MB - e) << 23));
  return fabsf(t - floorf(t) - 0.5f) > 4e-6f ? x : __fdiv_rn(p, s);
}
template <int F = 1>
__device__ __forceinline__ uint32_t fp8x2_fast(float pa, float pb, float s, float inv) {
  return (uint32_t)__nv_cvt_float2_to_fp8x2(make_float2(fp8_quotient<F>(pa, s, inv), fp8_quotient<F>(pb, s, inv)),
                                            __NV_SATFINITE, fp8_kind<F>());
}
// FP8 byte -> binary32 (exact: E4M3 and E5M2 values are binary16 values)
template <int F = 1>
__device__ __forceinline__ float fp8_val(uint32_t byte) {
  __half_raw h = __nv_cvt_fp8_to_halfraw((__nv_fp8_storage_t)(byte & 0xFF), fp8_kind<F>());
  return __half2float(__half(h));
}

// QSGD (NEXT-4, R32): counter-based uniforms.  splitmix64(z) = mix(z + gamma) (Steele, Lea &
// Flood 2014); per (seed, step, cluster, bucket, shard) a base state; output j =
// splitmix64(base + j * gamma) feeds elements 2j (bits 63..40) and 2j + 1 (bits 39..16), each
// scaled by 2^-24 (exact in binary32).
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t qsgd_key(uint32_t cluster, uint32_t shard, uint32_t bucket) {
  return ((((uint64_t)cluster * 65536u + shard) << 32) | bucket);
}
__device__ __forceinline__ uint64_t qsgd_base(uint64_t seed, uint64_t step, uint64_t key) {
  return splitmix64(seed ^ splitmix64(step ^ splitmix64(key)));
}
__device__ __forceinline__ uint64_t qsgd_h(uint64_t base, uint64_t j) {
  return splitmix64(base + j * 0x9E3779B97F4A7C15ull);
}
__device__ __forceinline__ float qsgd_hi(uint64_t h) { return (float)(uint32_t)(h >> 40) * 5.9604644775390625e-8f; }
__device__ __forceinline__ float qsgd_lo(uint64_t h) {
  return (float)(uint32_t)((h >> 16) & 0xFFFFFFu) * 5.9604644775390625e-8f;
}
__device__ __forceinline__ float qsgd_u(uint64_t base, uint64_t e) {   // one element (tails)
  const uint64_t h = qsgd_h(base, e >> 1);
  return (e & 1) ? qsgd_lo(h) : qsgd_hi(h);
}
// q = floor(x) + [u < x - floor(x)], x = fl(p / s) (IEEE division), clamped to [-127, 127]
__device__ __forceinline__ int qsgd_q(float p, float s, float u) {
  const float x = __fdiv_rn(p, s);
  const float f = floorf(x);
  const float q = __fadd_rn(f, u < __fsub_rn(x, f) ? 1.0f : 0.0f);
  return max(-127, min(127, (int)q));
}

// ---- the same quantiser without the SFU / conversion unit (the fused QSGD step was bound by
// its ~5 XU operations per element: reciprocal, floor, float<->int conversions).  Same bits.
//
// x = fl(p / s): q1 = q0 + fl(p - q0 s)·inv with q0 = fl(p·inv), inv = fl(1/s), accepted when
// |p - q1·s| < ulp(q1)/2 · s — then q1 IS the correctly rounded quotient (a quotient of two
// binary32 numbers never lies on a rounding midpoint; the FMA residuals are exact for a q
// within one ulp of p/s and no underflow, guarded by |p| >= 2^-90).  q1 a power of two (its
// rounding interval is asymmetric), a failed check, or inv == 0: the IEEE division.
__device__ __forceinline__ float div_rn_fma(float p, float s, float inv) {
  if (p == 0.0f) return p;                       // fl(+-0 / s) = +-0 for s > 0
  if (inv != 0.0f && fabsf(p) >= 8.077935669463161e-28f) {   // 2^-90
    const float q0 = __fmul_rn(p, inv);
    const float q1 = __fmaf_rn(__fmaf_rn(-q0, s, p), inv, q0);
    const uint32_t b = __float_as_uint(q1), e = b & 0x7F800000u;
    if (e >= (25u << 23) && e < 0x7F800000u && (b & 0x7FFFFFu) != 0u) {
      const float r1 = __fmaf_rn(-q1, s, p);
      if (fabsf(r1) < __fmul_rn(__uint_as_float(e - (24u << 23)), s)) return q1;
    }
  }
  return __fdiv_rn(p, s);
}
// m * 2^-24 for a 24-bit m, exactly, with integer / FMA-pipe operations only
__device__ __forceinline__ float u24_to_unit(uint32_t m) {
  return __fadd_rn(__fsub_rn(__uint_as_float(0x3F800000u | (m >> 1)), 1.0f), (m & 1u) ? 5.9604644775390625e-8f : 0.0f);
}
__device__ __forceinline__ float qsgd_hi_f(uint64_t h) { return u24_to_unit((uint32_t)(h >> 40)); }
__device__ __forceinline__ float qsgd_lo_f(uint64_t h) { return u24_to_unit((uint32_t)((h >> 16) & 0xFFFFFFu)); }
// the QSGD code as an integer-valued float in [-127, 127] (|x| <= 128: floor by the 1.5 * 2^23
// round-to-integer trick, exact for |x| < 2^22)
__device__ __forceinline__ float qsgd_qf(float p, float s, float inv, float u) {
  const float x = div_rn_fma(p, s, inv);
  const float rn = __fsub_rn(__fadd_rn(x, 12582912.0f), 12582912.0f);
  const float f = rn > x ? __fsub_rn(rn, 1.0f) : rn;
  const float q = __fadd_rn(f, u < __fsub_rn(x, f) ? 1.0f : 0.0f);
  return fminf(fmaxf(q, -127.0f), 127.0f);
}
// low byte of an integer-valued float in [-128, 127] (two's complement), no conversion unit
__device__ __forceinline__ uint32_t byte_of_intf(float q) {
  return (uint32_t)(__float_as_int(__fadd_rn(q, 12582912.0f)) - 0x4B400000) & 0xFFu;
}

// What the QSGD quantiser needs besides p and s: the generator state of this call.
struct SrArgs {
  uint64_t seed, step;
  uint32_t cluster0;   // cluster id of item sidx / num_buckets == 0 (LOOPBACK 0, else this rank's)
  uint32_t shard;      // local rank in the cluster (G > 1), else 0
  uint32_t num_buckets;
};

__device__ __forceinline__ uint32_t pack_i8x4(int a, int b, int c, int d) {
  return (uint32_t)(a & 0xFF) | ((uint32_t)(b & 0xFF) << 8) | ((uint32_t)(c & 0xFF) << 16) |
         ((uint32_t)(d & 0xFF) << 24);
}

// R16: fixed pairwise tree over cluster ids, sum(lo,hi) = sum(lo,mid) + sum(mid,hi) with
// mid = lo + ceil((hi-lo)/2); every '+' one binary32 rounding.
template <int LO, int HI>
__device__ __forceinline__ float tree_sum(const float* v) {
  if constexpr (HI - LO == 1) {
    return v[LO];
  } else {
    constexpr int MID = LO + (HI - LO + 1) / 2;
    return __fadd_rn(tree_sum<LO, MID>(v), tree_sum<MID, HI>(v));
  }
}

// System-scope flag protocol of the P2P exchanges (peers' words reached over NVLink).
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns_u64() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void write_preamble(uint8_t* slot, uint32_t method, uint32_t count, float scale,
                                               uint32_t aux) {
  uint4 pre = make_uint4(method, count, __float_as_uint(scale), aux);
  *reinterpret_cast<uint4*>(slot) = pre;
}

// Where a compressor writes its payload: p[0] = this cluster's own slot, p[1..n-1] = the same
// slot in every peer's (IPC-mapped, NVLink) slot buffer when the exchange is fused into the
// compress kernels (P2P push).  Offsets are identical on every rank.  Passed by value (kernel
// parameter space), n = 1 for LOOPBACK and for the NCCL all-gather exchange.
struct Dests {
  uint8_t* p[8];
  int n;
};
template <class T>
__device__ __forceinline__ void put(const Dests& d, uint64_t off, T v) {
#pragma unroll 1
  for (int k = 0; k < d.n; ++k) *reinterpret_cast<T*>(d.p[k] + off) = v;
}
// Push per-lane payload words to the PEERS (d.p[1..]) as 16-byte stores (NVLink moves wide
// stores far better than 4-byte ones).  Lanes holding consecutive words form groups — 4 lanes
// of u32 words or 2 lanes of u64 words — whose first lane is 16-byte aligned (callers keep
// word index % group == lane % group); full groups are written by their first lane, partial
// groups lane by lane.  Must be called by all 32 lanes (valid marks the lanes with a word).
__device__ __forceinline__ void push_u32(const Dests& d, uint64_t off, uint32_t w, bool valid) {
  if (d.n < 2) return;
  const unsigned lane = threadIdx.x & 31;
  const uint32_t w1 = __shfl_down_sync(0xFFFFFFFFu, w, 1), w2 = __shfl_down_sync(0xFFFFFFFFu, w, 2),
                 w3 = __shfl_down_sync(0xFFFFFFFFu, w, 3);
  const unsigned vm = __ballot_sync(0xFFFFFFFFu, valid);
  const bool full = ((vm >> (lane & ~3u)) & 0xFu) == 0xFu;
  if (full) {
    if ((lane & 3u) == 0)
#pragma unroll 1
      for (int k = 1; k < d.n; ++k) *reinterpret_cast<uint4*>(d.p[k] + off) = make_uint4(w, w1, w2, w3);
  } else if (valid) {
#pragma unroll 1
    for (int k = 1; k < d.n; ++k) *reinterpret_cast<uint32_t*>(d.p[k] + off) = w;
  }
}
__device__ __forceinline__ void push_u64(const Dests& d, uint64_t off, uint2 w, bool valid) {
  if (d.n < 2) return;
  const unsigned lane = threadIdx.x & 31;
  const uint32_t x1 = __shfl_down_sync(0xFFFFFFFFu, w.x, 1), y1 = __shfl_down_sync(0xFFFFFFFFu, w.y, 1);
  const unsigned vm = __ballot_sync(0xFFFFFFFFu, valid);
  const bool full = ((vm >> (lane & ~1u)) & 0x3u) == 0x3u;
  if (full) {
    if ((lane & 1u) == 0)
#pragma unroll 1
      for (int k = 1; k < d.n; ++k) *reinterpret_cast<uint4*>(d.p[k] + off) = make_uint4(w.x, w.y, x1, y1);
  } else if (valid) {
#pragma unroll 1
    for (int k = 1; k < d.n; ++k) *reinterpret_cast<uint2*>(d.p[k] + off) = w;
  }
}

__device__ __forceinline__ void put_preamble(const Dests& d, uint64_t off, uint32_t method, uint32_t count, float scale,
                                             uint32_t aux) {
  put(d, off, make_uint4(method, count, __float_as_uint(scale), aux));
}

}  // namespace nb
