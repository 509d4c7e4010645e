// dense_common.cuh — device helpers shared by the streaming (kernels_dense.cu) and the
// warp-specialised TMA (kernels_ws.cu) kernels.  Device code only; the oracle shares nothing.
#pragma once

#include <cuda_fp16.h>

#include "kernels.h"

namespace nb {

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}

__device__ __forceinline__ void zero_padding_t(const Dests& d, uint64_t body_off, uint64_t nbytes, int tid) {
  const uint64_t end = pad16(nbytes);
  const uint64_t z = nbytes + (tid >= 16 ? tid - 16 : end);
  if (z < end) put<uint8_t>(d, body_off + z, (uint8_t)0);
}

__device__ __forceinline__ float fp16_one(float p, uint16_t& hb, bool& bad, bool& ovf) {
  __half h = __float2half_rn(p);              // IEEE binary32 -> binary16, RNE, subnormals kept
  hb = __half_as_ushort(h);
  const uint32_t ab = abs_bits(p);
  bad |= nonfinite_bits(ab);
  ovf |= ((hb & 0x7FFFu) == 0x7C00u) && !nonfinite_bits(ab);   // finite p rounded to +-inf (R10)
  return __half2float(h);
}

// out = fl(tree_sum / P).  For P a power of two, x * (1/P) is the same correctly rounded
// value as x / P (1/P is exact), so the multiply is used; otherwise IEEE division.
template <int P>
__device__ __forceinline__ float div_p(float x) {
  if constexpr ((P & (P - 1)) == 0) return __fmul_rn(x, 1.0f / (float)P);
  else return __fdiv_rn(x, (float)P);
}

struct Slice {
  uint64_t q0, q1;
};
__device__ __forceinline__ Slice slice_of(uint64_t n4, unsigned G) {
  const uint64_t per = ((n4 + G - 1) / G + 3) & ~uint64_t(3);   // 4-quad aligned (16-B pushes)
  const uint64_t q0 = min(n4, (uint64_t)blockIdx.x * per);
  return Slice{q0, min(n4, q0 + per)};
}

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


}  // namespace nb
