// kernels_intra.cu — sm_100a kernels of the hierarchical (G > 1) intra-cluster hop over
// NVLink peer memory, replacing NCCL's ReduceScatter(avg) / AllGather with a FIXED order
// (R20; "standard parallelism" inside a cluster, PAPER.md:288 the
// fast intra / slow inter split):
//
//   k_rs_push   : GPU l stores slice j of its bucket into peer j's receive buffer, slot l
//                 (one NVLink write per element that leaves the GPU; 16-B stores)
//   (flags)     : k_exchange_flags on the RS arrival words (kernels_ws.cu)
//   k_rs_reduce : shard_l = fl(fl(...fl(x_0 + x_1) + ... + x_{G-1}) / G) — the G GPUs' slices
//                 summed in local-rank order, each '+' one binary32 rounding, then one IEEE
//                 division (a multiply by the exact 1/G when G is a power of two); x_l is read
//                 straight from the caller's gradient, x_j (j != l) from the receive buffer
//   (flags)     : k_exchange_flags on the AG arrival words
//   k_ag_pull   : out[slice j] = peer j's averaged shard, loaded over NVLink (own: local)
//   k_scale_mail: NEXT-3 exact cluster scale — every GPU's shard max-abs word to every peer,
//                 then the max over the G words (replaces a 4-byte ncclAllReduce(max))
//
// The oracle's hierarchical_step sums in the same order and divides once, so the cluster
// mean is bit-identical for ANY input (round 1 relied on dyadic inputs because ncclAvg's
// order and pre-scaling are NCCL's).
#include <algorithm>

#include "kernels.h"

namespace nb {

constexpr int kIThreads = 256;
constexpr uint64_t kIChunk = 4096;   // elements per chunk (16 per thread)

__device__ __forceinline__ float4 ld4_cg(const float* p) {   // L2 (or the peer's L2), never a stale L1 line
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float ld1_cg(const float* p) {
  float v;
  asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ float div_g(float x, int G, float inv) {
  return (G & (G - 1)) == 0 ? __fmul_rn(x, inv) : __fdiv_rn(x, (float)G);
}

// items: one per bucket of the call; item i covers chunks [chunk0, chunk0 + ceil(cn / 4096)).
template <bool VEC>
__global__ void __launch_bounds__(kIThreads) k_rs_push(const IItem* __restrict__ items, int nitems, uint64_t chunks,
                                                        const float* __restrict__ g, PeerF recv, uint64_t stride) {
  int hint = 0;
  const int G = recv.n, me = recv.me;
  for (uint64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    const int i = find_item(items, nitems, c, hint);
    hint = i;
    const IItem it = items[i];
    const uint64_t e0 = (c - it.chunk0) * kIChunk, e1 = min(it.cn, e0 + kIChunk);
    for (int j = 0; j < G; ++j) {
      if (j == me) continue;
      const float* src = g + it.off + (uint64_t)j * it.cn;
      float* dst = recv.p[j] + (uint64_t)me * stride + it.coff;   // peer j's slot `me`
      if (VEC) {
        for (uint64_t e = e0 + 4 * threadIdx.x; e < e1; e += 4 * kIThreads)
          *reinterpret_cast<float4*>(dst + e) = __ldg(reinterpret_cast<const float4*>(src + e));
      } else {
        for (uint64_t e = e0 + threadIdx.x; e < e1; e += kIThreads) dst[e] = src[e];
      }
    }
  }
  __threadfence_system();   // the stores reach the peers before the flag kernel's release
}

template <bool VEC>
__global__ void __launch_bounds__(kIThreads) k_rs_reduce(const IItem* __restrict__ items, int nitems, uint64_t chunks,
                                                          const float* __restrict__ g, const float* __restrict__ recv,
                                                          uint64_t stride, int G, int me, float* __restrict__ shard) {
  int hint = 0;
  const float inv = 1.0f / (float)G;   // exact when G is a power of two (the only case it is used)
  for (uint64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    const int i = find_item(items, nitems, c, hint);
    hint = i;
    const IItem it = items[i];
    const uint64_t e0 = (c - it.chunk0) * kIChunk, e1 = min(it.cn, e0 + kIChunk);
    const float* own = g + it.off + (uint64_t)me * it.cn;
    float* out = shard + it.coff;
    if (VEC) {
      for (uint64_t e = e0 + 4 * threadIdx.x; e < e1; e += 4 * kIThreads) {
        float4 acc = me == 0 ? __ldg(reinterpret_cast<const float4*>(own + e)) : ld4_cg(recv + it.coff + e);
        for (int j = 1; j < G; ++j) {
          const float4 x = j == me ? __ldg(reinterpret_cast<const float4*>(own + e))
                                   : ld4_cg(recv + (uint64_t)j * stride + it.coff + e);
          acc = make_float4(__fadd_rn(acc.x, x.x), __fadd_rn(acc.y, x.y), __fadd_rn(acc.z, x.z), __fadd_rn(acc.w, x.w));
        }
        *reinterpret_cast<float4*>(out + e) =
            make_float4(div_g(acc.x, G, inv), div_g(acc.y, G, inv), div_g(acc.z, G, inv), div_g(acc.w, G, inv));
      }
    } else {
      for (uint64_t e = e0 + threadIdx.x; e < e1; e += kIThreads) {
        float acc = me == 0 ? own[e] : ld1_cg(recv + it.coff + e);
        for (int j = 1; j < G; ++j) acc = __fadd_rn(acc, j == me ? own[e] : ld1_cg(recv + (uint64_t)j * stride + it.coff + e));
        out[e] = div_g(acc, G, inv);
      }
    }
  }
}

template <bool VEC>
__global__ void __launch_bounds__(kIThreads) k_ag_pull(const IItem* __restrict__ items, int nitems, uint64_t chunks,
                                                        PeerF shards, float* __restrict__ out) {
  int hint = 0;
  const int G = shards.n;
  for (uint64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    const int i = find_item(items, nitems, c, hint);
    hint = i;
    const IItem it = items[i];
    const uint64_t e0 = (c - it.chunk0) * kIChunk, e1 = min(it.cn, e0 + kIChunk);
    for (int j = 0; j < G; ++j) {
      const float* src = shards.p[j] + it.coff;
      float* dst = out + it.off + (uint64_t)j * it.cn;
      if (VEC) {
        for (uint64_t e = e0 + 4 * threadIdx.x; e < e1; e += 4 * kIThreads)
          *reinterpret_cast<float4*>(dst + e) = ld4_cg(src + e);
      } else {
        for (uint64_t e = e0 + threadIdx.x; e < e1; e += kIThreads) dst[e] = ld1_cg(src + e);
      }
    }
  }
}

// One thread per (bucket, peer): post this GPU's max-abs word of each bucket into every peer's
// mailbox [b][me] (plain stores, then a system-scope release of the bucket's arrival word),
// wait for every peer's word, and replace scratch[b] by the max of the G words (|p| bits order
// like the floats; NaN/Inf bits above every finite one, so a non-finite shard poisons all).
__global__ void k_scale_mail(Peers pe, PeerU mails, uint32_t* scratch, uint32_t* my_mail,
                             unsigned long long* local, int lo, int hi, unsigned long long seq, uint32_t* flags) {
  const int G = pe.n, me = pe.me, total = (hi - lo) * G;
  for (int x = threadIdx.x; x < total; x += blockDim.x) {
    const int b = lo + x / G, j = x % G;
    if (j == me) my_mail[(size_t)b * G + me] = scratch[b];
    else {
      volatile uint32_t* dst = mails.p[j] + (size_t)b * G + me;
      *dst = scratch[b];
    }
  }
  __threadfence_system();
  __syncthreads();
  for (int x = threadIdx.x; x < total; x += blockDim.x) {
    const int b = lo + x / G, j = x % G;
    if (j != me) st_release_sys_u64(pe.arrive[j] + (size_t)b * G + me, seq);
  }
  const unsigned long long t0 = globaltimer_ns_u64();
  bool timeout = false;
  for (int x = threadIdx.x; x < total && !timeout; x += blockDim.x) {
    const int b = lo + x / G, j = x % G;
    if (j == me) continue;
    while (ld_acquire_sys_u64(local + (size_t)b * G + j) < seq) {
      if (globaltimer_ns_u64() - t0 > 60ull * 1000000000ull) {
        atomicOr(flags, kFlagPeerTimeout);
        timeout = true;
        break;
      }
    }
  }
  __threadfence();
  __syncthreads();
  for (int b = lo + threadIdx.x; b < hi; b += blockDim.x) {
    uint32_t m = 0;
    for (int j = 0; j < G; ++j) m = max(m, *reinterpret_cast<volatile uint32_t*>(my_mail + (size_t)b * G + j));
    scratch[b] = m;
  }
}

void preload_intra() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, (const void*)k_rs_push<true>);
  cudaFuncGetAttributes(&a, (const void*)k_rs_push<false>);
  cudaFuncGetAttributes(&a, (const void*)k_rs_reduce<true>);
  cudaFuncGetAttributes(&a, (const void*)k_rs_reduce<false>);
  cudaFuncGetAttributes(&a, (const void*)k_ag_pull<true>);
  cudaFuncGetAttributes(&a, (const void*)k_ag_pull<false>);
  cudaFuncGetAttributes(&a, (const void*)k_scale_mail);
}

static unsigned grid_of(const Launch& L, uint64_t chunks, const void* f) {
  return persistent_grid(L, chunks, f, kIThreads);
}

void launch_rs_push(const Launch& L, bool vec, const IItem* items, int nitems, uint64_t chunks, const float* g,
                    const PeerF& recv, uint64_t stride) {
  if (!chunks) return;
  Mark mk(L, PH_RS_PUSH);
  if (vec) k_rs_push<true><<<grid_of(L, chunks, (const void*)k_rs_push<true>), kIThreads, 0, L.stream>>>(items, nitems, chunks, g, recv, stride);
  else k_rs_push<false><<<grid_of(L, chunks, (const void*)k_rs_push<false>), kIThreads, 0, L.stream>>>(items, nitems, chunks, g, recv, stride);
  ++*L.launches;
}

void launch_rs_reduce(const Launch& L, bool vec, const IItem* items, int nitems, uint64_t chunks, const float* g,
                      const float* recv, uint64_t stride, int G, int me, float* shard) {
  if (!chunks) return;
  Mark mk(L, PH_RS_REDUCE);
  if (vec) k_rs_reduce<true><<<grid_of(L, chunks, (const void*)k_rs_reduce<true>), kIThreads, 0, L.stream>>>(items, nitems, chunks, g, recv, stride, G, me, shard);
  else k_rs_reduce<false><<<grid_of(L, chunks, (const void*)k_rs_reduce<false>), kIThreads, 0, L.stream>>>(items, nitems, chunks, g, recv, stride, G, me, shard);
  ++*L.launches;
}

void launch_ag_pull(const Launch& L, bool vec, const IItem* items, int nitems, uint64_t chunks, const PeerF& shards,
                    float* out) {
  if (!chunks) return;
  Mark mk(L, PH_AG_PULL);
  if (vec) k_ag_pull<true><<<grid_of(L, chunks, (const void*)k_ag_pull<true>), kIThreads, 0, L.stream>>>(items, nitems, chunks, shards, out);
  else k_ag_pull<false><<<grid_of(L, chunks, (const void*)k_ag_pull<false>), kIThreads, 0, L.stream>>>(items, nitems, chunks, shards, out);
  ++*L.launches;
}

void launch_scale_mail(const Launch& L, const Peers& pe, const PeerU& mails, uint32_t* scratch, uint32_t* my_mail,
                       unsigned long long* local_arrive, int lo, int hi, uint64_t seq, uint32_t* flags) {
  Mark mk(L, PH_SCALE_MAIL);
  k_scale_mail<<<1, 256, 0, L.stream>>>(pe, mails, scratch, my_mail, local_arrive, lo, hi, (unsigned long long)seq, flags);
  ++*L.launches;
}

}  // namespace nb
