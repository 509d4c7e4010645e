// kernels_svd.cu — FP16(SVD(rho)) low-rank compressor of one fp32 matrix.
//
// A = U S V^T (Eq. 1), keep the top r singular triples (Eq. 2), send
// C_FP16(U_r, S_r, V_r) (Eq. 5); the receiver rebuilds A' = U_r S_r V_r^T (Eq. 3).  Ratio =
// Eq. 4 / 2.  Readings R29-R31: r from rho, sign convention, payload layout.
//
// Pipeline on the GPU, with B = A (m >= n, "tall") or B = A^T (m < n): k = min(m, n),
// L = max(m, n), B is L x k.
//   K_gram   G = B^T B             k x k, fp64 accumulation of exact fp32 products; the
//                                   contraction over L runs split across CTAs, upper-triangle
//                                   64 x 64 tiles only (G is symmetric)
//   syevd    G = Z diag(lambda) Z^T  cuSOLVER (the one library step: a dense symmetric
//                                   eigensolver); top r eigenpairs -> sigma_j = sqrt(lambda),
//                                   W_r = right singular vectors of B
//   K_prep   sigma, W_r (fp32)
//   K_proj   Y = B W_r              L x r fp32 GEMM; Y / sigma = left singular vectors of B
//   K_sign   per column: the largest-|.| entry of U_A must be positive (R30)
//   K_pack   preamble + binary16 U_r [m][r], S_r [r], V_r [n][r]
//   K_recon  A' = (U_r S_r) V_r^T   m x n fp32 GEMM from the binary16 payload (decompress)
//
// Why the Gram route: only V_r must be accurate for A' (A' = B W_r W_r^T for the tall case,
// whatever the rounding of U = Y / sigma), and fp64 accumulation keeps lambda accurate to
// ~1e-16 sigma_1^2, far below the binary16 rounding of the factors.  Every GEMM here is
// SIMT (64 x 64 tiles, 4 x 4 per thread, explicit FMA intrinsics); at the Table-5 shapes the
// step is bound by the eigensolver, not by these contractions.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <stdint.h>

#include <cmath>
#include <string>
#include <vector>

#include "nebula_sync.h"

namespace nbsvd {

constexpr int T = 64;      // output tile edge
constexpr int BK = 16;     // contraction slice per smem stage (GEMMs)
constexpr int GK = 32;     // contraction slice per smem stage (Gram, fp64)
constexpr int NT = 256;    // threads per CTA: 16 x 16, each a 4 x 4 sub-tile

enum : uint32_t { F_NONFINITE = 1u, F_OVERFLOW = 2u };

struct Shape {
  int64_t m, n;   // A is m x n row-major
  int k, r;       // k = min(m, n), r kept
  int64_t L;      // max(m, n)
  bool tall;      // m >= n: B = A, else B = A^T
};

// B(i, a) for i < L, a < k
__device__ __forceinline__ float bval(const float* A, const Shape& s, int64_t i, int64_t a) {
  return s.tall ? A[i * s.n + a] : A[a * s.n + i];
}

// Stage rows [i0, i0 + GK) of B's column tiles a0.. and b0.. (64 columns each) into shared
// memory as fp64.  VEC (A 16-B aligned, n % 4 == 0): one float4 per thread-iteration along the
// contiguous direction of A (columns of B when tall, rows of B when wide); partial float4s at
// the matrix edges fall back to scalar loads.  Returns whether a non-finite value was seen.
template <int NTH>
__device__ __forceinline__ bool stage_tiles(const float* __restrict__ A, const Shape& s, int a0, int b0, int64_t i0,
                                            int64_t i_end, double (*sa)[T + 1], double (*sb)[T + 1], bool vec) {
  bool bad = false;
  if (vec) {
#pragma unroll
    for (int u = 0; u < GK * T / 4 / NTH; ++u) {
      const int f = threadIdx.x + u * NTH;
      // tall: 16 float4 per B row (64 columns); wide: 8 float4 per A row (32 B rows)
      const int ii = s.tall ? f / (T / 4) : (f % (GK / 4)) * 4;
      const int aa = s.tall ? (f % (T / 4)) * 4 : f / (GK / 4);
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        const int c0 = side ? b0 : a0;
        double (*dst)[T + 1] = side ? sb : sa;
        float v[4];
        if (s.tall) {
          const int64_t i = i0 + ii;
          if (i < i_end && c0 + aa + 3 < s.k) {
            const float4 w = *reinterpret_cast<const float4*>(A + i * s.n + c0 + aa);
            v[0] = w.x; v[1] = w.y; v[2] = w.z; v[3] = w.w;
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) v[e] = (i < i_end && c0 + aa + e < s.k) ? A[i * s.n + c0 + aa + e] : 0.0f;
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) dst[ii][aa + e] = (double)v[e];
        } else {
          const int64_t i = i0 + ii, a = c0 + aa;
          if (a < s.k && i + 3 < i_end) {
            const float4 w = *reinterpret_cast<const float4*>(A + (int64_t)a * s.n + i);
            v[0] = w.x; v[1] = w.y; v[2] = w.z; v[3] = w.w;
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) v[e] = (a < s.k && i + e < i_end) ? A[(int64_t)a * s.n + i + e] : 0.0f;
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) dst[ii + e][aa] = (double)v[e];
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) bad |= !isfinite(v[e]);
      }
    }
  } else {
#pragma unroll
    for (int t = 0; t < GK * T / NTH; ++t) {
      const int idx = threadIdx.x + t * NTH;
      const int ii = s.tall ? idx / T : idx % GK;
      const int aa = s.tall ? idx % T : idx / GK;
      const int64_t i = i0 + ii;
      float va = 0.f, vb = 0.f;
      if (i < i_end) {
        if (a0 + aa < s.k) va = bval(A, s, i, a0 + aa);
        if (b0 + aa < s.k) vb = bval(A, s, i, b0 + aa);
      }
      bad |= !isfinite(va) || !isfinite(vb);
      sa[ii][aa] = (double)va;
      sb[ii][aa] = (double)vb;
    }
  }
  return bad;
}

// ---------------------------------------------------------------- K_gram: G += B^T B (upper tiles)
// grid: (tile pairs ta <= tb, splits over L).  Each CTA loads GK rows of B for both column
// tiles into shared memory as fp64 (fp32 * fp32 is exact in fp64) and accumulates 4 x 4 fp64
// per thread; the split partial sums meet in G with fp64 atomics (G zeroed first).
__global__ void __launch_bounds__(NT) k_gram(const float* __restrict__ A, Shape s, const int2* __restrict__ tiles,
                                            int64_t rows_per_split, double* __restrict__ G, uint32_t* flags, bool vec) {
  __shared__ double sa[GK][T + 1], sb[GK][T + 1];
  const int2 tp = tiles[blockIdx.x];
  const int a0 = tp.x * T, b0 = tp.y * T;
  const int64_t i_begin = (int64_t)blockIdx.y * rows_per_split;
  const int64_t i_end = min(s.L, i_begin + rows_per_split);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4] = {};
  bool bad = false;
  for (int64_t i0 = i_begin; i0 < i_end; i0 += GK) {
    bad |= stage_tiles<NT>(A, s, a0, b0, i0, i_end, sa, sb, vec);
    __syncthreads();
#pragma unroll 4
    for (int ii = 0; ii < GK; ++ii) {
      double x[4], y[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { x[u] = sa[ii][ty * 4 + u]; y[u] = sb[ii][tx * 4 + u]; }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(x[u], y[v], acc[u][v]);
    }
    __syncthreads();
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags, F_NONFINITE);
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int a = a0 + ty * 4 + u, b = b0 + tx * 4 + v;
      if (a < s.k && b < s.k && a <= b) atomicAdd(&G[(int64_t)a * s.k + b], acc[u][v]);
    }
}

// Same contraction on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64 — tcgen05 has no fp64
// kind; the default: with float4 staging of B the SIMT kernel takes 0.65 ms at 8192 x 768 and
// this one ~0.2 ms less, per the compress times in DESIGN.md §10): a CTA of 4 warps owns the 64 x 64 tile, each warp a 32 x 32 quarter = 4 x 4 MMA tiles
// of 8 x 8, 32 fp64 accumulators per thread.  Fragments (PTX m8n8k4 .f64): A row-major 8 x 4:
// a0 = A[g][t]; B col-major 4 x 8: b0 = B[t][g]; C 8 x 8: c{0,1} = C[g][2t + {0,1}], with
// g = lane / 4, t = lane % 4.  Here A[m][kk] = B(i0 + kk, a0 + m) and B[kk][n] = B(i0 + kk, b0 + n),
// both read from the fp64 shared slices of k_gram.  Products of fp32 values are exact in fp64
// and the accumulation is fp64, as in the SIMT kernel (the summation order differs).
constexpr int GT = 128;   // threads of k_gram_dmma
__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__global__ void __launch_bounds__(GT) k_gram_dmma(const float* __restrict__ A, Shape s, const int2* __restrict__ tiles,
                                                 int64_t rows_per_split, double* __restrict__ G, uint32_t* flags, bool vec) {
  __shared__ double sa[GK][T + 1], sb[GK][T + 1];
  const int2 tp = tiles[blockIdx.x];
  const int a0 = tp.x * T, b0 = tp.y * T;
  const int64_t i_begin = (int64_t)blockIdx.y * rows_per_split;
  const int64_t i_end = min(s.L, i_begin + rows_per_split);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;   // warp quarter of the 64 x 64 tile
  const int g = lane >> 2, t = lane & 3;
  double acc[4][4][2] = {};
  bool bad = false;
  for (int64_t i0 = i_begin; i0 < i_end; i0 += GK) {
    bad |= stage_tiles<GT>(A, s, a0, b0, i0, i_end, sa, sb, vec);
    __syncthreads();
#pragma unroll 2
    for (int kk = 0; kk < GK; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        fa[x] = sa[kk + t][wm + 8 * x + g];
        fb[x] = sb[kk + t][wn + 8 * x + g];
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) dmma_8x8x4(acc[x][y], fa[x], fb[y]);
    }
    __syncthreads();
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags, F_NONFINITE);
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int a = a0 + wm + 8 * x + g, b = b0 + wn + 8 * y + 2 * t + v;
        if (a < s.k && b < s.k && a <= b) atomicAdd(&G[(int64_t)a * s.k + b], acc[x][y][v]);
      }
}

// ---------------------------------------------------------------- K_prep: top-r eigenpairs
// cuSOLVER returns ascending lambda and, column-major, eigenvector j in column j: in our
// row-major view Z[j * k + a] = z_j[a].  sigma_j = sqrt(max(lambda_{k-1-j}, 0)) (fp64);
// Wr[a][j] = z_{k-1-j}[a] as fp32 (the GEMM operand).
__global__ void k_prep(Shape s, const double* __restrict__ lambda, const double* __restrict__ Z,
                       double* __restrict__ sigma, float* __restrict__ Wr) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < s.r) sigma[e] = sqrt(fmax(lambda[s.k - 1 - e], 0.0));
  if (e < (int64_t)s.k * s.r) {
    const int64_t a = e / s.r, j = e % s.r;
    Wr[e] = (float)Z[(int64_t)(s.k - 1 - j) * s.k + a];
  }
}

// ---------------------------------------------------------------- generic SIMT GEMM tile
// C[M x N] = sum_q Aop(i, q) * Bop(j, q); operands staged as BK x 64 slices in shared memory
// (stored [q][i] so the 4 x 4 inner product reads are conflict-free broadcasts), explicit
// __fmaf_rn (one rounding per multiply-add; the library is built with -fmad=false).
template <class LA, class LB, class EP>
__device__ __forceinline__ void gemm_tile(int64_t M, int64_t N, int64_t K, LA la, LB lb, EP ep) {
  __shared__ float sA[BK][T + 4], sB[BK][T + 4];
  const int64_t i0 = (int64_t)blockIdx.y * T, j0 = (int64_t)blockIdx.x * T;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int64_t q0 = 0; q0 < K; q0 += BK) {
#pragma unroll
    for (int t = 0; t < BK * T / NT; ++t) {
      const int idx = threadIdx.x + t * NT;
      // the loaders choose their own coalescing order via (row-fast | q-fast) mapping
      int rr, qq;
      if (la.q_fast) { qq = idx % BK; rr = idx / BK; } else { rr = idx % T; qq = idx / T; }
      const int64_t i = i0 + rr, q = q0 + qq;
      sA[qq][rr] = (i < M && q < K) ? la(i, q) : 0.f;
      if (lb.q_fast) { qq = idx % BK; rr = idx / BK; } else { rr = idx % T; qq = idx / T; }
      const int64_t j = j0 + rr, q2 = q0 + qq;
      sB[qq][rr] = (j < N && q2 < K) ? lb(j, q2) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int qq = 0; qq < BK; ++qq) {
      const float4 x = *reinterpret_cast<const float4*>(&sA[qq][ty * 4]);
      const float4 y = *reinterpret_cast<const float4*>(&sB[qq][tx * 4]);
      const float xa[4] = {x.x, x.y, x.z, x.w}, ya[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = __fmaf_rn(xa[u], ya[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t i = i0 + ty * 4 + u, j = j0 + tx * 4 + v;
      if (i < M && j < N) ep(i, j, acc[u][v]);
    }
}

// ---------------------------------------------------------------- K_proj: Y = B W_r
struct LoadB {
  const float* A;
  Shape s;
  bool q_fast;   // tall: B(i, q) = A[i n + q] is contiguous in q
  __device__ float operator()(int64_t i, int64_t q) const { return bval(A, s, i, q); }
};
struct LoadWrT {   // Bop(j, q) = Wr[q][j]: contiguous in j
  const float* Wr;
  int r;
  bool q_fast;
  __device__ float operator()(int64_t j, int64_t q) const { return Wr[q * r + j]; }
};
struct StoreY {
  float* Y;
  int r;
  __device__ void operator()(int64_t i, int64_t j, float v) const { Y[i * r + j] = v; }
};
__global__ void __launch_bounds__(NT) k_proj(const float* __restrict__ A, Shape s, const float* __restrict__ Wr,
                                            float* __restrict__ Y) {
  gemm_tile(s.L, s.r, s.k, LoadB{A, s, s.tall}, LoadWrT{Wr, s.r, false}, StoreY{Y, s.r});
}

// ---------------------------------------------------------------- K_sign (R30)
// Column j of U_A: tall -> Y[:, j] / sigma_j (L entries), wide -> Wr[:, j] (k entries).  The
// largest magnitude wins, ties -> lowest index: max over (|x| bits << 32 | ~index).
__global__ void __launch_bounds__(NT) k_sign(Shape s, const float* __restrict__ Y, const float* __restrict__ Wr,
                                            float* __restrict__ sign) {
  const int j = blockIdx.x;
  const float* col = s.tall ? Y : Wr;
  const int64_t len = s.tall ? s.L : s.k;
  unsigned long long best = 0;
  for (int64_t i = threadIdx.x; i < len; i += NT) {
    const float x = col[i * s.r + j];
    const unsigned long long key = ((unsigned long long)(__float_as_uint(x) & 0x7FFFFFFFu) << 32) |
                                   (unsigned long long)(0xFFFFFFFFu - (uint32_t)i);
    best = key > best ? key : best;
  }
  __shared__ unsigned long long sh[NT / 32];
  for (int o = 16; o; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xFFFFFFFFu, best, o);
    best = v > best ? v : best;
  }
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < NT / 32; ++w) best = sh[w] > best ? sh[w] : best;
    const uint32_t i = 0xFFFFFFFFu - (uint32_t)(best & 0xFFFFFFFFu);
    sign[j] = (best >> 32) == 0 ? 1.0f : (col[(int64_t)i * s.r + j] < 0.0f ? -1.0f : 1.0f);
  }
}

// ---------------------------------------------------------------- K_pack (R31)
// One grid-stride pass over the payload's binary16 elements: U_r [m][r], S_r [r], V_r [n][r]
// (+ zero padding of each section to 16 bytes).  tall: U = sign * Y / sigma, V = sign * Wr;
// wide: U = sign * Wr, V = sign * Y / sigma.  sigma = 0 -> that U / V column is 0 (R30).
__global__ void __launch_bounds__(NT) k_pack(Shape s, const float* __restrict__ Y, const float* __restrict__ Wr,
                                            const double* __restrict__ sigma, const float* __restrict__ sign,
                                            uint8_t* __restrict__ payload, uint32_t* flags) {
  const int64_t nU = s.m * s.r, nV = s.n * s.r;
  const int64_t oU = 16, oS = oU + ((2 * nU + 15) & ~15ll), oV = oS + ((2 * (int64_t)s.r + 15) & ~15ll);
  const int64_t end = oV + ((2 * nV + 15) & ~15ll);
  const int64_t halves = (end - 16) / 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    uint32_t* p = reinterpret_cast<uint32_t*>(payload);
    p[0] = 5u; p[1] = (uint32_t)s.m; p[2] = (uint32_t)s.n; p[3] = (uint32_t)s.r;
  }
  bool ovf = false;
  for (int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; h < halves; h += stride) {
    const int64_t byte = 16 + 2 * h;
    __half v = __float2half_rn(0.0f);
    if (byte < oU + 2 * nU) {
      const int64_t e = (byte - oU) / 2, i = e / s.r, j = e % s.r;
      const float sg = (float)sigma[j];
      float x;
      if (s.tall) x = sg == 0.0f ? 0.0f : __fdiv_rn(Y[i * s.r + j], sg);
      else x = Wr[i * s.r + j];
      v = __float2half_rn(__fmul_rn(x, sign[j]));
    } else if (byte >= oS && byte < oS + 2 * s.r) {
      const int64_t j = (byte - oS) / 2;
      v = __double2half(sigma[j]);
      ovf |= __hisinf(v) != 0;
    } else if (byte >= oV && byte < oV + 2 * nV) {
      const int64_t e = (byte - oV) / 2, i = e / s.r, j = e % s.r;
      const float sg = (float)sigma[j];
      float x;
      if (s.tall) x = Wr[i * s.r + j];
      else x = sg == 0.0f ? 0.0f : __fdiv_rn(Y[i * s.r + j], sg);
      v = __float2half_rn(__fmul_rn(x, sign[j]));
    }
    reinterpret_cast<__half*>(payload + 16)[h] = v;
  }
  if (ovf) atomicOr(flags, F_OVERFLOW);
}

// ---------------------------------------------------------------- K_recon: A' = (U_r S_r) V_r^T
struct LoadUS {   // Aop(i, q) = fl(U[i][q] * S[q]) — contiguous in q
  const __half* U;
  const __half* S;
  int r;
  bool q_fast;
  __device__ float operator()(int64_t i, int64_t q) const {
    return __fmul_rn(__half2float(U[i * r + q]), __half2float(S[q]));
  }
};
struct LoadV {    // Bop(j, q) = V[j][q] — contiguous in q
  const __half* V;
  int r;
  bool q_fast;
  __device__ float operator()(int64_t j, int64_t q) const { return __half2float(V[j * r + q]); }
};
struct StoreOut {
  float* out;
  int64_t n;
  __device__ void operator()(int64_t i, int64_t j, float v) const { out[i * n + j] = v; }
};
__global__ void __launch_bounds__(NT) k_recon(Shape s, const uint8_t* __restrict__ payload, float* __restrict__ out) {
  const int64_t nU = s.m * s.r;
  const int64_t oS = 16 + ((2 * nU + 15) & ~15ll), oV = oS + ((2 * (int64_t)s.r + 15) & ~15ll);
  const __half* U = reinterpret_cast<const __half*>(payload + 16);
  const __half* S = reinterpret_cast<const __half*>(payload + oS);
  const __half* V = reinterpret_cast<const __half*>(payload + oV);
  gemm_tile(s.m, s.n, s.r, LoadUS{U, S, s.r, true}, LoadV{V, s.r, true}, StoreOut{out, s.n});
}

}  // namespace nbsvd

using namespace nbsvd;

struct nebula_svd {
  Shape s{};
  int device = 0;
  cudaStream_t stream = nullptr;
  cusolverDnHandle_t solver = nullptr;
  double *G = nullptr, *lambda = nullptr, *work = nullptr, *sigma = nullptr;
  float *Wr = nullptr, *Y = nullptr, *sign = nullptr;
  int* info = nullptr;
  uint32_t* flags = nullptr;     // device sticky flags
  int2* tiles = nullptr;
  int ntiles = 0, splits = 1;
  int64_t rows_per_split = 0;
  int lwork = 0;
  int eig = 0;                   // 0: cusolverDnDsyevd (divide & conquer), 1: cusolverDnDsyevj (Jacobi)
  int gram_simt = 0;             // 0: FP64 tensor cores (DMMA, default), 1: SIMT fp64 FMA
  syevjInfo_t jinfo = nullptr;
  uint64_t launches = 0;
  std::string err;
};

static std::string g_svd_err;

static nebula_status svd_fail(nebula_svd* h, nebula_status st, const std::string& msg) {
  if (h) h->err = msg;
  else g_svd_err = msg;
  return st;
}

#define SVD_CK(h, x)                                                                          \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess) return svd_fail(h, NEBULA_ERR_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
  } while (0)

extern "C" {

// R29: r = clamp(floor(rho * min(m, n) + 1/2), 1, min(m, n)) — "r is the used ratio of the total
// singular values", rounded as R12.
int32_t nebula_svd_rank(int64_t m, int64_t n, double rho) {
  if (m < 1 || n < 1 || !(rho > 0.0 && rho <= 1.0)) return 0;
  const int64_t k = m < n ? m : n;
  double r = std::floor(rho * (double)k + 0.5);
  if (r < 1) r = 1;
  if (r > (double)k) r = (double)k;
  return (int32_t)r;
}

nebula_status nebula_svd_init_density(nebula_svd** out, int64_t m, int64_t n, double rho, int32_t device, void* stream) {
  if (!out) return svd_fail(nullptr, NEBULA_ERR_INVALID_ARG, "null out");
  *out = nullptr;
  const int32_t r = nebula_svd_rank(m, n, rho);
  if (r < 1) return svd_fail(nullptr, NEBULA_ERR_INVALID_ARG, "m, n must be >= 1 and rho in (0, 1]");
  return nebula_svd_init(out, m, n, r, device, stream);
}

nebula_status nebula_svd_init(nebula_svd** out, int64_t m, int64_t n, int32_t r, int32_t device, void* stream) {
  if (!out) return svd_fail(nullptr, NEBULA_ERR_INVALID_ARG, "null out");
  *out = nullptr;
  if (m < 1 || n < 1) return svd_fail(nullptr, NEBULA_ERR_INVALID_ARG, "m and n must be >= 1");
  const int64_t k = m < n ? m : n;
  if (k > 16384) return svd_fail(nullptr, NEBULA_ERR_INVALID_ARG, "min(m, n) must be <= 16384");
  if (r < 1 || r > k) return svd_fail(nullptr, NEBULA_ERR_INVALID_ARG, "r must be in [1, min(m, n)]");
  if (m >= (1ll << 31) || n >= (1ll << 31) || m * n >= (1ll << 40))
    return svd_fail(nullptr, NEBULA_ERR_INVALID_ARG, "matrix too large");
  if (device < 0) return svd_fail(nullptr, NEBULA_ERR_INVALID_ARG, "device must be >= 0");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device >= ndev)
    return svd_fail(nullptr, NEBULA_ERR_CUDA, "no CUDA device " + std::to_string(device));
  nebula_svd* h = new nebula_svd();
  h->device = device;
  h->stream = (cudaStream_t)stream;
  h->s.m = m; h->s.n = n; h->s.k = (int)k; h->s.r = r;
  h->s.L = m > n ? m : n;
  h->s.tall = m >= n;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  auto bail = [&](nebula_status st, const std::string& msg) {
    g_svd_err = msg;
    nebula_svd_destroy(h);
    cudaSetDevice(prev);
    return st;
  };
  // Gram tiling: upper-triangle 64 x 64 tiles; the contraction over L is split so the grid
  // covers the 148 SMs several times (fp64 atomics combine the split partial sums).
  const int nt = (int)((k + T - 1) / T);
  h->ntiles = nt * (nt + 1) / 2;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  int64_t want = (4ll * sms + h->ntiles - 1) / h->ntiles;
  int64_t max_split = (h->s.L + 4 * GK - 1) / (4 * GK);
  h->splits = (int)(want < 1 ? 1 : (want > max_split ? (max_split < 1 ? 1 : max_split) : want));
  h->rows_per_split = ((h->s.L + h->splits - 1) / h->splits + GK - 1) / GK * GK;
  h->splits = (int)((h->s.L + h->rows_per_split - 1) / h->rows_per_split);
  std::vector<int2> tl;
  for (int a = 0; a < nt; ++a)
    for (int b = a; b < nt; ++b) tl.push_back(make_int2(a, b));
  if (cudaMalloc(&h->tiles, sizeof(int2) * tl.size()) != cudaSuccess ||
      cudaMalloc(&h->G, sizeof(double) * k * k) != cudaSuccess || cudaMalloc(&h->lambda, sizeof(double) * k) != cudaSuccess ||
      cudaMalloc(&h->sigma, sizeof(double) * r) != cudaSuccess || cudaMalloc(&h->Wr, sizeof(float) * k * r) != cudaSuccess ||
      cudaMalloc(&h->Y, sizeof(float) * h->s.L * r) != cudaSuccess || cudaMalloc(&h->sign, sizeof(float) * r) != cudaSuccess ||
      cudaMalloc(&h->info, sizeof(int)) != cudaSuccess || cudaMalloc(&h->flags, 16) != cudaSuccess)
    return bail(NEBULA_ERR_OOM, "SVD workspace allocation failed");
  cudaMemcpy(h->tiles, tl.data(), sizeof(int2) * tl.size(), cudaMemcpyHostToDevice);
  cudaMemset(h->flags, 0, 16);
  if (cusolverDnCreate(&h->solver) != CUSOLVER_STATUS_SUCCESS) return bail(NEBULA_ERR_CUDA, "cusolverDnCreate failed");
  cusolverDnSetStream(h->solver, h->stream);
  if (cusolverDnDsyevd_bufferSize(h->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)k, h->G, (int)k,
                                  h->lambda, &h->lwork) != CUSOLVER_STATUS_SUCCESS)
    return bail(NEBULA_ERR_CUDA, "cusolverDnDsyevd_bufferSize failed");
  int lwj = 0;
  if (cusolverDnCreateSyevjInfo(&h->jinfo) != CUSOLVER_STATUS_SUCCESS ||
      cusolverDnXsyevjSetTolerance(h->jinfo, 1e-14) != CUSOLVER_STATUS_SUCCESS ||
      cusolverDnXsyevjSetMaxSweeps(h->jinfo, 30) != CUSOLVER_STATUS_SUCCESS ||
      cusolverDnDsyevj_bufferSize(h->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)k, h->G, (int)k,
                                  h->lambda, &lwj, h->jinfo) != CUSOLVER_STATUS_SUCCESS)
    return bail(NEBULA_ERR_CUDA, "cusolverDn syevj setup failed");
  if (lwj > h->lwork) h->lwork = lwj;
  if (cudaMalloc(&h->work, sizeof(double) * (h->lwork > 0 ? h->lwork : 1)) != cudaSuccess)
    return bail(NEBULA_ERR_OOM, "eigensolver workspace allocation failed");
  if (cudaDeviceSynchronize() != cudaSuccess) return bail(NEBULA_ERR_CUDA, "device sync after SVD init failed");
  cudaSetDevice(prev);
  *out = h;
  return NEBULA_OK;
}

nebula_status nebula_svd_payload_bytes(const nebula_svd* h, uint64_t* bytes) {
  if (!h || !bytes) return NEBULA_ERR_INVALID_ARG;
  auto p16 = [](uint64_t b) { return (b + 15) & ~uint64_t(15); };
  *bytes = 16 + p16(2ull * h->s.m * h->s.r) + p16(2ull * h->s.r) + p16(2ull * h->s.n * h->s.r);
  return NEBULA_OK;
}

nebula_status nebula_svd_compress(nebula_svd* h, const float* dev_A, void* dev_payload) {
  if (!h) return NEBULA_ERR_INVALID_ARG;
  if (!dev_A || !dev_payload) return svd_fail(h, NEBULA_ERR_INVALID_ARG, "null matrix or payload");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(h->device);
  const Shape s = h->s;
  SVD_CK(h, cudaMemsetAsync(h->G, 0, sizeof(double) * s.k * s.k, h->stream));
  const bool vec = (s.n % 4 == 0) && ((uintptr_t)dev_A % 16 == 0);
  if (!h->gram_simt)
    k_gram_dmma<<<dim3(h->ntiles, h->splits), GT, 0, h->stream>>>(dev_A, s, h->tiles, h->rows_per_split, h->G, h->flags, vec);
  else
    k_gram<<<dim3(h->ntiles, h->splits), NT, 0, h->stream>>>(dev_A, s, h->tiles, h->rows_per_split, h->G, h->flags, vec);
  ++h->launches;
  SVD_CK(h, cudaGetLastError());
  const cusolverStatus_t es =
      h->eig == 1 ? cusolverDnDsyevj(h->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, s.k, h->G, s.k, h->lambda,
                                     h->work, h->lwork, h->info, h->jinfo)
                  : cusolverDnDsyevd(h->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, s.k, h->G, s.k, h->lambda,
                                     h->work, h->lwork, h->info);
  if (es != CUSOLVER_STATUS_SUCCESS) {
    cudaSetDevice(prev);
    return svd_fail(h, NEBULA_ERR_CUDA, "cusolverDnDsyevd failed to launch");
  }
  const int64_t prep = (int64_t)s.k * s.r > s.r ? (int64_t)s.k * s.r : s.r;
  k_prep<<<(unsigned)((prep + 255) / 256), 256, 0, h->stream>>>(s, h->lambda, h->G, h->sigma, h->Wr);
  k_proj<<<dim3((unsigned)((s.r + T - 1) / T), (unsigned)((s.L + T - 1) / T)), NT, 0, h->stream>>>(dev_A, s, h->Wr, h->Y);
  k_sign<<<s.r, NT, 0, h->stream>>>(s, h->Y, h->Wr, h->sign);
  k_pack<<<4 * 148, NT, 0, h->stream>>>(s, h->Y, h->Wr, h->sigma, h->sign, (uint8_t*)dev_payload, h->flags);
  h->launches += 4;
  SVD_CK(h, cudaGetLastError());
  cudaSetDevice(prev);
  return NEBULA_OK;
}

nebula_status nebula_svd_decompress(nebula_svd* h, const void* dev_payload, float* dev_out) {
  if (!h) return NEBULA_ERR_INVALID_ARG;
  if (!dev_payload || !dev_out) return svd_fail(h, NEBULA_ERR_INVALID_ARG, "null payload or output");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(h->device);
  const Shape s = h->s;
  k_recon<<<dim3((unsigned)((s.n + T - 1) / T), (unsigned)((s.m + T - 1) / T)), NT, 0, h->stream>>>(
      s, (const uint8_t*)dev_payload, dev_out);
  ++h->launches;
  SVD_CK(h, cudaGetLastError());
  cudaSetDevice(prev);
  return NEBULA_OK;
}

nebula_status nebula_svd_check(nebula_svd* h) {
  if (!h) return NEBULA_ERR_INVALID_ARG;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(h->device);
  uint32_t f = 0;
  int info = 0;
  SVD_CK(h, cudaStreamSynchronize(h->stream));
  SVD_CK(h, cudaMemcpy(&f, h->flags, 4, cudaMemcpyDeviceToHost));
  SVD_CK(h, cudaMemcpy(&info, h->info, sizeof(int), cudaMemcpyDeviceToHost));
  SVD_CK(h, cudaMemset(h->flags, 0, 4));
  cudaSetDevice(prev);
  if (f & F_NONFINITE) return svd_fail(h, NEBULA_ERR_NONFINITE, "non-finite matrix entry");
  if (info != 0) return svd_fail(h, NEBULA_ERR_CUDA, "eigensolver did not converge (info " + std::to_string(info) + ")");
  if (f & F_OVERFLOW) return svd_fail(h, NEBULA_ERR_OVERFLOW, "a singular value overflows binary16 (>= 65520)");
  return NEBULA_OK;
}

nebula_status nebula_svd_set_stream(nebula_svd* h, void* stream) {
  if (!h) return NEBULA_ERR_INVALID_ARG;
  h->stream = (cudaStream_t)stream;
  if (h->solver) cusolverDnSetStream(h->solver, h->stream);
  return NEBULA_OK;
}

uint64_t nebula_svd_kernel_launches(const nebula_svd* h) { return h ? h->launches : 0; }

nebula_status nebula_svd_set_eigensolver(nebula_svd* h, int32_t which) {
  if (!h) return NEBULA_ERR_INVALID_ARG;
  if (which < 0 || which > 3) return svd_fail(h, NEBULA_ERR_INVALID_ARG, "eigensolver option must be in [0, 3]");
  h->eig = which & 1;
  h->gram_simt = (which >> 1) & 1;
  return NEBULA_OK;
}

nebula_status nebula_svd_destroy(nebula_svd* h) {
  if (!h) return NEBULA_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->jinfo) cusolverDnDestroySyevjInfo(h->jinfo);
  if (h->solver) cusolverDnDestroy(h->solver);
  cudaFree(h->G); cudaFree(h->lambda); cudaFree(h->work); cudaFree(h->sigma); cudaFree(h->Wr); cudaFree(h->Y);
  cudaFree(h->sign); cudaFree(h->info); cudaFree(h->flags); cudaFree(h->tiles);
  cudaSetDevice(prev);
  delete h;
  return NEBULA_OK;
}

const char* nebula_svd_last_error(const nebula_svd* h) { return h ? h->err.c_str() : g_svd_err.c_str(); }

}  // extern "C"
