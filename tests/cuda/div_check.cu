// Exhaustive check of div_rn_fma (the SFU-free quotient of the QSGD quantiser,
// csrc/nebula_internal.cuh) against the IEEE division __fdiv_rn: for NS scales s (random
// significands plus the edge significands 1.0, 1.0 + 2^-23, 2 - 2^-23) and EVERY binary32
// significand of p in a window of exponents around s (|p / s| up to 2^8, below 2^-20, both
// signs), the two must return the same bits.  Prints "DIV_CHECK mismatches=<n> checked=<m>".
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#include "../../paper_2205_09470_b200/csrc/nebula_internal.cuh"

__global__ void k_check(const float* svals, int ns, int e_lo, int e_hi, unsigned long long* bad,
                        unsigned long long* checked) {
  const int si = blockIdx.y;
  const float s = svals[si];
  const float inv = __fdiv_rn(1.0f, s);
  const uint32_t sexp = (__float_as_uint(s) >> 23) & 0xFF;
  unsigned long long nbad = 0, n = 0;
  for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x; m < (1u << 23); m += gridDim.x * blockDim.x) {
    for (int de = e_lo; de <= e_hi; ++de) {
      const int pe = (int)sexp + de;
      if (pe < 1 || pe > 254) continue;
      for (int sg = 0; sg < 2; ++sg) {
        const float p = __uint_as_float(((uint32_t)sg << 31) | ((uint32_t)pe << 23) | m);
        const float a = nb::div_rn_fma(p, s, inv), b = __fdiv_rn(p, s);
        nbad += __float_as_uint(a) != __float_as_uint(b);
        ++n;
      }
    }
  }
  atomicAdd(bad, nbad);
  atomicAdd(checked, n);
}

int main(int argc, char** argv) {
  const int ns = argc > 1 ? atoi(argv[1]) : 256;
  float* hs = (float*)malloc(sizeof(float) * ns);
  uint64_t z = 0x9E3779B97F4A7C15ull;
  for (int i = 0; i < ns; ++i) {
    z = z * 6364136223846793005ull + 1442695040888963407ull;
    uint32_t mant = (uint32_t)(z >> 41);
    if (i == 0) mant = 0;
    if (i == 1) mant = 1;
    if (i == 2) mant = 0x7FFFFF;
    const int ex = 127 - 20 + (int)((z >> 20) % 40);   // s in [2^-20, 2^20)
    hs[i] = __builtin_bit_cast(float, ((uint32_t)ex << 23) | mant);
  }
  float* ds;
  unsigned long long *dbad, *dn;
  cudaMalloc(&ds, sizeof(float) * ns);
  cudaMalloc(&dbad, 8);
  cudaMalloc(&dn, 8);
  cudaMemcpy(ds, hs, sizeof(float) * ns, cudaMemcpyHostToDevice);
  cudaMemset(dbad, 0, 8);
  cudaMemset(dn, 0, 8);
  k_check<<<dim3(64, ns), 256>>>(ds, ns, -21, 8, dbad, dn);
  unsigned long long bad = 0, n = 0;
  cudaMemcpy(&bad, dbad, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(&n, dn, 8, cudaMemcpyDeviceToHost);
  const cudaError_t e = cudaGetLastError();
  printf("DIV_CHECK mismatches=%llu checked=%llu err=%s\n", bad, n, cudaGetErrorString(e));
  return (bad == 0 && e == cudaSuccess) ? 0 : 1;
}
