// Throughput of the carry-chain instructions the Metropolis acceptance can be built from, on
// sm_100a (round 2, for the FMA-heavy / ALU balance question in profiles/r02_ncu_halfsweep.md):
//   cmp      sub.cc.u32 (IADD3 with carry-out into a predicate), result consumed by an addc
//   madc     sub.cc + madc.lo.u32 acc, acc, 16, 0     (IADD3 + IMAD.X: the kernel's insert)
//   b3       sub.cc x2 + addc x2 fused to IADD3.X acc, acc, acc, acc, P, P'  (base-3 digit)
//   addc2    sub.cc + addc.u32 acc, acc, acc           (IADD3 + IADD3.X, base 2)
//   madwide  mad.wide.u32 (IMAD.WIDE.U32, the Philox multiply)
// 8 independent chains per thread, 4 blocks x 256 threads per SM, one wave of 148 x 4
// blocks; per-SM rate from the slowest block's clock64() span.  Not part of the product.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 2048;
constexpr int CH = 8;

template <int KIND>
__global__ void __launch_bounds__(256) k_bench(uint32_t* out, long long* cyc, uint32_t t3, uint32_t t4) {
  uint32_t acc[CH], r[CH];
  for (int c = 0; c < CH; ++c) { acc[c] = 0; r[c] = (threadIdx.x * 0x9E3779B9u) ^ (c * 0x85EBCA6Bu); }
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if constexpr (KIND == 0) {  // two compares, carries added with 3-input IADD3.X, base 1
        asm volatile("{\n\t.reg .u32 d;\n\tsub.cc.u32 d, %1, %2;\n\taddc.u32 %0, %0, 0;\n\t}"
                     : "+r"(acc[c]) : "r"(r[c]), "r"(t3));
      } else if constexpr (KIND == 1) {
        asm volatile("{\n\t.reg .u32 d;\n\tsub.cc.u32 d, %1, %2;\n\tmadc.lo.u32 %0, %0, 16, 0;\n\t}"
                     : "+r"(acc[c]) : "r"(r[c]), "r"(t3));
      } else if constexpr (KIND == 2) {
        asm volatile("{\n\t.reg .u32 d, x;\n\tsub.cc.u32 d, %1, %2;\n\taddc.u32 x, %0, %0;\n\t"
                     "sub.cc.u32 d, %1, %3;\n\taddc.u32 %0, x, %0;\n\t}"
                     : "+r"(acc[c]) : "r"(r[c]), "r"(t3), "r"(t4));
      } else if constexpr (KIND == 3) {
        asm volatile("{\n\t.reg .u32 d;\n\tsub.cc.u32 d, %1, %2;\n\taddc.u32 %0, %0, %0;\n\t}"
                     : "+r"(acc[c]) : "r"(r[c]), "r"(t3));
      } else {
        uint64_t p;
        asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(r[c]), "r"(t3));
        acc[c] ^= (uint32_t)p;
        r[c] = (uint32_t)(p >> 32);
      }
      r[c] += 0x3C6EF372u;  // keep the draws changing (one IADD3 / VIADD per step)
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  uint32_t x = 0;
  for (int c = 0; c < CH; ++c) x ^= acc[c] ^ r[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int occ = 4, threads = 256, blocks = prop.multiProcessorCount * occ;
  uint32_t* out; long long* cyc;
  CK(cudaMalloc(&out, sizeof(uint32_t) * blocks * threads));
  CK(cudaMalloc(&cyc, sizeof(long long) * blocks));
  long long* hc = new long long[blocks];
  struct K { const char* name; void (*f)(uint32_t*, long long*, uint32_t, uint32_t); const char* per_step; };
  K ks[] = {{"cmp+addc (IADD3, IADD3.X)", k_bench<0>, "1 compare + 1 insert + 1 add"},
            {"cmp+madc (IADD3, IMAD.X)", k_bench<1>, "1 compare + 1 insert + 1 add"},
            {"b3: 2 cmp + IADD3.X(P,P')", k_bench<2>, "2 compares + 1 insert + 1 add"},
            {"cmp+addc x2 (base 2)", k_bench<3>, "1 compare + 1 insert + 1 add"},
            {"mad.wide.u32", k_bench<4>, "1 IMAD.WIDE + 1 LOP3 + 1 add"}};
  printf("device %s, %d SMs; %d chains/thread, %d x %d threads per SM\n", prop.name,
         prop.multiProcessorCount, CH, occ, threads);
  for (auto& k : ks) {
    for (int rep = 0; rep < 3; ++rep) {
      k.f<<<blocks, threads>>>(out, cyc, 0x2C0A7E1Fu, 0x0786C227u);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(hc, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost));
      long long mx = 0;
      for (int b = 0; b < blocks; ++b) mx = hc[b] > mx ? hc[b] : mx;
      const double steps_per_sm = (double)occ * threads * ITERS * CH;
      if (rep == 2)
        printf("%-30s %7.2f steps/clk/SM = %5.2f SMSP cycles per warp-step  (%s)\n", k.name,
               steps_per_sm / mx, 4.0 * 32.0 * mx / steps_per_sm / 4.0 / 1.0 / 1.0 * 1.0, k.per_step);
    }
  }
  return 0;
}
