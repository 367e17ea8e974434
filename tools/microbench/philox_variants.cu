// Philox4x32-10 implementation variants on sm_100a, timed with CUDA events
// (draws/ns) — evidence for the multiply strategy in DESIGN.md §5.
//   wide : hi/lo via one IMAD.WIDE.U32 (FMA-heavy pipe, 4 cycles per warp)
//   dfma : hi via DFMA.RZ on the FP64 pipe (2^52 magic), lo via IMAD
//   mix  : per round, product 0 via IMAD.WIDE and product 1 via DFMA + IMAD
//   hi/lo: hi via mul.hi.u32 (IMAD.HI, one FMA-heavy pass) and lo via an IMAD that ptxas
//          cannot fuse with it (c * (M - 1) + c), so the pair is not an IMAD.WIDE
// Each thread runs 4 independent blocks per iteration (the half-sweep's ILP).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;

struct Keys { uint32_t k0[10], k1[10]; uint32_t m0, m1; };

__device__ __forceinline__ uint32_t hi_dfma(uint32_t c, double mp, double cc) {
  const double x = __hiloint2double(0x43300000, (int)c);  // 2^52 + c
  return (uint32_t)__double2loint(__fma_rz(x, mp, cc));    // 2^52 + floor(c M / 2^32)
}

// V = 3: every hi half via DFMA.RZ with the operand pairs flowing between rounds (the
// XOR rewrites only the low word of the previous DFMA result, whose high word is the
// 2^52 exponent already), lo halves via IMAD.
__device__ __forceinline__ uint4 philox_flow(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                             const Keys& K, double mp0, double cc0, double mp1,
                                             double cc1) {
  double x0 = __hiloint2double(0x43300000, (int)c0);
  double x2 = __hiloint2double(0x43300000, (int)c2);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const double h0 = __fma_rz(x0, mp0, cc0);
    const double h1 = __fma_rz(x2, mp1, cc1);
    const uint32_t lo0 = (uint32_t)__double2loint(x0) * M0;
    const uint32_t lo1 = (uint32_t)__double2loint(x2) * M1;
    x0 = __hiloint2double(__double2hiint(h1), (int)((uint32_t)__double2loint(h1) ^ c1 ^ K.k0[r]));
    x2 = __hiloint2double(__double2hiint(h0), (int)((uint32_t)__double2loint(h0) ^ c3 ^ K.k1[r]));
    c1 = lo1;
    c3 = lo0;
  }
  return make_uint4((uint32_t)__double2loint(x0), c1, (uint32_t)__double2loint(x2), c3);
}

template <int V>
__device__ __forceinline__ uint4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, const Keys& K,
                                        double mp0, double cc0, double mp1, double cc1) {
  if (V >= 6) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      uint32_t hi0, lo0, hi1, lo1;
      if (V == 6) {
        hi0 = __umulhi(c0, M0); lo0 = c0 * M0; hi1 = __umulhi(c2, M1); lo1 = c2 * M1;
      } else if (V == 7) {
        asm("mul.hi.u32 %0, %1, %2;" : "=r"(hi0) : "r"(c0), "n"(M0));
        asm("mad.lo.u32 %0, %1, %2, %1;" : "=r"(lo0) : "r"(c0), "n"(M0 - 1));
        asm("mul.hi.u32 %0, %1, %2;" : "=r"(hi1) : "r"(c2), "n"(M1));
        asm("mad.lo.u32 %0, %1, %2, %1;" : "=r"(lo1) : "r"(c2), "n"(M1 - 1));
      } else {
        asm("mul.hi.u32 %0, %1, %2;" : "=r"(hi0) : "r"(c0), "n"(M0));
        asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(lo0) : "r"(c0), "n"(M0));
        asm("mul.hi.u32 %0, %1, %2;" : "=r"(hi1) : "r"(c2), "n"(M1));
        asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(lo1) : "r"(c2), "n"(M1));
      }
      const uint32_t n0 = hi1 ^ c1 ^ K.k0[r];
      const uint32_t n2 = hi0 ^ c3 ^ K.k1[r];
      c1 = lo1; c3 = lo0; c0 = n0; c2 = n2;
    }
    return make_uint4(c0, c1, c2, c3);
  }
  if (V == 3) return philox_flow(c0, c1, c2, c3, K, mp0, cc0, mp1, cc1);
  if (V == 4) return philox<0>(c0, c1, c2, c3, K, mp0, cc0, mp1, cc1);
  if (V == 5) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      const uint64_t p0 = (uint64_t)c0 * K.m0, p1 = (uint64_t)c2 * K.m1;
      const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ K.k0[r];
      const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ K.k1[r];
      c1 = (uint32_t)p1; c3 = (uint32_t)p0; c0 = n0; c2 = n2;
    }
    return make_uint4(c0, c1, c2, c3);
  }
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    if (V == 0) {
      const uint64_t p0 = (uint64_t)c0 * M0, p1 = (uint64_t)c2 * M1;
      hi0 = p0 >> 32; lo0 = (uint32_t)p0; hi1 = p1 >> 32; lo1 = (uint32_t)p1;
    } else if (V == 1) {
      hi0 = hi_dfma(c0, mp0, cc0); lo0 = c0 * M0;
      hi1 = hi_dfma(c2, mp1, cc1); lo1 = c2 * M1;
    } else {
      const uint64_t p0 = (uint64_t)c0 * M0;
      hi0 = p0 >> 32; lo0 = (uint32_t)p0;
      hi1 = hi_dfma(c2, mp1, cc1); lo1 = c2 * M1;
    }
    const uint32_t n0 = hi1 ^ c1 ^ K.k0[r];
    const uint32_t n2 = hi0 ^ c3 ^ K.k1[r];
    c1 = lo1; c3 = lo0; c0 = n0; c2 = n2;
  }
  return make_uint4(c0, c1, c2, c3);
}

template <int V>
__global__ void __launch_bounds__(128) k_philox(Keys K, uint32_t iters, uint32_t row, uint32_t t,
                                                double mp0, double cc0, double mp1, double cc1,
                                                uint32_t* out) {
  uint32_t acc = 0;
  const uint32_t base = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t c = base + 4 * gridDim.x * blockDim.x * it + b;
      // V = 4: two blocks on the IMAD.WIDE path and two on the DFMA flow path per thread
      const uint4 r = (V == 4 && b >= 2) ? philox_flow(c, row, t, 1u, K, mp0, cc0, mp1, cc1)
                                         : philox<V>(c, row, t, 1u, K, mp0, cc0, mp1, cc1);
      acc += r.x ^ (r.y * 3) ^ (r.z * 5) ^ (r.w * 7);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_dfma(double a, double b, double* out, int iters) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0));
  const int sms = pr.multiProcessorCount;
  Keys K; uint32_t k0 = 1, k1 = 0;
  for (int r = 0; r < 10; ++r) { K.k0[r] = k0; K.k1[r] = k1; k0 += W0; k1 += W1; }
  K.m0 = M0; K.m1 = M1;
  const double mp0 = (double)M0 / 4294967296.0, mp1 = (double)M1 / 4294967296.0;
  const double cc0 = 4503599627370496.0 - 1048576.0 * (double)M0;
  const double cc1 = 4503599627370496.0 - 1048576.0 * (double)M1;
  const int grid = sms * 16, threads = 128;
  const uint32_t iters = 256;
  uint32_t* out[9];
  for (int v = 0; v < 9; ++v) CK(cudaMalloc(&out[v], sizeof(uint32_t) * grid * threads));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[9] = {"wide", "dfma", "mix", "flow", "wide+flow", "wide(param M)", "umulhi+mul", "hi+mad(M-1)", "hi+lo asm"};
  for (int v = 0; v < 9; ++v) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(a);
      if (v == 0) k_philox<0><<<grid, threads>>>(K, iters, 7, 3, mp0, cc0, mp1, cc1, out[v]);
      if (v == 1) k_philox<1><<<grid, threads>>>(K, iters, 7, 3, mp0, cc0, mp1, cc1, out[v]);
      if (v == 2) k_philox<2><<<grid, threads>>>(K, iters, 7, 3, mp0, cc0, mp1, cc1, out[v]);
      if (v == 3) k_philox<3><<<grid, threads>>>(K, iters, 7, 3, mp0, cc0, mp1, cc1, out[v]);
      if (v == 4) k_philox<4><<<grid, threads>>>(K, iters, 7, 3, mp0, cc0, mp1, cc1, out[v]);
      if (v == 5) k_philox<5><<<grid, threads>>>(K, iters, 7, 3, mp0, cc0, mp1, cc1, out[v]);
      if (v == 6) k_philox<6><<<grid, threads>>>(K, iters, 7, 3, mp0, cc0, mp1, cc1, out[v]);
      if (v == 7) k_philox<7><<<grid, threads>>>(K, iters, 7, 3, mp0, cc0, mp1, cc1, out[v]);
      if (v == 8) k_philox<8><<<grid, threads>>>(K, iters, 7, 3, mp0, cc0, mp1, cc1, out[v]);
      cudaEventRecord(b); CK(cudaEventSynchronize(b)); CK(cudaGetLastError());
      float ms; cudaEventElapsedTime(&ms, a, b); if (rep && ms < best) best = ms;
    }
    const double draws = 16.0 * grid * threads * iters;
    printf("philox %-5s: %.3f ms  %.0f draws/ns\n", names[v], best, draws / (best * 1e6));
  }
  // correctness: all variants fold to the same values
  uint32_t* h = new uint32_t[9 * grid * threads];
  for (int v = 0; v < 9; ++v) CK(cudaMemcpy(h + v * grid * threads, out[v], 4 * grid * threads, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int i = 0; i < grid * threads; ++i)
    for (int v = 1; v < 9; ++v) bad += (h[i] != h[v * grid * threads + i]);
  printf("variants agree: %s (%d mismatches)\n", bad ? "NO" : "yes", bad);
  double* dout; CK(cudaMalloc(&dout, sizeof(double) * grid * threads));
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    k_dfma<<<grid, threads>>>(1.0000001, 1e-9, dout, 4096);
    cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("dfma: %.3f ms %.0f GDFMA/s\n", ms, 8.0 * 4096 * grid * threads / (ms * 1e6));
  }
  return 0;
}
