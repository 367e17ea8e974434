// Day-1 integer-pipe microbenchmark for sm_100a.
//
// Measures, per SM per SM-clock, the sustained thread-op throughput of the
// instructions the Philox4x32-10 + nibble-acceptance path is made of:
//   mad.wide.u32 (IMAD.WIDE.U32), mad.lo.u32 (IMAD), mad.hi.u32 (IMAD.HI),
//   lop3.b32 (LOP3), iadd3, and a full Philox4x32-10 block.
// Each kernel runs 8 independent dependency chains per thread, 256 threads x
// 8 resident blocks per SM, exactly one wave of 148*8 blocks; cycles come from
// clock64() per block, so results are in ops/clk/SM independent of DVFS.
// Not part of the product; evidence for DESIGN.md's ALU roofline.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;
constexpr int CH = 8;

__global__ void k_madwide(uint64_t* out, long long* cyc, uint32_t m) {
  uint64_t p[CH];
  for (int c = 0; c < CH; ++c) p[c] = threadIdx.x * 7u + c;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(p[c]) : "r"((uint32_t)p[c]), "r"(m));
  }
  __syncthreads();
  long long t1 = clock64();
  uint64_t acc = 0;
  for (int c = 0; c < CH; ++c) acc ^= p[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_madlo(uint64_t* out, long long* cyc, uint32_t m) {
  uint32_t p[CH];
  for (int c = 0; c < CH; ++c) p[c] = threadIdx.x * 7u + c;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(p[c]) : "r"(m));
  }
  __syncthreads();
  long long t1 = clock64();
  uint64_t acc = 0;
  for (int c = 0; c < CH; ++c) acc ^= p[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_madhi(uint64_t* out, long long* cyc, uint32_t m) {
  uint32_t p[CH];
  for (int c = 0; c < CH; ++c) p[c] = threadIdx.x * 7u + c;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mad.hi.u32 %0, %0, %1, %0;" : "+r"(p[c]) : "r"(m));
  }
  __syncthreads();
  long long t1 = clock64();
  uint64_t acc = 0;
  for (int c = 0; c < CH; ++c) acc ^= p[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_lop3(uint64_t* out, long long* cyc, uint32_t m) {
  uint32_t p[CH];
  for (int c = 0; c < CH; ++c) p[c] = threadIdx.x * 7u + c;
  uint32_t q = m ^ threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(p[c]) : "r"(m), "r"(q));
  }
  __syncthreads();
  long long t1 = clock64();
  uint64_t acc = 0;
  for (int c = 0; c < CH; ++c) acc ^= p[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_iadd3(uint64_t* out, long long* cyc, uint32_t m) {
  uint32_t p[CH];
  for (int c = 0; c < CH; ++c) p[c] = threadIdx.x * 7u + c;
  uint32_t q = m ^ threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(p[c]) : "r"(m), "r"(q));
  }
  __syncthreads();
  long long t1 = clock64();
  uint64_t acc = 0;
  for (int c = 0; c < CH; ++c) acc ^= p[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// Mixed: one mad.wide + one lop3 per step (Philox's round shape).
__global__ void k_mix(uint64_t* out, long long* cyc, uint32_t m) {
  uint64_t p[CH];
  uint32_t x[CH];
  for (int c = 0; c < CH; ++c) { p[c] = threadIdx.x * 7u + c; x[c] = c; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(p[c]) : "r"(x[c]), "r"(m));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"((uint32_t)(p[c] >> 32)), "r"(m));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  uint64_t acc = 0;
  for (int c = 0; c < CH; ++c) acc ^= p[c] ^ x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__device__ __forceinline__ void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3,
                                             uint32_t k0, uint32_t k1) {
  uint64_t p0 = (uint64_t)0xD2511F53u * c0;
  uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
  uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
  uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
  c1 = (uint32_t)p1;
  c3 = (uint32_t)p0;
  c0 = n0;
  c2 = n2;
}

// Philox4x32-10 blocks, counter {x varying, row, t, colour} (uniform words as in the
// contract), outputs XOR-folded.  PHILOX_PER_THREAD blocks per thread.
constexpr int PB = 4096;
__global__ void k_philox(uint64_t* out, long long* cyc, uint32_t seed_lo, uint32_t seed_hi, uint32_t t) {
  uint32_t acc = 0;
  uint32_t row = blockIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int b = 0; b < PB; ++b) {
    uint32_t c0 = (uint32_t)(b * blockDim.x + threadIdx.x), c1 = row, c2 = t, c3 = 1;
    uint32_t k0 = seed_lo, k1 = seed_hi;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      philox_round(c0, c1, c2, c3, k0, k1);
      k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    acc ^= c0 ^ c1 ^ c2 ^ c3;
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int dev = 0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  int sms = pr.multiProcessorCount;
  printf("device %s sms %d cc %d.%d\n", pr.name, sms, pr.major, pr.minor);
  const int threads = 256, occ = 8, blocks = sms * occ;
  uint64_t* out; long long* cyc;
  CK(cudaMalloc(&out, sizeof(uint64_t) * blocks * threads));
  CK(cudaMalloc(&cyc, sizeof(long long) * blocks));
  long long* hc = new long long[blocks];
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct K { const char* name; int kind; double ops_per_thread; };
  K ks[] = {
    {"mad.wide.u32", 0, (double)ITERS * CH}, {"mad.lo.u32", 1, (double)ITERS * CH},
    {"mad.hi.u32", 2, (double)ITERS * CH},   {"lop3.b32", 3, (double)ITERS * CH},
    {"add.u32(x2)", 4, (double)ITERS * CH * 2}, {"madwide+lop3 (pairs)", 5, (double)ITERS * CH},
    {"philox4x32-10 blocks", 6, (double)PB},
  };
  for (auto& k : ks) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      switch (k.kind) {
        case 0: k_madwide<<<blocks, threads>>>(out, cyc, 0xD2511F53u); break;
        case 1: k_madlo<<<blocks, threads>>>(out, cyc, 0xD2511F53u); break;
        case 2: k_madhi<<<blocks, threads>>>(out, cyc, 0xD2511F53u); break;
        case 3: k_lop3<<<blocks, threads>>>(out, cyc, 0xD2511F53u); break;
        case 4: k_iadd3<<<blocks, threads>>>(out, cyc, 0xD2511F53u); break;
        case 5: k_mix<<<blocks, threads>>>(out, cyc, 0xD2511F53u); break;
        case 6: k_philox<<<blocks, threads>>>(out, cyc, 1u, 0u, 1u); break;
      }
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      CK(cudaMemcpy(hc, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost));
      double mean = 0; long long mx = 0;
      for (int b = 0; b < blocks; ++b) { mean += hc[b]; if (hc[b] > mx) mx = hc[b]; }
      mean /= blocks;
      // occ blocks share an SM: per-SM thread-ops per clk ~ occ*threads*ops / block_cycles
      double per_clk_sm = occ * threads * k.ops_per_thread / mean;
      double total = (double)blocks * threads * k.ops_per_thread;
      printf("%-24s rep %d: %8.3f ms  %9.2f Gop/s  %7.2f thread-ops/clk/SM (mean blk cyc %.0f, max %lld)  implied clk %.0f MHz\n",
             k.name, rep, ms, total / ms / 1e6, per_clk_sm, mean, mx, mx / (ms * 1e3));
    }
  }
  return 0;
}
