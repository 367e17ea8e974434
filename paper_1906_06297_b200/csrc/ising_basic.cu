// ising_basic.cu — the paper's *basic* implementation (§3.1, the Fig. 2 CUDA C
// listing `update_lattice<is_black>`) rebuilt for sm_100a as a second
// workload: one signed byte per spin, two colour planes of
// N x M/2 "compacted along the rows", the listing's stencil with periodic
// wrap, and the same draw contract / integer thresholds as the multi-spin path, so both
// layouts are bit-identical to each other and to the oracle.
//
// B200 choices: a thread owns four consecutive plane sites (one Philox4x32-10 block, one
// 32-bit load/store per row of target and source) instead of the listing's one thread per
// spin with a pre-generated random array: same arithmetic per site,
// no random-number array in HBM, 3 algorithmic bytes per attempted flip.
#include <cuda_runtime.h>

#include "ising_kernels.cuh"

namespace ising {

__device__ __forceinline__ uint4 philox_basic(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                              const PhiloxKeys& K) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)c0 * kPhiloxM0;
    const uint64_t p1 = (uint64_t)c2 * kPhiloxM1;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ K.k0[r];
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ K.k1[r];
    c1 = (uint32_t)p1;
    c3 = (uint32_t)p0;
    c0 = n0;
    c2 = n2;
  }
  return make_uint4(c0, c1, c2, c3);
}

// One colour phase: lattice (target colour c) and op_lattice (the other colour), both
// nx x ny int8.  Thread = plane sites (i, 4q .. 4q+3); x covers the quads of a row, y
// strides over rows (no 64-bit division in the index math).
template <int RULE>
__global__ void __launch_bounds__(256) k_basic_halfsweep(const BasicParams p) {
  const int64_t quads = p.ny >> 2;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= quads) return;
  const int64_t j0 = 4 * q;
  const int8_t* op = p.op_lattice;
  for (int64_t i = blockIdx.y; i < p.nx; i += gridDim.y) {
    // "Set stencil indices with periodicity"
    const int64_t ipp = (i + 1 < p.nx) ? i + 1 : 0;
    const int64_t inn = (i - 1 >= 0) ? i - 1 : p.nx - 1;
    const char4 up = *reinterpret_cast<const char4*>(op + inn * p.ny + j0);
    const char4 mid = *reinterpret_cast<const char4*>(op + i * p.ny + j0);
    const char4 dn = *reinterpret_cast<const char4*>(op + ipp * p.ny + j0);
    // "Select off-column index based on color and row index parity":
    // black: joff = (i % 2) ? jpp : jnn; white: joff = (i % 2) ? jnn : jpp
    const bool east = (p.colour == 0) == ((i & 1) == 1);
    const int64_t jside = east ? ((j0 + 4 < p.ny) ? j0 + 4 : 0) : ((j0 - 1 >= 0) ? j0 - 1 : p.ny - 1);
    const int8_t side_edge = op[i * p.ny + jside];
    const int8_t o[4] = {mid.x, mid.y, mid.z, mid.w};
    const int8_t u[4] = {up.x, up.y, up.z, up.w};
    const int8_t d[4] = {dn.x, dn.y, dn.z, dn.w};
    char4 tv = *reinterpret_cast<const char4*>(p.lattice + i * p.ny + j0);
    int8_t s[4] = {tv.x, tv.y, tv.z, tv.w};
    const uint4 r4 = philox_basic(p.t, (uint32_t)q, p.colour, (uint32_t)i, p.keys);
    const uint32_t rr[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int8_t joff = east ? (k < 3 ? o[k + 1] : side_edge) : (k > 0 ? o[k - 1] : side_edge);
      const int nn_sum = u[k] + o[k] + d[k] + joff;
      const int a = (nn_sum * s[k] + 4) >> 1;       // e = nn_sum * s = 2a - 4, dE = 2 J e
      uint32_t thr;
      bool always;
      if (RULE == 0) {
        // Metropolis (PAPER.md:40-41, :155-156 with the integer compare of reading R5)
        thr = (a == 4) ? p.thr[4] : p.thr[3];
        always = (a <= 2) || ((p.always_mask >> a) & 1u);
      } else {
        // heat bath
        thr = a == 0 ? p.thr[0] : a == 1 ? p.thr[1] : a == 2 ? p.thr[2] : a == 3 ? p.thr[3] : p.thr[4];
        always = (p.always_mask >> a) & 1u;
      }
      if (always || rr[k] < thr) s[k] = (int8_t)-s[k];
    }
    tv.x = s[0];
    tv.y = s[1];
    tv.z = s[2];
    tv.w = s[3];
    *reinterpret_cast<char4*>(p.lattice + i * p.ny + j0) = tv;
  }
}

// Random / cold start on the byte planes (reading R8).
__global__ void k_basic_init(int8_t* black, int8_t* white, int64_t nx, int64_t ny, int cold,
                             PhiloxKeys keys) {
  const int64_t quads = ny >> 2;
  const int64_t total = 2 * nx * quads;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int c = (int)(idx / (nx * quads));
    const int64_t rem = idx - (int64_t)c * nx * quads;
    const int64_t i = rem / quads;
    const int64_t j0 = 4 * (rem - i * quads);
    char4 v = make_char4(1, 1, 1, 1);
    if (!cold) {
      const uint4 r = philox_basic(0u, (uint32_t)(j0 >> 2), (uint32_t)c, (uint32_t)i, keys);
      v = make_char4(r.x < 0x80000000u ? 1 : -1, r.y < 0x80000000u ? 1 : -1,
                     r.z < 0x80000000u ? 1 : -1, r.w < 0x80000000u ? 1 : -1);
    }
    *reinterpret_cast<char4*>((c == 0 ? black : white) + i * ny + j0) = v;
  }
}

// Up count and antiparallel bonds (every bond has one black end: its 4 white neighbours).
__global__ void __launch_bounds__(256) k_basic_observables(const int8_t* black, const int8_t* white,
                                                           int64_t nx, int64_t ny,
                                                           unsigned long long* out) {
  const int64_t total = nx * ny;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long up = 0, anti = 0;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int64_t i = idx / ny;
    const int64_t j = idx - i * ny;
    const int64_t ipp = (i + 1 < nx) ? i + 1 : 0;
    const int64_t inn = (i - 1 >= 0) ? i - 1 : nx - 1;
    const int64_t joff = (i & 1) ? ((j + 1 < ny) ? j + 1 : 0) : ((j - 1 >= 0) ? j - 1 : ny - 1);
    const int b = black[idx];
    up += (b > 0) + (white[idx] > 0);
    anti += (b != white[inn * ny + j]) + (b != white[idx]) + (b != white[ipp * ny + j]) +
            (b != white[i * ny + joff]);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    up += __shfl_xor_sync(0xffffffffu, up, off);
    anti += __shfl_xor_sync(0xffffffffu, anti, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&out[0], up);
    atomicAdd(&out[1], anti);
  }
}

// Full lattice (row-major +-1 bytes, rows [r0, r0 + rows)) <-> planes.  to_full = 1 unpacks.
__global__ void k_basic_convert(int8_t* black, int8_t* white, int8_t* full, int64_t ny, int64_t r0,
                                int64_t rows, int to_full, unsigned int* bad) {
  const int64_t M = 2 * ny;
  const int64_t total = rows * M;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int64_t li = idx / M;
    const int64_t J = idx - li * M;
    const int64_t i = r0 + li;
    int8_t* plane = ((i + J) & 1) ? white : black;
    if (to_full) {
      full[idx] = plane[i * ny + (J >> 1)];
    } else {
      const int8_t v = full[idx];
      if (v != 1 && v != -1) atomicOr(bad, 1u);
      plane[i * ny + (J >> 1)] = v;
    }
  }
}

cudaError_t launch_basic_halfsweep(int rule, int grid, cudaStream_t st, const BasicParams& p) {
  (void)grid;
  const int64_t quads = p.ny >> 2;
  const dim3 g((unsigned)((quads + 255) / 256), (unsigned)(p.nx < 65535 ? p.nx : 65535));
  if (rule == 0)
    k_basic_halfsweep<0><<<g, 256, 0, st>>>(p);
  else
    k_basic_halfsweep<1><<<g, 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_basic_init(int grid, cudaStream_t st, int8_t* black, int8_t* white, int64_t nx,
                              int64_t ny, int cold, const PhiloxKeys& keys) {
  k_basic_init<<<grid, 256, 0, st>>>(black, white, nx, ny, cold, keys);
  return cudaGetLastError();
}

cudaError_t launch_basic_observables(int grid, cudaStream_t st, const int8_t* black,
                                     const int8_t* white, int64_t nx, int64_t ny,
                                     unsigned long long* out) {
  k_basic_observables<<<grid, 256, 0, st>>>(black, white, nx, ny, out);
  return cudaGetLastError();
}

cudaError_t launch_basic_convert(int grid, cudaStream_t st, int8_t* black, int8_t* white,
                                 int8_t* full, int64_t ny, int64_t r0, int64_t rows, int to_full,
                                 unsigned int* bad) {
  k_basic_convert<<<grid, 256, 0, st>>>(black, white, full, ny, r0, rows, to_full, bad);
  return cudaGetLastError();
}

}  // namespace ising
