// ising_kernels.cuh — device-side layout, Philox and kernel parameter blocks.
//
// Layout (DESIGN.md §Data layout; §3.3): each colour plane of a slab
// is a row-major array of (R + 2) rows x W uint64 words, W = L_cols / 32.  Array
// row 0 is the top halo (global row row0 - 1 mod N), rows 1..R the slab's rows,
// row R + 1 the bottom halo (global row row0 + R mod N).  Lane k of word w (bits
// [4k, 4k+4)) holds plane column j = 16 w + k; nibble value 1 = spin +1,
// 0 = spin -1 ("-1/1 are mapped to 0/1").  Site (i, J) is black iff
// i + J is even and sits in plane column J / 2 (reading R1).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace ising {

constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

// Per-launch Philox key schedule (k0, k1 for each of the 10 rounds), computed on
// the host once per seed so the kernels read it from the constant bank.
struct PhiloxKeys {
  uint32_t k0[10];
  uint32_t k1[10];
};

// Acceptance parameters for one half-sweep.  Class a = number of neighbours
// aligned with the spin (0..4), e = s*h = 2a - 4.  thr[a] is the low 32 bits of
// the threshold T[e] (flip iff r < T[e]); bit a of always_mask marks T[e] = 2^32.
struct Accept {
  uint32_t thr[5];
  uint32_t always_mask;
  uint32_t keep3, keep4;  // Metropolis: 0 if T[a=3] / T[a=4] is 2^32, else ~0
  uint32_t nc_const;      // RULE 4: [r >= T3] + [r >= T4] per lane (draw-independent)
};

struct HalfSweepParams {
  uint64_t* tgt;          // target plane (colour c), padded (R + 2) x W
  const uint64_t* src;    // source plane (colour 1 - c), padded (R + 2) x W
  uint64_t* halo_up;      // destination row for local row 0 (upper slab's bottom halo) or null
  uint64_t* halo_dn;      // destination row for local row R - 1 (lower slab's top halo) or null
  int64_t W;              // words per plane row (multiple of 2)
  int64_t row0;           // global row of local row 0
  int32_t R;              // rows in the slab
  int32_t r_begin;        // first local row to update
  int32_t r_end;          // one past the last local row to update
  int32_t H;              // rows per work item (register-rolling band)
  int64_t items;          // number of work items = (W / 2) * ceil((r_end - r_begin) / H)
  int32_t tail_band8;     // staged kernel guided tail: first 8-row band (0: no tail)
  int32_t tail_band4;     //   first 4-row band
  int32_t tail_row4;      //   first row (relative to r_begin) of the 4-row bands
  int32_t tail_h1, tail_h2;  // tail band heights (8, 4)
  int32_t pdl;            // staged kernel launched as a programmatic dependent launch
  int32_t mirror;         // staged kernel: bands walk the rows bottom-up (row r -> r_begin +
                          // r_end - 1 - r): the first wave reads what the previous phase wrote last
  uint32_t t;             // sweep index (>= 1), or the offset added to *t_dev
  const uint32_t* t_dev;  // graph replays: device-resident sweep base (null otherwise)
  uint32_t colour;        // 0 black, 1 white
  PhiloxKeys keys;
  Accept acc;
  // Peer synchronisation of rank-p2p mode (all null otherwise).  The kernel starts when
  // both neighbours have finished phase wait_value (their halo stores into this slab are
  // done and they have finished reading the halo rows this launch overwrites), and its
  // last block publishes signal_value into the neighbours' flags after a system fence.
  const unsigned long long* wait_flags;  // this rank's [from_up, from_dn]
  unsigned long long wait_value;
  unsigned long long* signal_up;         // upper neighbour's from_dn flag (peer memory)
  unsigned long long* signal_dn;         // lower neighbour's from_up flag (peer memory)
  unsigned long long signal_value;
  unsigned int* done_counter;            // block counter for the last-block signal
  // white phase of a measured sweep: add [up count, antiparallel bonds] of the resulting
  // state into obs_out[0..1] (null: no measurement)
  unsigned long long* obs_out;
  const uint32_t* slot_dev;  // graph replays: device-resident sample index added to obs_out
  // black phase of a measured sweep: zero these two counters (the slot the white phase adds
  // into) — replaces a separate memset node between the sweeps of a measured chain
  unsigned long long* obs_clear;
};

// Persistent multi-sweep kernel for small lattices (one slab, one device).
struct PersistentParams {
  HalfSweepParams ph[2];          // black and white phase parameters
  uint32_t t0;                    // runs sweeps t0 + 1 .. t0 + n
  uint32_t n;
  unsigned int* bar_count;        // grid barrier state (zero-initialised)
  unsigned int* bar_gen;
  unsigned long long* obs_base;   // measured chain: slot k = after sweep (k + 1) * every
  uint32_t every;
};

// Rank-p2p synchronisation helpers (one thread each).
struct SyncParams {
  const unsigned long long* wait_flags;  // spin until all wait_count flags >= wait_value
  int wait_count;
  unsigned long long wait_value;
  unsigned long long* signal[2];         // then store signal_value into these (peer) flags
  unsigned long long signal_value;
};

// Observable all-reduce across ranks over peer memory: each rank stores its partials
// into slot `rank` of every rank's gather area, then spins until all slots carry epoch.
constexpr int kMaxRanks = 8;

// TMA-staged half-sweep: a block owns a span of kStageWords words of a row band (2 words per
// thread); widths that are a multiple of the span use it.  (The tile is static shared memory:
// (rows + 2) x kStageWords x 8 B must stay within 48 KB.)
#ifndef ISING_STAGE_WORDS
#define ISING_STAGE_WORDS 256
#endif
constexpr int kStageWords = ISING_STAGE_WORDS;
constexpr int kStageThreads = kStageWords / 2;
struct GatherParams {
  const unsigned long long* local;       // this rank's [up, anti] partials
  unsigned long long* slots[kMaxRanks];  // rank r's gather area: 2 parities x kMaxRanks x 3 u64
  unsigned long long* mine;              // this rank's gather area
  unsigned long long* out;               // summed [up, anti]
  int world;
  int rank;
  unsigned long long epoch;
};

struct InitParams {
  uint64_t* plane[2];
  int64_t W;
  int64_t row0;           // global row of local row 0
  int64_t N;              // total rows (for the halo wrap)
  int32_t R;
  int32_t cold;
  PhiloxKeys keys;
};

struct ObsParams {
  const uint64_t* black;
  const uint64_t* white;
  int64_t W;
  int64_t row0;
  int32_t R;
  unsigned long long* out;  // [0] = up count, [1] = antiparallel bonds
};

struct PackParams {
  uint64_t* plane[2];
  const int8_t* full;     // staging: rows [ra, rb) of the slab's padded row range, M bytes each
  int64_t W;
  int64_t M;
  int64_t row0;
  int64_t N;
  int32_t ra;             // first padded local row in staging (may be -1)
  int32_t rb;
  unsigned int* bad;      // set to 1 if a value is not -1/+1
};

// Bit-packed host format (ising_write_lattice_bits / ising_read_lattice_bits): bit (J & 7) of
// byte (i L_cols + J) / 8 is 1 for spin +1; staging rows of L_cols / 8 bytes.  One thread per
// 32 full columns = one 64-bit word of each colour plane.
struct PackBitsParams {
  uint64_t* plane[2];
  const uint32_t* bits;   // staging: rows [ra, rb) of the padded row range, W 32-bit words each
  int64_t W;
  int64_t row0;
  int64_t N;
  int32_t ra;             // first padded local row in staging (may be -1)
  int32_t rb;
};
struct UnpackBitsParams {
  const uint64_t* plane[2];
  uint32_t* bits;         // staging: rows [ra, rb) of the slab (interior rows only)
  int64_t W;
  int64_t row0;
  int32_t ra;
  int32_t rb;
};
cudaError_t launch_pack_bits(int grid, cudaStream_t st, const PackBitsParams& p);
cudaError_t launch_unpack_bits(int grid, cudaStream_t st, const UnpackBitsParams& p);

struct UnpackParams {
  const uint64_t* plane[2];
  int8_t* full;           // staging: rows [ra, rb) of the slab (interior rows only)
  int64_t W;
  int64_t M;
  int64_t row0;
  int32_t ra;
  int32_t rb;
};

// The basic byte-per-spin layout (ising_basic.cu, §3.1).
struct BasicParams {
  int8_t* lattice;           // target colour plane, nx x ny
  const int8_t* op_lattice;  // the other colour
  int64_t nx, ny;
  uint32_t t, colour;
  Accept acc;  // same threshold table / variant flags as the multi-spin path
  PhiloxKeys keys;
  unsigned long long* obs_out;  // white phase of a measured sweep: += [up, antiparallel] (or null)
};
// rule: kernel variant as for launch_halfsweep (0, 2, 4 Metropolis; 3, 5, 6, 1 heat bath).
// listing != 0 selects the per-site kernel that mirrors the Fig. 2 listing line by line.
cudaError_t launch_basic_halfsweep(int rule, int listing, int sms, cudaStream_t st,
                                   const BasicParams& p);
cudaError_t launch_basic_init(int grid, cudaStream_t st, int8_t* black, int8_t* white, int64_t nx,
                              int64_t ny, int cold, const PhiloxKeys& keys);
cudaError_t launch_basic_observables(int grid, cudaStream_t st, const int8_t* black,
                                     const int8_t* white, int64_t nx, int64_t ny,
                                     unsigned long long* out);
cudaError_t launch_basic_convert(int grid, cudaStream_t st, int8_t* black, int8_t* white,
                                 int8_t* full, int64_t ny, int64_t r0, int64_t rows, int to_full,
                                 unsigned int* bad);

// Batches of small lattices (ising_batch_*: temperature scans and the
// Binder analysis run many independent small lattices, which one-lattice launches leave
// launch-bound).  One CTA per lattice: both colour planes (N x W words each, no halo rows —
// the wrap is modular indexing) live in shared memory for a whole chunk of sweeps.
struct BatchLattice {
  PhiloxKeys keys;  // this lattice's seed
  Accept acc;       // this lattice's beta (thresholds as Accept of the generic kernels)
};
struct BatchParams {
  uint64_t* planes;                // lattice k: planes + k * 2 * N * W (black, then white)
  const BatchLattice* lat;         // one per lattice
  int32_t N, W;                    // rows, words per plane row
  uint32_t t0;                     // sweeps t0 + 1 .. t0 + sweeps
  uint32_t sweeps;
  uint32_t every;                  // > 0: observables after every `every` sweeps
  uint32_t n_samples;              // slots per lattice in obs
  uint32_t s_base;                 // sweeps of the call done before this launch: sample slot
                                   // of local sweep s is (s_base + s) / every - 1
  unsigned long long* obs;         // [lattice][sample][up, antiparallel] or null
  int32_t measure_only;            // 1: no sweeps, observables of the current state
};
constexpr int kBatchMaxThreads = 512;
// Row bands per lattice: a thread owns one 128-bit column pair of a band of consecutive rows,
// W / 2 pairs per row, at most kBatchMaxThreads threads (the CTA: batch_threads).
__host__ __device__ inline int batch_bands(int N, int W) {
  const int per = kBatchMaxThreads / (W / 2);
  return N < per ? N : per;
}
__host__ __device__ inline int batch_threads(int N, int W) {
  return (batch_bands(N, W) * (W / 2) + 31) / 32 * 32;
}
constexpr size_t kBatchMaxSmem = 200 * 1024;  // both planes, bytes
// variant: kernel variant shared by every lattice (0 / 2 / 3 / 5 / 6 / 7), 1 = generic heat bath
cudaError_t launch_batch_sweeps(int variant, int n_lattices, int threads, size_t smem,
                                cudaStream_t st, const BatchParams& p);
// Lattices beyond one CTA: a thread-block cluster of `cluster` CTAs per lattice.
cudaError_t launch_batch_cluster_sweeps(int variant, int n_lattices, int cluster, int threads,
                                        size_t smem, cudaStream_t st, const BatchParams& p);
cudaError_t launch_batch_init(int n_lattices, int cold, cudaStream_t st, const BatchParams& p);
cudaError_t launch_batch_unpack(int lattice, cudaStream_t st, const BatchParams& p, int8_t* full);
cudaError_t launch_batch_pack(int lattice, cudaStream_t st, const BatchParams& p, const int8_t* full,
                              unsigned int* bad);

// Host-side launchers (defined in ising_kernels.cu).
cudaError_t launch_sync(cudaStream_t st, const SyncParams& p);
cudaError_t launch_halfsweep_staged(int rule, int64_t slots, cudaStream_t st, HalfSweepParams p);
cudaError_t staged_occupancy(int* blocks_per_sm);
cudaError_t launch_persistent(int rule, int grid, cudaStream_t st, const PersistentParams& P);
cudaError_t persistent_occupancy(int* blocks_per_sm);
cudaError_t launch_set_u32(cudaStream_t st, uint32_t* dst, uint32_t v, int add);
cudaError_t launch_zero_u64(cudaStream_t st, unsigned long long* dst, int n);
cudaError_t preload_kernels();  // force-load every kernel of the slab / rank paths (lazy loading)
cudaError_t launch_copy_u64(cudaStream_t st, uint64_t* dst, const uint64_t* src, int64_t n);
cudaError_t launch_gather(cudaStream_t st, const GatherParams& p);
cudaError_t launch_halfsweep(int rule, int grid, cudaStream_t st, const HalfSweepParams& p);
cudaError_t halfsweep_occupancy(int* blocks_per_sm);
cudaError_t launch_philox_probe(int grid, cudaStream_t st, const PhiloxKeys& K,
                                uint32_t blocks_per_thread, unsigned int* sink);

}  // namespace ising
