// ising_runtime.cu — host runtime behind include/ising.h.
//
// Owns the per-device slabs (two padded colour planes each), streams, events,
// the NCCL communicator of rank mode, the host-side threshold table and the sweep
// counter.  Every step of the path runs in the kernels of ising_kernels.cu; this
// file only allocates, launches, synchronises and exchanges halo rows.
//
// Multi-GPU (§4): the lattice is split into row
// slabs.  Handle modes:
//   LOCAL (ising_create / ising_create_slabs): one process drives every slab; the
//     half-sweep kernel stores its boundary rows straight into the neighbouring
//     slab's halo row (same device, or a peer device over NVLink P2P), and each
//     phase waits on the neighbours' previous phase (RAW on the halo it reads, WAR
//     on the halo it writes).
//   RANK-P2P (ising_create_rank_p2p, the default of bench.py --gpus N): one process
//     per GPU; the neighbours' planes and flag words are mapped through CUDA IPC, the
//     half-sweep kernel stores its boundary rows into the neighbours' halo rows over
//     NVLink, waits for / raises phase flags in peer memory (prologue / last block).
//   RANK (ising_create_rank): one process per GPU; per phase the two boundary
//     rows are updated first, then ncclSend/ncclRecv move them on a comm stream
//     while the interior rows update (the classic halo/bulk overlap the paper cites,
//     PAPER.md:224).
// Small single-device lattices replay CUDA graphs (plain and measured chains); the basic
// byte-per-spin layout (ising_create_basic, §3.1) has its own kernels.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>
#include <nvtx3/nvToolsExt.h>
#include <sched.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/ising.h"
#include "ising_kernels.cuh"

namespace ising {
__global__ void k_init(const InitParams p);
__global__ void k_observables(const ObsParams p);
__global__ void k_pack(const PackParams p);
__global__ void k_unpack(const UnpackParams p);
}  // namespace ising

using namespace ising;

namespace {

thread_local std::string g_last_error;

void nvtx_yield() { sched_yield(); }

// NVTX ranges (SURVEY §5 tracing): one per API call that enqueues sweeps and one per
// half-sweep launch, visible in nsys / ncu timelines; no cost without a tool attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  NvtxRange(const char* fmt, long long a, long long b) {
    char buf[96];
    snprintf(buf, sizeof buf, fmt, a, b);
    nvtxRangePushA(buf);
  }
  ~NvtxRange() { nvtxRangePop(); }
};

int fail_cuda(cudaError_t e, const char* what, int line) {
  char buf[512];
  snprintf(buf, sizeof buf, "%s: %s (ising_runtime.cu:%d)", what, cudaGetErrorString(e), line);
  g_last_error = buf;
  return e == cudaErrorMemoryAllocation ? ISING_ERR_OOM : ISING_ERR_CUDA;
}

int fail_nccl(ncclResult_t r, const char* what, int line) {
  char buf[512];
  snprintf(buf, sizeof buf, "%s: %s (ising_runtime.cu:%d)", what, ncclGetErrorString(r), line);
  g_last_error = buf;
  return ISING_ERR_NCCL;
}

#define CU(x)                                                  \
  do {                                                         \
    cudaError_t e_ = (x);                                      \
    if (e_ != cudaSuccess) return fail_cuda(e_, #x, __LINE__); \
  } while (0)

#define NC(x)                                                   \
  do {                                                          \
    ncclResult_t r_ = (x);                                      \
    if (r_ != ncclSuccess) return fail_nccl(r_, #x, __LINE__);  \
  } while (0)

#define TRY(x)                 \
  do {                         \
    int s_ = (x);              \
    if (s_ != ISING_OK) return s_; \
  } while (0)

constexpr size_t kStagingBytes = size_t(64) << 20;  // pack/unpack staging chunk
#ifndef ISING_VPT
#define ISING_VPT 1
#endif
constexpr int64_t kWordsPerItem = 2 * ISING_VPT;  // must match the kernel's kWords
constexpr size_t kSyncBytes = 4096;                   // rank-p2p flags + gather area
constexpr int kGatherOffset = 8;                      // u64 index of the gather area
static_assert((kGatherOffset + 2 * 3 * ising::kMaxRanks) * 8 <= (int)kSyncBytes,
              "gather slots (2 parities x kMaxRanks x 3 u64) must fit the sync buffer");
constexpr int64_t kMaxProfiledLaunches = 4096;        // profiling times the first launches
constexpr uint32_t kIpcMagic = 0x49534e47u;           // "ISNG"

struct IpcBlob {  // ising_ipc_handle payload (<= ISING_IPC_BLOB_BYTES)
  uint32_t magic;
  int32_t rank, world, pad;
  int64_t R, W;
  cudaIpcMemHandle_t plane[2];
  cudaIpcMemHandle_t sync;
  unsigned char uuid[16];  // the exporting rank's GPU (ranks of several processes may share one)
};
static_assert(sizeof(IpcBlob) <= ISING_IPC_BLOB_BYTES, "IPC blob too large");

static bool env_is_zero(const char* name) {
  const char* v = getenv(name);
  return v && v[0] == '0';
}
static bool env_is_one(const char* name) {
  const char* v = getenv(name);
  return v && v[0] == '1';
}

struct Device {
  int dev = -1;
  int sms = 0;
  int hs_blocks_per_sm = 0;  // occupancy of k_halfsweep<0>
  int staged_blocks_per_sm = 0;  // occupancy of k_halfsweep_staged<0>
  cudaStream_t stream = nullptr;
  cudaStream_t comm = nullptr;
  cudaEvent_t ev_phase = nullptr;  // end of the latest phase on this device
  cudaEvent_t ev_bnd = nullptr;    // rank mode: boundary rows done
  cudaEvent_t ev_comm = nullptr;   // rank mode: halo exchange done
  cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr;
  // host <-> device staging of the +-1 byte lattice, double-buffered: chunk k uses buffer
  // k & 1; copies run on `copy`, pack / unpack kernels on `stream`, ordered by the events
  // (ev_copy[b]: last copy through buffer b done; ev_stage[b]: last kernel on b done)
  int8_t* staging[2] = {nullptr, nullptr};
  size_t staging_bytes = 0;
  cudaStream_t copy = nullptr;
  cudaEvent_t ev_copy[2] = {nullptr, nullptr}, ev_stage[2] = {nullptr, nullptr};
  unsigned long long* red = nullptr;  // [0] up, [1] antiparallel, [2] bad-value flag
  unsigned long long* meas = nullptr; // ising_sweep_measure: 2 per sample
  size_t meas_cap = 0;
};

struct Slab {
  int devi = 0;      // index into ctx->devs
  int64_t row0 = 0;  // global row of local row 0
  int64_t R = 0;
  uint64_t* plane[2] = {nullptr, nullptr};  // (R + 2) x W words each
};

}  // namespace

// One ising_sweep_measure_async call whose results are still in flight.
struct PendingMeasure {
  int64_t ticket = -1;  // -1: free slot
  int64_t* up = nullptr;
  int64_t* energy = nullptr;
  int64_t n = 0;
  bool ready = false;   // completed synchronously (fallback path): nothing to wait for
  double ms = 0;
  cudaEvent_t t0 = nullptr, t1 = nullptr, done = nullptr;
  unsigned long long* host = nullptr;  // pinned landing buffer of the [up, anti] pairs
  size_t host_cap = 0;                 // in pairs
};
constexpr int kMaxPending = 8;

struct ising_ctx {
  int64_t N = 0, M = 0, W = 0;
  uint64_t seed = 0;
  bool rank_mode = false;
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  bool comm_aborted = false;  // an asynchronous NCCL error aborted comm: every later call fails
  std::vector<Device> devs;
  std::vector<Slab> slabs;
  std::vector<int> slab_of_rank;  // unused in local mode
  int rule = ISING_RULE_METROPOLIS;
  double beta = 0;
  bool beta_set = false, state_set = false;
  uint64_t T[5] = {0, 0, 0, 0, 0};
  Accept acc{};
  PhiloxKeys keys{};
  uint64_t t = 0;
  double last_ms = 0;
  bool profiling = false;
  bool prof_active = false;  // inside ising_sweep with profiling on: launches are timed
  double kernel_ms = 0;
  int64_t kernel_launches = 0;
  int64_t launch_count = 0;
  std::vector<cudaEvent_t> prof_events;
  int rows_per_item_override = 0;
  // rank-p2p transport (ising_create_rank_p2p): halos by peer stores, flags in peer memory
  bool p2p = false, connected = false;
  // world == 1 rank handles with ISING_SELF_EXCHANGE=1: the rank is its own neighbour through
  // the full protocol (p2p: flags / fences / peer-store path; NCCL: a one-rank communicator
  // with self send / recv of the halo rows) — the per-GPU cost of each transport, measured
  // on one device
  bool self_exchange = false;
  unsigned long long* sync = nullptr;      // [0] from_up, [1] from_dn, [8 + 3 r ..] gather
  unsigned int* done_counter = nullptr;
  uint64_t* up_plane[2] = {nullptr, nullptr};
  uint64_t* dn_plane[2] = {nullptr, nullptr};
  unsigned long long* peer_sync[kMaxRanks] = {};
  std::vector<void*> opened;               // IPC mappings to close
  // rank-lsa transport (ising_create_rank_lsa): the planes and the flag area live in NCCL
  // symmetric memory (ncclMemAlloc + ncclCommWindowRegister) and the neighbours' addresses
  // come from the NCCL device API (ncclGetLsaPointer) instead of CUDA IPC
  bool lsa = false;
  ncclWindow_t win[3] = {nullptr, nullptr, nullptr};  // plane 0, plane 1, sync
  unsigned long long phase = 0;            // completed phases (init/write count as one)
  unsigned long long gather_epoch = 0;
  // CUDA graph of kGraphSweeps sweeps for small lattices (launch-bound), single device
  cudaGraphExec_t gexec = nullptr;
  uint32_t* t_dev = nullptr;               // device-resident sweep base read by the kernels
  int64_t graph_launches = 0;              // kernel nodes per graph replay
  cudaGraphExec_t gexec_meas = nullptr;    // measured-chain graph (ising_sweep_measure)
  int64_t meas_every = 0, meas_samples = 0, meas_graph_launches = 0;
  unsigned long long* meas_base = nullptr;
  bool graphs_enabled = true;
  bool persistent_enabled = false;         // opt-in (ISING_PERSISTENT=1): measured slower
                                           // than graph replay on B200 (grid barrier ~3 us)
  bool staged = true;                      // TMA-staged half-sweep (ISING_STAGED=0: off)
  bool guided_tail = !env_is_zero("ISING_TAIL");  // staged kernel: 8- / 4-row last waves
  bool pdl = !env_is_zero("ISING_PDL");  // staged kernel: programmatic dependent launch
  // staged kernel: white phases walk the bands bottom-up (ISING_MIRROR=0: off); C3 1552 ->
  // 1567, 16384 x 32768 1515 -> 1542 flips/ns (profiles/r02_ncu_halfsweep.md)
  bool mirror = !env_is_zero("ISING_MIRROR");
  // heat-bath variant 7 (ISING_HB_SYMMETRIC=0: off, for every handle type)
  bool symmetric_hb_enabled = !env_is_zero("ISING_HB_SYMMETRIC");
  bool draw_free_enabled = true;           // beta in {0, inf}: skip Philox (ISING_DRAW_FREE=0)
  unsigned int* bar = nullptr;             // persistent kernel's grid barrier state
  int persist_blocks_per_sm = 0;
  // basic byte-per-spin layout (ising_create_basic; §3.1)
  bool basic = false;
  int8_t* bplane[2] = {nullptr, nullptr};
  PendingMeasure pending[kMaxPending];
  int64_t next_ticket = 0;
  // ISING_TRACE=file.csv: timing events around the pieces of the first kMaxTracedPhases
  // half-sweeps (boundary rows, halo transfer on the comm stream, interior), written at
  // destroy as "phase,name,stream,ms" relative to the first event — a timeline of the
  // halo / interior overlap without a system profiler
  std::string trace_path;
  struct TraceEvent {
    int64_t phase;
    const char* name;
    const char* stream;
    cudaEvent_t ev;
  };
  std::vector<TraceEvent> trace;
  int64_t traced_phases = 0;
};
constexpr int64_t kMaxTracedPhases = 64;

namespace {

// ------------------------------------------------------------ thresholds
// Reading R5: u = r 2^-32 < P  <=>  r < ceil(2^32 P) (ldexp is exact; the only
// rounding is the host libm exp).  2^32 encodes "always".
uint64_t ceil_2p32(double P) {
  if (!(P > 0.0)) return 0;
  if (P >= 1.0) return uint64_t(1) << 32;
  const double x = std::ceil(std::ldexp(P, 32));
  if (x >= 4294967296.0) return uint64_t(1) << 32;
  return (uint64_t)x;
}

void compute_thresholds(double beta, int rule, uint64_t T[5]) {
  for (int a = 0; a < 5; ++a) {
    const int e = 2 * a - 4;  // e = s * h, dE = 2 e (J = 1)
    double P;
    if (rule == ISING_RULE_METROPOLIS) {
      // accept if dE <= 0, else with exp(-beta dE)
      P = (e <= 0) ? 1.0 : (std::isinf(beta) ? 0.0 : std::exp(-2.0 * beta * (double)e));
    } else {
      // heat bath: exp(-beta dE) / (exp(-beta dE) + 1)
      if (std::isinf(beta)) {
        P = e < 0 ? 1.0 : (e == 0 ? 0.5 : 0.0);
      } else {
        const double p = std::exp(-2.0 * beta * (double)e);
        P = std::isinf(p) ? 1.0 : p / (p + 1.0);
      }
    }
    T[a] = ceil_2p32(P);
  }
}

// The kernels' form of a threshold table: low 32 bits, "always" (2^32) classes as a mask
// (and, for Metropolis, as keep masks of the generic kernel).
Accept make_accept(const uint64_t T[5]) {
  Accept acc{};
  acc.keep3 = acc.keep4 = 0xffffffffu;
  for (int a = 0; a < 5; ++a) {
    if (T[a] >= (uint64_t(1) << 32)) {
      acc.always_mask |= 1u << a;
      acc.thr[a] = 0xffffffffu;
      if (a == 3) acc.keep3 = 0;
      if (a == 4) acc.keep4 = 0;
    } else {
      acc.thr[a] = (uint32_t)T[a];
    }
  }
  // draw-free Metropolis (beta = 0 or inf): T = 0 contributes one "no flip" per class
  acc.nc_const = (T[3] == 0 ? 0x11111111u : 0u) + (T[4] == 0 ? 0x11111111u : 0u);
  return acc;
}

void make_keys(uint64_t seed, PhiloxKeys* K) {
  uint32_t k0 = (uint32_t)(seed & 0xffffffffu), k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    K->k0[r] = k0;
    K->k1[r] = k1;
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
  }
}

// Size limits (include/ising.h).  The draw counter (reading R6) carries the global row in a
// 32-bit word and the plane column j / 4 = M / 8 at most in another, so L_rows <= 2^32 and
// L_cols <= 2^35 keep every site's counter distinct; slab rows are int32 in the kernels'
// row arithmetic (with margins for the halo rows and band heights), so R <= 2^30.
constexpr int64_t kMaxRows = int64_t(1) << 32;
constexpr int64_t kMaxCols = int64_t(1) << 35;
constexpr int64_t kMaxSlabRows = int64_t(1) << 30;

int check_shape(int64_t N, int64_t M, int n_slabs) {
  if (N < 2 || (N & 1) || M < 64 || (M % 64) != 0 || ((M / 32) % kWordsPerItem) != 0 ||
      n_slabs < 1 || N % n_slabs != 0 || N / n_slabs < 2) {
    g_last_error = "shape: need L_rows even, L_rows % n == 0, L_rows/n >= 2, L_cols % 64 == 0";
    return ISING_ERR_ARG;
  }
  if (N > kMaxRows || M > kMaxCols || N / n_slabs > kMaxSlabRows) {
    g_last_error = "shape: need L_rows <= 2^32, L_cols <= 2^35, L_rows / n <= 2^30";
    return ISING_ERR_ARG;
  }
  return ISING_OK;
}

int setup_device(Device& d, int dev) {
  int ndev = 0;
  CU(cudaGetDeviceCount(&ndev));
  if (dev < 0 || dev >= ndev) {
    g_last_error = "device index out of range";
    return ISING_ERR_DEVICE;
  }
  cudaDeviceProp pr;
  CU(cudaGetDeviceProperties(&pr, dev));
  if (pr.major != 10) {
    g_last_error = std::string("device is not sm_100 (Blackwell B200): ") + pr.name;
    return ISING_ERR_DEVICE;
  }
  d.dev = dev;
  d.sms = pr.multiProcessorCount;
  CU(cudaSetDevice(dev));
  CU(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithFlags(&d.comm, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithFlags(&d.copy, cudaStreamNonBlocking));
  for (int b = 0; b < 2; ++b) {
    CU(cudaEventCreateWithFlags(&d.ev_copy[b], cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&d.ev_stage[b], cudaEventDisableTiming));
  }
  CU(cudaEventCreateWithFlags(&d.ev_phase, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&d.ev_bnd, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&d.ev_comm, cudaEventDisableTiming));
  CU(cudaEventCreate(&d.ev_t0));
  CU(cudaEventCreate(&d.ev_t1));
  CU(cudaMalloc(&d.red, 4 * sizeof(unsigned long long)));
  CU(halfsweep_occupancy(&d.hs_blocks_per_sm));
  if (d.hs_blocks_per_sm < 1) d.hs_blocks_per_sm = 1;
  CU(staged_occupancy(&d.staged_blocks_per_sm));
  if (d.staged_blocks_per_sm < 1) d.staged_blocks_per_sm = 1;
  {  // once per device and process (see preload_kernels)
    static std::mutex mu;
    static std::vector<bool> loaded;
    std::lock_guard<std::mutex> lock(mu);
    if ((int)loaded.size() <= dev) loaded.resize(dev + 1, false);
    if (!loaded[dev]) {
      CU(preload_kernels());
      loaded[dev] = true;
    }
  }
  return ISING_OK;
}

int alloc_slabs(ising_ctx* h) {
  for (auto& s : h->slabs) {
    CU(cudaSetDevice(h->devs[s.devi].dev));
    const size_t bytes = (size_t)(s.R + 2) * (size_t)h->W * sizeof(uint64_t);
    for (int c = 0; c < 2; ++c) {
      CU(cudaMalloc(&s.plane[c], bytes));
      CU(cudaMemsetAsync(s.plane[c], 0, bytes, h->devs[s.devi].stream));
    }
  }
  for (auto& d : h->devs) {
    CU(cudaSetDevice(d.dev));
    CU(cudaStreamSynchronize(d.stream));
  }
  return ISING_OK;
}

// The neighbours' plane addresses and every rank's flag area in this rank's address space,
// from the NCCL device API (LSA pointers of symmetric windows); out[0..1] up planes,
// out[2..3] down planes, out[4 + q] rank q's sync area.
__global__ void k_lsa_pointers(ncclWindow_t w0, ncclWindow_t w1, ncclWindow_t ws, int up, int dn,
                               const int* lsa_rank, int world, void** out) {
  out[0] = ncclGetLsaPointer(w0, 0, up);
  out[1] = ncclGetLsaPointer(w1, 0, up);
  out[2] = ncclGetLsaPointer(w0, 0, dn);
  out[3] = ncclGetLsaPointer(w1, 0, dn);
  for (int q = 0; q < world; ++q) out[4 + q] = ncclGetLsaPointer(ws, 0, lsa_rank[q]);
}

cudaError_t lsa_peer_pointers(cudaStream_t st, const ncclWindow_t win[3], int up, int dn,
                              const int* lsa_rank, int world, void** host_out) {
  int* d_rank = nullptr;
  void** d_out = nullptr;
  cudaError_t e = cudaMalloc(&d_rank, sizeof(int) * kMaxRanks);
  if (e == cudaSuccess) e = cudaMalloc(&d_out, sizeof(void*) * (4 + kMaxRanks));
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_rank, lsa_rank, sizeof(int) * world, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    k_lsa_pointers<<<1, 1, 0, st>>>(win[0], win[1], win[2], up, dn, d_rank, world, d_out);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(host_out, d_out, sizeof(void*) * (4 + world), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (d_rank) cudaFree(d_rank);
  if (d_out) cudaFree(d_out);
  return e;
}

// Release every resource of a Device (streams, events, buffers); safe on a partial setup.
void teardown_device(Device& d) {
  if (d.dev < 0) return;
  cudaSetDevice(d.dev);
  for (int b = 0; b < 2; ++b) {
    if (d.staging[b]) cudaFree(d.staging[b]);
    d.staging[b] = nullptr;
  }
  if (d.red) cudaFree(d.red);
  if (d.meas) cudaFree(d.meas);
  d.red = nullptr;
  d.meas = nullptr;
  for (cudaEvent_t e : {d.ev_phase, d.ev_bnd, d.ev_comm, d.ev_t0, d.ev_t1, d.ev_copy[0],
                        d.ev_copy[1], d.ev_stage[0], d.ev_stage[1]})
    if (e) cudaEventDestroy(e);
  for (cudaStream_t s : {d.stream, d.comm, d.copy})
    if (s) cudaStreamDestroy(s);
  d.dev = -1;
}

// Two staging buffers of max(64 MiB, one lattice row) bytes: a chunk always holds at least
// one full row (the pack / unpack kernels work on whole rows).
int ensure_staging(Device& d, int64_t row_bytes) {
  const size_t want = std::max<size_t>(kStagingBytes, (size_t)row_bytes);
  if (d.staging[0] && d.staging_bytes >= want) return ISING_OK;
  CU(cudaSetDevice(d.dev));
  for (int b = 0; b < 2; ++b) {
    if (d.staging[b]) {
      CU(cudaStreamSynchronize(d.stream));
      CU(cudaStreamSynchronize(d.copy));
      CU(cudaFree(d.staging[b]));
      d.staging[b] = nullptr;
    }
  }
  d.staging_bytes = 0;
  for (int b = 0; b < 2; ++b) CU(cudaMalloc(&d.staging[b], want));
  d.staging_bytes = want;
  return ISING_OK;
}

int64_t staging_rows(const Device& d, int64_t row_bytes) {
  return std::max<int64_t>(1, (int64_t)(d.staging_bytes / (size_t)row_bytes));
}

// Host -> device in chunks: copy(k, buf, copy_stream) fills staging buffer k & 1 on the copy
// stream while kern(k, buf, stream) consumes the previous chunk on the compute stream.
template <typename C, typename K>
int pipeline_in(Device& d, int64_t nchunks, C&& copy, K&& kern) {
  for (int64_t k = 0; k < nchunks; ++k) {
    const int b = (int)(k & 1);
    CU(cudaStreamWaitEvent(d.copy, d.ev_stage[b], 0));  // the kernel that last read b is done
    TRY(copy(k, d.staging[b], d.copy));
    CU(cudaEventRecord(d.ev_copy[b], d.copy));
    CU(cudaStreamWaitEvent(d.stream, d.ev_copy[b], 0));
    TRY(kern(k, d.staging[b], d.stream));
    CU(cudaEventRecord(d.ev_stage[b], d.stream));
  }
  return ISING_OK;
}

// Device -> host in chunks: kern(k, buf, stream) fills staging buffer k & 1 on the compute
// stream while copy(k, buf, copy_stream) drains the previous chunk; the compute stream then
// waits for the last copies (so later calls on it see the host buffer complete).
template <typename K, typename C>
int pipeline_out(Device& d, int64_t nchunks, K&& kern, C&& copy) {
  for (int64_t k = 0; k < nchunks; ++k) {
    const int b = (int)(k & 1);
    CU(cudaStreamWaitEvent(d.stream, d.ev_copy[b], 0));  // the copy that last read b is done
    TRY(kern(k, d.staging[b], d.stream));
    CU(cudaEventRecord(d.ev_stage[b], d.stream));
    CU(cudaStreamWaitEvent(d.copy, d.ev_stage[b], 0));
    TRY(copy(k, d.staging[b], d.copy));
    CU(cudaEventRecord(d.ev_copy[b], d.copy));
  }
  for (int b = 0; b < 2; ++b) CU(cudaStreamWaitEvent(d.stream, d.ev_copy[b], 0));
  return ISING_OK;
}

int p2p_wait(ising_ctx* h);

// rank-p2p handle whose half-sweeps run the flag protocol (neighbours, or itself)
bool p2p_flags(const ising_ctx* h) { return h->p2p && (h->world > 1 || h->self_exchange); }
// rank handle whose halos move by NCCL send / recv (neighbours, or itself)
bool nccl_halos(const ising_ctx* h) {
  return h->rank_mode && !h->p2p && (h->comm != nullptr || h->comm_aborted);
}

void trace_dump(ising_ctx* h);

void destroy_ctx(ising_ctx* h) {
  if (!h) return;
  trace_dump(h);
  if (p2p_flags(h) && h->connected && !h->devs.empty()) {
    // the neighbours may still be storing into this slab's halo rows (their last phase):
    // wait for them before the memory goes away (best effort: errors are ignored here)
    cudaSetDevice(h->devs[0].dev);
    if (p2p_wait(h) == ISING_OK) cudaStreamSynchronize(h->devs[0].stream);
    cudaGetLastError();
  }
  if (h->lsa) {  // symmetric memory: deregister (collective) and free through NCCL
    if (!h->devs.empty()) cudaSetDevice(h->devs[0].dev);
    for (auto& w : h->win)
      if (w && h->comm && !h->comm_aborted) ncclCommWindowDeregister(h->comm, w);
    for (auto& s : h->slabs)
      for (int c = 0; c < 2; ++c)
        if (s.plane[c]) ncclMemFree(s.plane[c]);
    if (h->sync) ncclMemFree(h->sync);
    for (auto& s : h->slabs) s.plane[0] = s.plane[1] = nullptr;
    h->sync = nullptr;
  }
  for (auto& s : h->slabs) {
    if (s.devi < (int)h->devs.size()) cudaSetDevice(h->devs[s.devi].dev);
    for (int c = 0; c < 2; ++c)
      if (s.plane[c]) cudaFree(s.plane[c]);
  }
  if (h->comm && !h->comm_aborted) ncclCommDestroy(h->comm);
  for (void* ptr : h->opened) cudaIpcCloseMemHandle(ptr);
  if (h->sync) cudaFree(h->sync);
  if (h->done_counter) cudaFree(h->done_counter);
  for (auto& d : h->devs) teardown_device(d);
  for (cudaEvent_t e : h->prof_events) cudaEventDestroy(e);
  for (auto& pm : h->pending) {
    for (cudaEvent_t e : {pm.t0, pm.t1, pm.done})
      if (e) cudaEventDestroy(e);
    if (pm.host) cudaFreeHost(pm.host);
  }
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  for (int c = 0; c < 2; ++c)
    if (h->bplane[c]) cudaFree(h->bplane[c]);
  if (h->t_dev) cudaFree(h->t_dev);
  if (h->gexec_meas) cudaGraphExecDestroy(h->gexec_meas);
  if (h->bar) cudaFree(h->bar);
  delete h;
}

// Launch geometry for rows [ra, rb) of a slab: H rows per work item, one item per
// thread, blocks of 128; H chosen so the grid is >= ~4 waves of resident blocks.
void halfsweep_geometry(const ising_ctx* h, const Device& d, int64_t rows, int* H,
                        int64_t* items, int* grid) {
  const int64_t chunks = h->W / kWordsPerItem;
  int hh = h->rows_per_item_override;
  if (hh <= 0) {
    const int64_t resident = (int64_t)d.sms * d.hs_blocks_per_sm * 128;
    int64_t want = (chunks * rows) / (resident * 4);
    hh = 1;
    while (hh * 2 <= want && hh < 32) hh *= 2;
  }
  *H = hh;
  *items = chunks * ((rows + hh - 1) / hh);
  *grid = (int)std::min<int64_t>((*items + 127) / 128, int64_t(1) << 30);
}

// kernel variant: 0 = Metropolis with both thresholds < 2^32 (the fast path),
// 2 = Metropolis generic (tiny beta), 4 = Metropolis draw-free (T3, T4 in {0, 2^32});
// heat bath 3 / 5 / 6 = fast path with 0 / 1 / 2 "always" classes (T = 2^32), 1 = generic,
// 7 = symmetric thresholds (T[0] + T[4] = T[1] + T[3] = 2^32 + 1, T[2] = 2^31)
int kernel_variant(const ising_ctx* h) {
  if (h->rule == ISING_RULE_METROPOLIS) {
    const bool t3_fixed = h->T[3] == 0 || h->T[3] == (uint64_t(1) << 32);
    const bool t4_fixed = h->T[4] == 0 || h->T[4] == (uint64_t(1) << 32);
    if (t3_fixed && t4_fixed && h->draw_free_enabled) return 4;  // no draw needed
    return (h->acc.keep3 & h->acc.keep4) ? 0 : 2;
  }
  // symmetric thresholds (P(e) + P(-e) = 1 survived the rounding): the 2-compare kernel
  const uint64_t two32p1 = (uint64_t(1) << 32) + 1;
  if (h->symmetric_hb_enabled && h->T[2] == (uint64_t(1) << 31) && h->T[0] + h->T[4] == two32p1 &&
      h->T[1] + h->T[3] == two32p1)
    return 7;
  switch (h->acc.always_mask) {  // the "always" classes form a prefix of the non-increasing T
    case 0: return 3;
    case 1: return 5;
    case 3: return 6;
    default: return 1;  // not reachable from compute_thresholds; kept exact anyway
  }
}

int run_halfsweep(ising_ctx* h, Slab& s, int c, int r_begin, int r_end, uint64_t* halo_up,
                     uint64_t* halo_dn, uint32_t t, bool t_from_dev = false,
                     unsigned long long* obs = nullptr, bool slot_from_dev = false) {
  if (r_end <= r_begin) return ISING_OK;
  Device& d = h->devs[s.devi];
  HalfSweepParams p{};
  p.tgt = s.plane[c];
  p.src = s.plane[1 - c];
  p.halo_up = halo_up;
  p.halo_dn = halo_dn;
  p.W = h->W;
  p.row0 = s.row0;
  p.R = (int32_t)s.R;
  p.r_begin = r_begin;
  p.r_end = r_end;
  int grid;
  halfsweep_geometry(h, d, r_end - r_begin, &p.H, &p.items, &grid);
  p.t = t;
  p.t_dev = t_from_dev ? h->t_dev : nullptr;
  // measured sweeps: the white phase adds into obs, the black phase before it zeroes it
  // (graph replays index a device-resident slot and keep the memset of all slots instead)
  p.obs_out = c == 1 ? obs : nullptr;
  p.obs_clear = (c == 0 && obs && !slot_from_dev) ? obs : nullptr;
  p.slot_dev = (c == 1 && obs && slot_from_dev) ? h->t_dev + 1 : nullptr;
  p.colour = (uint32_t)c;
  p.keys = h->keys;
  p.acc = h->acc;
  if (p2p_flags(h)) {
    // wait for both neighbours to finish the previous phase; publish this one
    const int up = (h->rank + h->world - 1) % h->world, dn = (h->rank + 1) % h->world;
    p.wait_flags = h->sync;
    p.wait_value = h->phase;
    p.signal_up = h->peer_sync[up] + 1;  // I am my upper neighbour's lower neighbour
    p.signal_dn = h->peer_sync[dn] + 0;
    p.signal_value = h->phase + 1;
    p.done_counter = h->done_counter;
  }
  const bool prof = h->prof_active && s.devi == 0 &&
                    (size_t)(2 * h->kernel_launches + 1) < h->prof_events.size();
  if (prof) CU(cudaEventRecord(h->prof_events[2 * h->kernel_launches], d.stream));
  p.pdl = h->pdl ? 1 : 0;
  // Alternate the band order between phases, so each phase's first wave reads the rows the
  // previous phase wrote last (still in L2).  (Rank-p2p: the edge bands stay first in the grid;
  // mirroring swaps which rows the first and last logical band hold, both still edge rows.)
  p.mirror = (h->mirror && c == 1) ? 1 : 0;
  if (h->staged && h->W % kStageWords == 0) {
    CU(launch_halfsweep_staged(kernel_variant(h),
                               h->guided_tail ? (int64_t)d.sms * d.staged_blocks_per_sm : 0, d.stream, p));
  } else {
    CU(launch_halfsweep(kernel_variant(h), grid, d.stream, p));
  }
  if (prof) {
    CU(cudaEventRecord(h->prof_events[2 * h->kernel_launches + 1], d.stream));
    ++h->kernel_launches;
  }
  ++h->launch_count;
  return ISING_OK;
}

// NCCL reports failures of a peer / the network asynchronously: poll the communicator's
// error state (SURVEY §5 failure detection).  On an error the communicator is aborted, so a
// stream blocked in an NCCL kernel does not hang the process.
int nccl_poll(ising_ctx* h) {
  if (h->comm_aborted) {
    g_last_error = "NCCL communicator aborted after an asynchronous error";
    return ISING_ERR_NCCL;
  }
  if (!h->comm) return ISING_OK;
  ncclResult_t ae = ncclSuccess;
  NC(ncclCommGetAsyncError(h->comm, &ae));
  if (ae != ncclSuccess && ae != ncclInProgress) {
    const int st = fail_nccl(ae, "NCCL asynchronous error (communicator aborted)", __LINE__);
    ncclCommAbort(h->comm);  // frees the communicator; the handle is unusable from here on
    h->comm = nullptr;
    h->comm_aborted = true;
    return st;
  }
  return ISING_OK;
}

// A stream that makes no progress for this long in NCCL rank mode is a hung peer that reported
// no error (ISING_NCCL_TIMEOUT_S, default 300 s): the communicator is aborted and the call
// fails with ISING_ERR_NCCL instead of blocking the process forever.
double nccl_timeout_s() {
  const char* v = getenv("ISING_NCCL_TIMEOUT_S");
  const double t = v ? atof(v) : 300.0;
  return t > 0 ? t : 300.0;
}

// Wait for a stream; in NCCL rank mode by polling, checking the communicator meanwhile.
int wait_stream(ising_ctx* h, cudaStream_t st) {
  if (!h->comm) {
    CU(cudaStreamSynchronize(st));
    return h->comm_aborted ? nccl_poll(h) : ISING_OK;
  }
  const auto t0 = std::chrono::steady_clock::now();
  const double limit = nccl_timeout_s();
  for (;;) {
    const cudaError_t e = cudaStreamQuery(st);
    if (e == cudaSuccess) return nccl_poll(h);
    if (e != cudaErrorNotReady) return fail_cuda(e, "cudaStreamQuery", __LINE__);
    TRY(nccl_poll(h));
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit) {
      ncclCommAbort(h->comm);
      h->comm = nullptr;
      h->comm_aborted = true;
      g_last_error = "NCCL rank mode: no progress within ISING_NCCL_TIMEOUT_S (communicator aborted)";
      return ISING_ERR_NCCL;
    }
    nvtx_yield();
  }
}

int sync_all(ising_ctx* h) {
  for (auto& d : h->devs) {
    CU(cudaSetDevice(d.dev));
    TRY(wait_stream(h, d.stream));
    TRY(wait_stream(h, d.comm));
    TRY(wait_stream(h, d.copy));
  }
  return ISING_OK;
}

// Profiling: one event pair per timed half-sweep launch of ising_sweep (at most
// kMaxProfiledLaunches).  Only ising_sweep times launches (h->prof_active, set after this
// sizing); the launch paths also check the pool size, so no path can index past it.
int ensure_prof_events(ising_ctx* h, int64_t n_sweeps) {
  if (!h->profiling) return ISING_OK;
  const size_t per_phase = std::max<size_t>(3, h->slabs.size());
  const size_t want = (size_t)std::min<int64_t>(std::max<int64_t>(n_sweeps, 1), kMaxProfiledLaunches);
  const size_t need = std::min<size_t>(want * 2 * 2 * per_phase, 2 * kMaxProfiledLaunches);
  if (!h->devs.empty()) CU(cudaSetDevice(h->devs[0].dev));
  while (h->prof_events.size() < need) {
    cudaEvent_t e;
    CU(cudaEventCreate(&e));
    h->prof_events.push_back(e);
  }
  return ISING_OK;
}

// Record a timing event of the trace (no-op unless ISING_TRACE is set).
int trace_mark(ising_ctx* h, const char* name, cudaStream_t st, const char* stream_name) {
  if (h->trace_path.empty() || h->traced_phases >= kMaxTracedPhases) return ISING_OK;
  cudaEvent_t e;
  CU(cudaEventCreate(&e));
  h->trace.push_back({h->traced_phases, name, stream_name, e});
  CU(cudaEventRecord(e, st));
  return ISING_OK;
}

void trace_dump(ising_ctx* h) {
  if (h->trace.empty()) return;
  for (auto& t : h->trace) cudaEventSynchronize(t.ev);  // this handle's events only
  FILE* f = fopen(h->trace_path.c_str(), "w");
  if (f) {
    fprintf(f, "phase,name,stream,ms\n");
    for (auto& t : h->trace) {
      float ms = 0;
      cudaEventElapsedTime(&ms, h->trace[0].ev, t.ev);
      fprintf(f, "%lld,%s,%s,%.6f\n", (long long)t.phase, t.name, t.stream, ms);
    }
    fclose(f);
  }
  for (auto& t : h->trace) cudaEventDestroy(t.ev);
  h->trace.clear();
}

// One colour phase, LOCAL mode.
int phase_local(ising_ctx* h, int c, uint32_t t, bool t_from_dev = false,
                const std::vector<unsigned long long*>* obs = nullptr, bool slot_from_dev = false) {
  NvtxRange range("half-sweep c=%lld t=%lld", c, t);
  const int n = (int)h->slabs.size();
  const bool multi_dev = h->devs.size() > 1;
  if (multi_dev) {
    // phase p on device d waits for phase p-1 on the devices of its slabs' neighbours
    for (int di = 0; di < (int)h->devs.size(); ++di) {
      std::vector<int> waits;
      for (int k = 0; k < n; ++k) {
        if (h->slabs[k].devi != di) continue;
        for (int nb : {(k + n - 1) % n, (k + 1) % n}) {
          const int nd = h->slabs[nb].devi;
          if (nd != di && std::find(waits.begin(), waits.end(), nd) == waits.end()) waits.push_back(nd);
        }
      }
      CU(cudaSetDevice(h->devs[di].dev));
      for (int nd : waits) CU(cudaStreamWaitEvent(h->devs[di].stream, h->devs[nd].ev_phase, 0));
    }
  }
  for (int k = 0; k < n; ++k) {
    Slab& s = h->slabs[k];
    Slab& up = h->slabs[(k + n - 1) % n];
    Slab& dn = h->slabs[(k + 1) % n];
    CU(cudaSetDevice(h->devs[s.devi].dev));
    // local row 0 -> upper slab's bottom halo (padded row R+1); local row R-1 -> lower
    // slab's top halo (padded row 0).
    TRY(run_halfsweep(h, s, c, 0, (int)s.R, up.plane[c] + (up.R + 1) * h->W, dn.plane[c], t,
                      t_from_dev, obs ? (*obs)[s.devi] : nullptr, slot_from_dev));
  }
  if (multi_dev) {
    for (auto& d : h->devs) {
      CU(cudaSetDevice(d.dev));
      CU(cudaEventRecord(d.ev_phase, d.stream));
    }
  }
  return ISING_OK;
}

// One colour phase, RANK mode (world >= 2): boundary rows, then NCCL halo exchange
// overlapped with the interior rows.
int phase_rank(ising_ctx* h, int c, uint32_t t) {
  NvtxRange range("half-sweep nccl c=%lld t=%lld", c, t);
  Slab& s = h->slabs[0];
  Device& d = h->devs[0];
  const int R = (int)s.R;
  const size_t W = (size_t)h->W;
  TRY(trace_mark(h, "boundary_start", d.stream, "compute"));
  TRY(run_halfsweep(h, s, c, 0, 1, nullptr, nullptr, t));
  if (R > 1) TRY(run_halfsweep(h, s, c, R - 1, R, nullptr, nullptr, t));
  TRY(trace_mark(h, "boundary_end", d.stream, "compute"));
  CU(cudaEventRecord(d.ev_bnd, d.stream));
  CU(cudaStreamWaitEvent(d.comm, d.ev_bnd, 0));
  TRY(trace_mark(h, "halo_start", d.comm, "comm"));
  const int up = (h->rank + h->world - 1) % h->world, dn = (h->rank + 1) % h->world;
  uint64_t* pl = s.plane[c];
  NC(ncclGroupStart());
  NC(ncclSend(pl + 1 * W, W, ncclUint64, up, h->comm, d.comm));        // row 0 -> up's bottom halo
  NC(ncclRecv(pl + (size_t)(R + 1) * W, W, ncclUint64, dn, h->comm, d.comm));
  NC(ncclSend(pl + (size_t)R * W, W, ncclUint64, dn, h->comm, d.comm)); // row R-1 -> dn's top halo
  NC(ncclRecv(pl, W, ncclUint64, up, h->comm, d.comm));
  NC(ncclGroupEnd());
  TRY(trace_mark(h, "halo_end", d.comm, "comm"));
  CU(cudaEventRecord(d.ev_comm, d.comm));
  TRY(trace_mark(h, "interior_start", d.stream, "compute"));
  TRY(run_halfsweep(h, s, c, 1, R - 1, nullptr, nullptr, t));
  TRY(trace_mark(h, "interior_end", d.stream, "compute"));
  CU(cudaStreamWaitEvent(d.stream, d.ev_comm, 0));
  if (!h->trace_path.empty()) ++h->traced_phases;
  return ISING_OK;
}

// One colour phase, RANK-P2P mode (world >= 2): the half-sweep kernel waits for the
// neighbours' previous phase, stores its boundary rows straight into their halo rows
// over NVLink, and its last block raises their flags — compute and exchange in one kernel.
int phase_p2p(ising_ctx* h, int c, uint32_t t, unsigned long long* obs = nullptr) {
  NvtxRange range("half-sweep p2p c=%lld t=%lld", c, t);
  Slab& s = h->slabs[0];
  TRY(trace_mark(h, "phase_start", h->devs[0].stream, "compute"));
  TRY(run_halfsweep(h, s, c, 0, (int)s.R, h->up_plane[c] + (s.R + 1) * h->W, h->dn_plane[c], t,
                    false, obs));
  TRY(trace_mark(h, "phase_end", h->devs[0].stream, "compute"));
  if (!h->trace_path.empty()) ++h->traced_phases;
  ++h->phase;
  return ISING_OK;
}

// Rank mode after loading only this rank's rows: move both planes' boundary rows into the
// neighbours' halo rows (peer stores for p2p, ncclSend/Recv for NCCL).
int exchange_halos(ising_ctx* h) {
  Slab& s = h->slabs[0];
  Device& d = h->devs[0];
  const size_t W = (size_t)h->W;
  const int R = (int)s.R;
  if (h->p2p) {  // peer stores by a kernel (see launch_copy_u64)
    for (int c = 0; c < 2; ++c) {
      CU(launch_copy_u64(d.stream, h->up_plane[c] + (size_t)(R + 1) * W, s.plane[c] + W, (int64_t)W));
      CU(launch_copy_u64(d.stream, h->dn_plane[c], s.plane[c] + (size_t)R * W, (int64_t)W));
      h->launch_count += 2;
    }
    return ISING_OK;
  }
  const int up = (h->rank + h->world - 1) % h->world, dn = (h->rank + 1) % h->world;
  for (int c = 0; c < 2; ++c) {
    uint64_t* pl = s.plane[c];
    NC(ncclGroupStart());
    NC(ncclSend(pl + W, W, ncclUint64, up, h->comm, d.stream));
    NC(ncclRecv(pl + (size_t)(R + 1) * W, W, ncclUint64, dn, h->comm, d.stream));
    NC(ncclSend(pl + (size_t)R * W, W, ncclUint64, dn, h->comm, d.stream));
    NC(ncclRecv(pl, W, ncclUint64, up, h->comm, d.stream));
    NC(ncclGroupEnd());
  }
  return ISING_OK;
}

// RANK-P2P: wait until both neighbours have finished every phase issued so far (before
// this rank overwrites its halo rows or reads them).
int p2p_wait(ising_ctx* h) {
  if (!p2p_flags(h)) return ISING_OK;
  SyncParams p{};
  p.wait_flags = h->sync;
  p.wait_count = 2;
  p.wait_value = h->phase;
  CU(launch_sync(h->devs[0].stream, p));
  ++h->launch_count;
  return ISING_OK;
}

// RANK-P2P: a state reset (init / write) counts as a phase: publish it to the neighbours.
int p2p_publish(ising_ctx* h) {
  if (!p2p_flags(h)) return ISING_OK;
  const int up = (h->rank + h->world - 1) % h->world, dn = (h->rank + 1) % h->world;
  SyncParams p{};
  p.signal[0] = h->peer_sync[up] + 1;
  p.signal[1] = h->peer_sync[dn] + 0;
  p.signal_value = ++h->phase;
  CU(launch_sync(h->devs[0].stream, p));
  ++h->launch_count;
  return ISING_OK;
}

// Small lattices are launch-bound (a C2 half-sweep is ~1.5 us of GPU work): sweeps are
// replayed from a CUDA graph of kGraphSweeps sweeps whose kernels read the sweep base from
// device memory (h->t_dev) and whose last node advances it.  Single-device LOCAL mode only.
constexpr int kGraphSweeps = 64;
constexpr int64_t kGraphMaxSpins = int64_t(1) << 26;

bool graph_eligible(const ising_ctx* h) {
  return h->graphs_enabled && !h->rank_mode && h->devs.size() == 1 && !h->profiling &&
         h->N * h->M <= kGraphMaxSpins;
}

int build_graph(ising_ctx* h) {
  Device& d = h->devs[0];
  CU(cudaSetDevice(d.dev));
  if (!h->t_dev) CU(cudaMalloc(&h->t_dev, 2 * sizeof(uint32_t)));  // [sweep base, sample base]
  if (h->gexec) {
    CU(cudaGraphExecDestroy(h->gexec));
    h->gexec = nullptr;
  }
  const int64_t before = h->launch_count;
  cudaGraph_t g = nullptr;
  CU(cudaStreamBeginCapture(d.stream, cudaStreamCaptureModeThreadLocal));
  int st = ISING_OK;
  for (int k = 1; k <= kGraphSweeps && st == ISING_OK; ++k)
    for (int c = 0; c < 2 && st == ISING_OK; ++c) st = phase_local(h, c, (uint32_t)k, true);
  cudaError_t e = launch_set_u32(d.stream, h->t_dev, kGraphSweeps, 1);
  cudaError_t e2 = cudaStreamEndCapture(d.stream, &g);
  if (st != ISING_OK) return st;
  CU(e);
  CU(e2);
  e = cudaGraphInstantiate(&h->gexec, g, 0);
  cudaGraphDestroy(g);
  CU(e);
  h->graph_launches = h->launch_count - before + 1;
  h->launch_count = before;
  return ISING_OK;
}

// Measured-chain graph: S = max(1, kGraphSweeps / every) samples of `every` sweeps each,
// the white phase of each sample's last sweep reducing its observables into slot
// (sample base + k) of `base`; the last nodes advance the sweep and sample bases.
int build_measure_graph(ising_ctx* h, int64_t every, unsigned long long* base) {
  Device& d = h->devs[0];
  CU(cudaSetDevice(d.dev));
  if (!h->t_dev) CU(cudaMalloc(&h->t_dev, 2 * sizeof(uint32_t)));
  if (h->gexec_meas) {
    CU(cudaGraphExecDestroy(h->gexec_meas));
    h->gexec_meas = nullptr;
  }
  const int64_t S = std::max<int64_t>(1, kGraphSweeps / every);
  const int64_t before = h->launch_count;
  cudaGraph_t g = nullptr;
  CU(cudaStreamBeginCapture(d.stream, cudaStreamCaptureModeThreadLocal));
  int st = ISING_OK;
  for (int64_t k = 0; k < S && st == ISING_OK; ++k) {
    std::vector<unsigned long long*> slot(1, base + 2 * k);
    for (int64_t sw = 1; sw <= every && st == ISING_OK; ++sw)
      for (int c = 0; c < 2 && st == ISING_OK; ++c)
        st = phase_local(h, c, (uint32_t)(k * every + sw), true, sw == every ? &slot : nullptr, true);
  }
  cudaError_t e = launch_set_u32(d.stream, h->t_dev, (uint32_t)(S * every), 1);
  cudaError_t e1 = launch_set_u32(d.stream, h->t_dev + 1, (uint32_t)S, 1);
  cudaError_t e2 = cudaStreamEndCapture(d.stream, &g);
  if (st != ISING_OK) return st;
  CU(e);
  CU(e1);
  CU(e2);
  e = cudaGraphInstantiate(&h->gexec_meas, g, 0);
  cudaGraphDestroy(g);
  CU(e);
  h->meas_graph_launches = h->launch_count - before + 2;
  h->launch_count = before;
  h->meas_every = every;
  h->meas_base = base;
  h->meas_samples = S;
  return ISING_OK;
}

int enable_peers(ising_ctx* h) {
  const int n = (int)h->slabs.size();
  for (int k = 0; k < n; ++k) {
    const int a = h->devs[h->slabs[k].devi].dev;
    for (int nb : {(k + n - 1) % n, (k + 1) % n}) {
      const int b = h->devs[h->slabs[nb].devi].dev;
      if (a == b) continue;
      int can = 0;
      CU(cudaDeviceCanAccessPeer(&can, a, b));
      if (!can) {
        g_last_error = "no P2P access between neighbouring slab devices";
        return ISING_ERR_DEVICE;
      }
      CU(cudaSetDevice(a));
      cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else if (e != cudaSuccess) {
        return fail_cuda(e, "cudaDeviceEnablePeerAccess", __LINE__);
      }
    }
  }
  return ISING_OK;
}

// Experiment / test knobs read once at creation (every handle type).
void read_env_knobs(ising_ctx* h) {
  if (const char* tr = getenv("ISING_TRACE")) h->trace_path = tr;
  const char* env = getenv("ISING_ROWS_PER_ITEM");
  if (env) h->rows_per_item_override = atoi(env);
  if (env_is_zero("ISING_GRAPHS")) h->graphs_enabled = false;
  if (env_is_zero("ISING_DRAW_FREE")) h->draw_free_enabled = false;
  if (env_is_zero("ISING_STAGED")) h->staged = false;
  if (env_is_one("ISING_PERSISTENT")) h->persistent_enabled = true;
}

int create_local(ising_t* out, int64_t N, int64_t M, uint64_t seed, int n_slabs, const int* devices) {
  if (!out) return ISING_ERR_ARG;
  *out = nullptr;
  TRY(check_shape(N, M, n_slabs));
  ising_ctx* h = new (std::nothrow) ising_ctx;
  if (!h) return ISING_ERR_OOM;
  h->N = N;
  h->M = M;
  h->W = M / 32;
  h->seed = seed;
  make_keys(seed, &h->keys);
  const int64_t R = N / n_slabs;
  for (int k = 0; k < n_slabs; ++k) {
    int di = -1;
    for (int j = 0; j < (int)h->devs.size(); ++j)
      if (h->devs[j].dev == devices[k]) di = j;
    if (di < 0) {
      h->devs.emplace_back();
      int st = setup_device(h->devs.back(), devices[k]);
      if (st != ISING_OK) {
        destroy_ctx(h);
        return st;
      }
      di = (int)h->devs.size() - 1;
    }
    Slab s;
    s.devi = di;
    s.row0 = k * R;
    s.R = R;
    h->slabs.push_back(s);
  }
  int st = enable_peers(h);
  if (st == ISING_OK) st = alloc_slabs(h);
  if (st != ISING_OK) {
    destroy_ctx(h);
    return st;
  }
  read_env_knobs(h);
  *out = h;
  return ISING_OK;
}

int run_init(ising_ctx* h, int cold) {
  if (h->p2p && h->world > 1 && !h->connected) {
    g_last_error = "rank-p2p handle used before ising_ipc_connect";
    return ISING_ERR_STATE;
  }
  TRY(p2p_wait(h));
  for (auto& s : h->slabs) {
    Device& d = h->devs[s.devi];
    CU(cudaSetDevice(d.dev));
    InitParams p;
    p.plane[0] = s.plane[0];
    p.plane[1] = s.plane[1];
    p.W = h->W;
    p.row0 = s.row0;
    p.N = h->N;
    p.R = (int32_t)s.R;
    p.cold = cold;
    p.keys = h->keys;
    const int64_t total = 2 * (s.R + 2) * h->W;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)d.sms * 64);
    k_init<<<grid, 256, 0, d.stream>>>(p);
    CU(cudaGetLastError());
    ++h->launch_count;
  }
  TRY(p2p_publish(h));
  TRY(sync_all(h));
  h->t = 0;
  h->state_set = true;
  return ISING_OK;
}

// Copy global rows [g, g + n) (wrapping mod N) of the host lattice to dst.
int h2d_rows(ising_ctx* h, int8_t* dst, const int8_t* in, int64_t g, int64_t n, cudaStream_t st,
             int64_t row_bytes) {
  g %= h->N;
  if (g < 0) g += h->N;
  while (n > 0) {
    const int64_t run = std::min(n, h->N - g);
    CU(cudaMemcpyAsync(dst, in + g * row_bytes, (size_t)(run * row_bytes), cudaMemcpyHostToDevice, st));
    dst += run * row_bytes;
    n -= run;
    g = 0;
  }
  return ISING_OK;
}

// Persistent multi-sweep launch (small single-slab lattices): sweeps t+1 .. t+n in one
// cooperative kernel; with obs_base, slot k receives the observables after sweep
// t + (k+1) * every.
constexpr int64_t kPersistMaxSpins = int64_t(1) << 24;

bool persistent_eligible(const ising_ctx* h) {
  return h->persistent_enabled && !h->rank_mode && !h->basic && h->devs.size() == 1 &&
         h->slabs.size() == 1 && !h->profiling && h->N * h->M <= kPersistMaxSpins;
}

int run_persistent(ising_ctx* h, int64_t n, unsigned long long* obs_base, int64_t every) {
  Device& d = h->devs[0];
  Slab& s = h->slabs[0];
  CU(cudaSetDevice(d.dev));
  if (!h->bar) {
    CU(cudaMalloc(&h->bar, 2 * sizeof(unsigned int)));
    CU(cudaMemsetAsync(h->bar, 0, 2 * sizeof(unsigned int), d.stream));
  }
  if (h->persist_blocks_per_sm <= 0) {
    CU(persistent_occupancy(&h->persist_blocks_per_sm));
    if (h->persist_blocks_per_sm < 1) h->persist_blocks_per_sm = 1;
  }
  const int grid = d.sms * h->persist_blocks_per_sm;
  PersistentParams P{};
  for (int c = 0; c < 2; ++c) {
    HalfSweepParams& p = P.ph[c];
    p.tgt = s.plane[c];
    p.src = s.plane[1 - c];
    p.halo_up = s.plane[c] + (s.R + 1) * h->W;  // one slab: its own halo rows
    p.halo_dn = s.plane[c];
    p.W = h->W;
    p.row0 = s.row0;
    p.R = (int32_t)s.R;
    p.r_begin = 0;
    p.r_end = (int32_t)s.R;
    // H = 1 unless the grid has more threads than chunk-rows
    const int64_t chunks = h->W / kWordsPerItem;
    int hh = 1;
    while (hh < 32 && chunks * ((s.R + 2 * hh - 1) / (2 * hh)) >= (int64_t)grid * 512) hh *= 2;
    p.H = hh;
    p.items = chunks * ((s.R + hh - 1) / hh);
    p.colour = (uint32_t)c;
    p.keys = h->keys;
    p.acc = h->acc;
  }
  P.t0 = (uint32_t)h->t;
  P.n = (uint32_t)n;
  P.bar_count = h->bar;
  P.bar_gen = h->bar + 1;
  P.obs_base = obs_base;
  P.every = (uint32_t)std::max<int64_t>(every, 1);
  CU(launch_persistent(kernel_variant(h), grid, d.stream, P));
  ++h->launch_count;
  h->t += (uint64_t)n;
  return ISING_OK;
}

// Enqueue sweeps t+1 .. t+n on the handle's streams (no synchronisation); t += n.  With
// obs (LOCAL mode), the white phase of sweep t+n also reduces the observables of the state
// it produces into obs[device][0..1] (fused; no extra pass).
int enqueue_sweeps(ising_ctx* h, int64_t n, const std::vector<unsigned long long*>* obs = nullptr) {
  if (n > 0 && persistent_eligible(h)) return run_persistent(h, n, obs ? (*obs)[0] : nullptr, n);
  int64_t k0 = 1;
  const int64_t n_graph = obs ? n - 1 : n;  // the measured sweep is launched directly
  if (graph_eligible(h) && n_graph >= kGraphSweeps) {
    if (!h->gexec) TRY(build_graph(h));
    Device& d = h->devs[0];
    CU(launch_set_u32(d.stream, h->t_dev, (uint32_t)h->t, 0));
    ++h->launch_count;
    const int64_t reps = n_graph / kGraphSweeps;
    for (int64_t r = 0; r < reps; ++r) {
      CU(cudaGraphLaunch(h->gexec, d.stream));
      h->launch_count += h->graph_launches;
    }
    k0 = reps * kGraphSweeps + 1;
  }
  for (int64_t k = k0; k <= n; ++k) {
    const uint32_t t = (uint32_t)(h->t + (uint64_t)k);
    for (int c = 0; c < 2; ++c) {
      if (p2p_flags(h))
        TRY(phase_p2p(h, c, t, (k == n && obs) ? (*obs)[0] : nullptr));
      else if (nccl_halos(h))
        TRY(phase_rank(h, c, t));
      else
        TRY(phase_local(h, c, t, false, k == n ? obs : nullptr));
    }
  }
  h->t += (uint64_t)n;
  return ISING_OK;
}

// Enqueue the observables reduction of every slab; slab partials of device d are added
// (atomics) into out[d][0..1] (zeroed by the caller).
int enqueue_observables(ising_ctx* h, const std::vector<unsigned long long*>& out) {
  for (auto& s : h->slabs) {
    Device& d = h->devs[s.devi];
    CU(cudaSetDevice(d.dev));
    ObsParams p;
    p.black = s.plane[0];
    p.white = s.plane[1];
    p.W = h->W;
    p.row0 = s.row0;
    p.R = (int32_t)s.R;
    p.out = out[s.devi];
    const int64_t total = s.R * h->W;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)d.sms * 8);
    k_observables<<<grid, 256, 0, d.stream>>>(p);
    CU(cudaGetLastError());
    ++h->launch_count;
  }
  return ISING_OK;
}

// Unpack local rows [la, lb) of slab s into host rows at dst (row-major, M bytes each):
// unpack of chunk k + 1 overlaps the D2H copy of chunk k (pipeline_out).
int unpack_rows_to_host(ising_ctx* h, Slab& s, int64_t la, int64_t lb, int8_t* dst,
                        bool bits = false) {
  Device& d = h->devs[s.devi];
  CU(cudaSetDevice(d.dev));
  const int64_t row_bytes = bits ? h->M / 8 : h->M;
  TRY(ensure_staging(d, row_bytes));
  const int64_t rpc = staging_rows(d, row_bytes);
  auto span = [&](int64_t k, int64_t* ra, int64_t* rb) {
    *ra = la + k * rpc;
    *rb = std::min<int64_t>(*ra + rpc, lb);
  };
  auto kern = [&](int64_t k, int8_t* buf, cudaStream_t st) -> int {
    int64_t ra, rb;
    span(k, &ra, &rb);
    if (bits) {
      UnpackBitsParams p;
      p.plane[0] = s.plane[0];
      p.plane[1] = s.plane[1];
      p.bits = reinterpret_cast<uint32_t*>(buf);
      p.W = h->W;
      p.row0 = s.row0;
      p.ra = (int32_t)ra;
      p.rb = (int32_t)rb;
      const int64_t total = (rb - ra) * h->W;
      CU(launch_unpack_bits((int)std::min<int64_t>((total + 255) / 256, (int64_t)d.sms * 64), st, p));
      ++h->launch_count;
      return ISING_OK;
    }
    UnpackParams p;
    p.plane[0] = s.plane[0];
    p.plane[1] = s.plane[1];
    p.full = buf;
    p.W = h->W;
    p.M = h->M;
    p.row0 = s.row0;
    p.ra = (int32_t)ra;
    p.rb = (int32_t)rb;
    const int64_t total = 2 * (rb - ra) * h->W;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)d.sms * 64);
    k_unpack<<<grid, 256, 0, st>>>(p);
    CU(cudaGetLastError());
    ++h->launch_count;
    return ISING_OK;
  };
  auto copy = [&](int64_t k, int8_t* buf, cudaStream_t st) -> int {
    int64_t ra, rb;
    span(k, &ra, &rb);
    CU(cudaMemcpyAsync(dst + (ra - la) * row_bytes, buf, (size_t)((rb - ra) * row_bytes),
                       cudaMemcpyDeviceToHost, st));
    return ISING_OK;
  };
  return pipeline_out(d, (lb - la + rpc - 1) / rpc, kern, copy);
}

// ------------------------------------------------------------- basic layout
int basic_grid(const Device& d, int64_t work) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, (int64_t)d.sms * 32));
}

int basic_init(ising_ctx* h, int cold) {
  Device& d = h->devs[0];
  CU(cudaSetDevice(d.dev));
  const int64_t ny = h->M / 2;
  CU(launch_basic_init(basic_grid(d, 2 * h->N * (ny / 4)), d.stream, h->bplane[0], h->bplane[1],
                       h->N, ny, cold, h->keys));
  ++h->launch_count;
  CU(cudaStreamSynchronize(d.stream));
  h->t = 0;
  h->state_set = true;
  return ISING_OK;
}

bool basic_listing() {
  const char* listing_env = getenv("ISING_BASIC_LISTING");
  return listing_env && listing_env[0] == '1';
}

// The basic layout's measured chains fuse the observables into the SWAR kernel's white phase.
bool basic_fused_obs(const ising_ctx* h) { return !basic_listing() && ((h->M / 2) & 15) == 0; }

// obs: add the observables of the state after the last sweep into obs[0..1] (SWAR kernel).
int basic_enqueue_sweeps(ising_ctx* h, int64_t n, unsigned long long* obs = nullptr) {
  Device& d = h->devs[0];
  const int64_t ny = h->M / 2;
  const int rule = kernel_variant(h);
  const int listing = basic_listing() ? 1 : 0;
  for (int64_t k = 1; k <= n; ++k) {
    for (int c = 0; c < 2; ++c) {
      BasicParams p{};
      p.lattice = h->bplane[c];
      p.op_lattice = h->bplane[1 - c];
      p.nx = h->N;
      p.ny = ny;
      p.t = (uint32_t)(h->t + (uint64_t)k);
      p.colour = (uint32_t)c;
      p.acc = h->acc;
      p.keys = h->keys;
      p.obs_out = (k == n && c == 1) ? obs : nullptr;
      const bool prof = h->prof_active && (size_t)(2 * h->kernel_launches + 1) < h->prof_events.size();
      if (prof) CU(cudaEventRecord(h->prof_events[2 * h->kernel_launches], d.stream));
      CU(launch_basic_halfsweep(rule, listing, d.sms, d.stream, p));
      if (prof) {
        CU(cudaEventRecord(h->prof_events[2 * h->kernel_launches + 1], d.stream));
        ++h->kernel_launches;
      }
      ++h->launch_count;
    }
  }
  h->t += (uint64_t)n;
  return ISING_OK;
}

int basic_convert(ising_ctx* h, int8_t* host, bool to_host) {
  Device& d = h->devs[0];
  CU(cudaSetDevice(d.dev));
  TRY(ensure_staging(d, h->M));
  const int64_t ny = h->M / 2;
  CU(cudaMemsetAsync(d.red, 0, 4 * sizeof(unsigned long long), d.stream));
  const int64_t rpc = staging_rows(d, h->M);
  const int64_t nchunks = (h->N + rpc - 1) / rpc;
  auto rows_of = [&](int64_t k) { return std::min<int64_t>(rpc, h->N - k * rpc); };
  auto kern = [&](int64_t k, int8_t* buf, cudaStream_t st) -> int {
    CU(launch_basic_convert(basic_grid(d, rows_of(k) * h->M), st, h->bplane[0], h->bplane[1], buf,
                            ny, k * rpc, rows_of(k), to_host ? 1 : 0,
                            reinterpret_cast<unsigned int*>(d.red + 2)));
    ++h->launch_count;
    return ISING_OK;
  };
  auto copy = [&](int64_t k, int8_t* buf, cudaStream_t st) -> int {
    const size_t bytes = (size_t)(rows_of(k) * h->M);
    if (to_host)
      CU(cudaMemcpyAsync(host + k * rpc * h->M, buf, bytes, cudaMemcpyDeviceToHost, st));
    else
      CU(cudaMemcpyAsync(buf, host + k * rpc * h->M, bytes, cudaMemcpyHostToDevice, st));
    return ISING_OK;
  };
  if (to_host)
    TRY(pipeline_out(d, nchunks, kern, copy));
  else
    TRY(pipeline_in(d, nchunks, copy, kern));
  CU(cudaStreamSynchronize(d.stream));
  CU(cudaStreamSynchronize(d.copy));
  if (!to_host) {
    unsigned long long bad = 0;
    CU(cudaMemcpy(&bad, d.red + 2, sizeof bad, cudaMemcpyDeviceToHost));
    if (bad & 0xffffffffull) {
      g_last_error = "ising_write_lattice: values must be -1 or +1";
      return ISING_ERR_ARG;
    }
  }
  return ISING_OK;
}

int basic_observables(ising_ctx* h, int64_t* up, int64_t* E) {
  Device& d = h->devs[0];
  CU(cudaSetDevice(d.dev));
  CU(cudaMemsetAsync(d.red, 0, 2 * sizeof(unsigned long long), d.stream));
  CU(launch_basic_observables(basic_grid(d, h->N * h->M / 2), d.stream, h->bplane[0],
                              h->bplane[1], h->N, h->M / 2, d.red));
  ++h->launch_count;
  unsigned long long v[2];
  CU(cudaMemcpyAsync(v, d.red, sizeof v, cudaMemcpyDeviceToHost, d.stream));
  CU(cudaStreamSynchronize(d.stream));
  *up = (int64_t)v[0];
  *E = 2 * (int64_t)v[1] - 2 * h->N * h->M;
  return ISING_OK;
}

}  // namespace

// ======================================================================= C ABI
extern "C" {

int ising_create(ising_t* out, int64_t L_rows, int64_t L_cols, uint64_t seed, int n_gpus) {
  if (n_gpus < 1) return ISING_ERR_ARG;
  std::vector<int> devs(n_gpus);
  for (int k = 0; k < n_gpus; ++k) devs[k] = k;
  return create_local(out, L_rows, L_cols, seed, n_gpus, devs.data());
}

int ising_create_slabs(ising_t* out, int64_t L_rows, int64_t L_cols, uint64_t seed, int n_slabs,
                       const int* devices) {
  if (!devices || n_slabs < 1) return ISING_ERR_ARG;
  return create_local(out, L_rows, L_cols, seed, n_slabs, devices);
}

int ising_nccl_unique_id(void* id, size_t id_len) {
  if (!id || id_len < sizeof(ncclUniqueId)) return ISING_ERR_ARG;
  ncclUniqueId u;
  NC(ncclGetUniqueId(&u));
  memcpy(id, &u, sizeof u);
  return ISING_OK;
}

int ising_create_rank(ising_t* out, int64_t L_rows, int64_t L_cols, uint64_t seed, int rank,
                      int world, int device, const void* nccl_id, size_t id_len) {
  if (!out || world < 1 || rank < 0 || rank >= world) return ISING_ERR_ARG;
  if (world > 1 && (!nccl_id || id_len < sizeof(ncclUniqueId))) return ISING_ERR_ARG;
  *out = nullptr;
  TRY(check_shape(L_rows, L_cols, world));
  ising_ctx* h = new (std::nothrow) ising_ctx;
  if (!h) return ISING_ERR_OOM;
  h->N = L_rows;
  h->M = L_cols;
  h->W = L_cols / 32;
  h->seed = seed;
  h->rank_mode = true;
  h->rank = rank;
  h->world = world;
  make_keys(seed, &h->keys);
  h->devs.emplace_back();
  int st = setup_device(h->devs[0], device);
  if (st != ISING_OK) {
    destroy_ctx(h);
    return st;
  }
  Slab s;
  s.devi = 0;
  s.R = L_rows / world;
  s.row0 = rank * s.R;
  h->slabs.push_back(s);
  st = alloc_slabs(h);
  h->self_exchange = world == 1 && env_is_one("ISING_SELF_EXCHANGE");
  if (st == ISING_OK && (world > 1 || h->self_exchange)) {
    ncclUniqueId u;
    ncclResult_t r = ncclSuccess;
    if (world > 1)
      memcpy(&u, nccl_id, sizeof u);
    else
      r = ncclGetUniqueId(&u);  // a one-rank communicator: the rank exchanges with itself
    cudaSetDevice(device);
    if (r == ncclSuccess) r = ncclCommInitRank(&h->comm, world, u, rank);
    if (r != ncclSuccess) st = fail_nccl(r, "ncclCommInitRank", __LINE__);
  }
  if (st != ISING_OK) {
    destroy_ctx(h);
    return st;
  }
  read_env_knobs(h);
  *out = h;
  return ISING_OK;
}

int ising_create_rank_p2p(ising_t* out, int64_t L_rows, int64_t L_cols, uint64_t seed, int rank,
                          int world, int device) {
  if (!out || world < 1 || world > kMaxRanks || rank < 0 || rank >= world) return ISING_ERR_ARG;
  *out = nullptr;
  TRY(check_shape(L_rows, L_cols, world));
  ising_ctx* h = new (std::nothrow) ising_ctx;
  if (!h) return ISING_ERR_OOM;
  h->N = L_rows;
  h->M = L_cols;
  h->W = L_cols / 32;
  h->seed = seed;
  h->rank_mode = true;
  h->p2p = true;
  h->rank = rank;
  h->world = world;
  make_keys(seed, &h->keys);
  h->devs.emplace_back();
  int st = setup_device(h->devs[0], device);
  if (st != ISING_OK) {
    destroy_ctx(h);
    return st;
  }
  Slab s;
  s.devi = 0;
  s.R = L_rows / world;
  s.row0 = rank * s.R;
  h->slabs.push_back(s);
  st = alloc_slabs(h);
  if (st == ISING_OK) {
    // zeroed on the handle's (non-blocking) stream and synchronised: a legacy-stream
    // cudaMemset is not ordered before work on a non-blocking stream
    cudaStream_t st0 = h->devs[0].stream;
    cudaError_t e = cudaMalloc(&h->sync, kSyncBytes);
    if (e == cudaSuccess) e = cudaMemsetAsync(h->sync, 0, kSyncBytes, st0);
    if (e == cudaSuccess) e = cudaMalloc(&h->done_counter, sizeof(unsigned int));
    if (e == cudaSuccess) e = cudaMemsetAsync(h->done_counter, 0, sizeof(unsigned int), st0);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st0);
    if (e != cudaSuccess) st = fail_cuda(e, "rank-p2p sync buffers", __LINE__);
  }
  if (st != ISING_OK) {
    destroy_ctx(h);
    return st;
  }
  if (world == 1) {  // its own neighbour: fused halos into its own rows (flags only in
                     // self-exchange mode)
    h->up_plane[0] = h->dn_plane[0] = h->slabs[0].plane[0];
    h->up_plane[1] = h->dn_plane[1] = h->slabs[0].plane[1];
    h->peer_sync[0] = h->sync;
    h->self_exchange = env_is_one("ISING_SELF_EXCHANGE");
    h->connected = true;
  }
  read_env_knobs(h);
  *out = h;
  return ISING_OK;
}

int ising_create_rank_lsa(ising_t* out, int64_t L_rows, int64_t L_cols, uint64_t seed, int rank,
                          int world, int device, const void* nccl_id, size_t id_len) {
  if (!out || world < 1 || world > kMaxRanks || rank < 0 || rank >= world) return ISING_ERR_ARG;
  if (world > 1 && (!nccl_id || id_len < sizeof(ncclUniqueId))) return ISING_ERR_ARG;
  *out = nullptr;
  TRY(check_shape(L_rows, L_cols, world));
  ising_ctx* h = new (std::nothrow) ising_ctx;
  if (!h) return ISING_ERR_OOM;
  h->N = L_rows;
  h->M = L_cols;
  h->W = L_cols / 32;
  h->seed = seed;
  h->rank_mode = true;
  h->p2p = true;  // the same fused peer-store + flag protocol as rank-p2p
  h->lsa = true;
  h->rank = rank;
  h->world = world;
  make_keys(seed, &h->keys);
  h->devs.emplace_back();
  auto fail = [&](int st) {
    destroy_ctx(h);
    return st;
  };
  int st = setup_device(h->devs[0], device);
  if (st != ISING_OK) return fail(st);
  Device& d = h->devs[0];
  {
    ncclUniqueId u;
    ncclResult_t r = ncclSuccess;
    if (world > 1)
      memcpy(&u, nccl_id, sizeof u);
    else
      r = ncclGetUniqueId(&u);
    if (r == ncclSuccess) r = ncclCommInitRank(&h->comm, world, u, rank);
    if (r != ncclSuccess) return fail(fail_nccl(r, "ncclCommInitRank", __LINE__));
  }
  Slab sl;
  sl.devi = 0;
  sl.R = L_rows / world;
  sl.row0 = rank * sl.R;
  h->slabs.push_back(sl);
  Slab& s = h->slabs[0];
  const size_t bytes = (size_t)(s.R + 2) * (size_t)h->W * sizeof(uint64_t);
  // symmetric allocations and windows, in the same order on every rank (collective)
  ncclResult_t r = ncclSuccess;
  for (int c = 0; c < 2 && r == ncclSuccess; ++c) r = ncclMemAlloc((void**)&s.plane[c], bytes);
  if (r == ncclSuccess) r = ncclMemAlloc((void**)&h->sync, kSyncBytes);
  if (r != ncclSuccess) return fail(fail_nccl(r, "ncclMemAlloc", __LINE__));
  cudaError_t e = cudaSuccess;
  for (int c = 0; c < 2 && e == cudaSuccess; ++c) e = cudaMemsetAsync(s.plane[c], 0, bytes, d.stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(h->sync, 0, kSyncBytes, d.stream);
  if (e == cudaSuccess) e = cudaMalloc(&h->done_counter, sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemsetAsync(h->done_counter, 0, sizeof(unsigned int), d.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(d.stream);
  if (e != cudaSuccess) return fail(fail_cuda(e, "rank-lsa buffers", __LINE__));
  for (int c = 0; c < 2 && r == ncclSuccess; ++c)
    r = ncclCommWindowRegister(h->comm, s.plane[c], bytes, &h->win[c], NCCL_WIN_COLL_SYMMETRIC);
  if (r == ncclSuccess)
    r = ncclCommWindowRegister(h->comm, h->sync, kSyncBytes, &h->win[2], NCCL_WIN_COLL_SYMMETRIC);
  if (r != ncclSuccess) return fail(fail_nccl(r, "ncclCommWindowRegister", __LINE__));
  // every rank must be reachable by load / store (one NVLink domain): LSA rank of each rank
  const ncclTeam_t wt = ncclTeamWorld(h->comm), lt = ncclTeamLsa(h->comm);
  int lsa_rank[kMaxRanks];
  for (int q = 0; q < world; ++q) {
    if (!ncclTeamRankIsMember(lt, wt, q)) {
      g_last_error = "ising_create_rank_lsa: a rank is outside this rank's load/store (LSA) team";
      return fail(ISING_ERR_NCCL);
    }
    lsa_rank[q] = ncclTeamRankToLsa(h->comm, wt, q);
  }
  void* ptrs[2 + 2 + kMaxRanks] = {};  // up planes, down planes, every rank's sync area
  const int up = (rank + world - 1) % world, dn = (rank + 1) % world;
  e = lsa_peer_pointers(d.stream, h->win, lsa_rank[up], lsa_rank[dn], lsa_rank, world, ptrs);
  if (e != cudaSuccess) return fail(fail_cuda(e, "ncclGetLsaPointer", __LINE__));
  for (int c = 0; c < 2; ++c) {
    h->up_plane[c] = (uint64_t*)ptrs[c];
    h->dn_plane[c] = (uint64_t*)ptrs[2 + c];
  }
  for (int q = 0; q < world; ++q) h->peer_sync[q] = (unsigned long long*)ptrs[4 + q];
  h->self_exchange = world == 1 && env_is_one("ISING_SELF_EXCHANGE");
  h->connected = true;
  read_env_knobs(h);
  *out = h;
  return ISING_OK;
}

int ising_create_basic(ising_t* out, int64_t L_rows, int64_t L_cols, uint64_t seed, int device) {
  if (!out) return ISING_ERR_ARG;
  *out = nullptr;
  if (L_rows < 2 || (L_rows & 1) || L_cols < 8 || (L_cols % 8) != 0) {
    g_last_error = "basic layout: need L_rows even >= 2 and L_cols % 8 == 0";
    return ISING_ERR_ARG;
  }
  if (L_rows > kMaxRows || L_cols > kMaxCols) {  // same draw-counter limits as check_shape
    g_last_error = "basic layout: need L_rows <= 2^32 and L_cols <= 2^35";
    return ISING_ERR_ARG;
  }
  ising_ctx* h = new (std::nothrow) ising_ctx;
  if (!h) return ISING_ERR_OOM;
  h->N = L_rows;
  h->M = L_cols;
  h->W = 0;
  h->seed = seed;
  h->basic = true;
  make_keys(seed, &h->keys);
  h->devs.emplace_back();
  int st = setup_device(h->devs[0], device);
  if (st == ISING_OK) {
    const size_t bytes = (size_t)(L_rows * (L_cols / 2));
    for (int c = 0; c < 2 && st == ISING_OK; ++c) {
      // same stream as every later kernel on these planes (k_basic_init must not race a
      // legacy-stream memset)
      cudaError_t e = cudaMalloc(&h->bplane[c], bytes);
      if (e == cudaSuccess) e = cudaMemsetAsync(h->bplane[c], 1, bytes, h->devs[0].stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(h->devs[0].stream);
      if (e != cudaSuccess) st = fail_cuda(e, "basic planes", __LINE__);
    }
  }
  if (st != ISING_OK) {
    destroy_ctx(h);
    return st;
  }
  read_env_knobs(h);
  *out = h;
  return ISING_OK;
}

int ising_ipc_handle(ising_t h, void* blob, size_t len) {
  if (!h || !blob || len < ISING_IPC_BLOB_BYTES || !h->p2p) return ISING_ERR_ARG;
  IpcBlob b{};
  b.magic = kIpcMagic;
  b.rank = h->rank;
  b.world = h->world;
  b.R = h->slabs[0].R;
  b.W = h->W;
  CU(cudaSetDevice(h->devs[0].dev));
  CU(cudaIpcGetMemHandle(&b.plane[0], h->slabs[0].plane[0]));
  CU(cudaIpcGetMemHandle(&b.plane[1], h->slabs[0].plane[1]));
  CU(cudaIpcGetMemHandle(&b.sync, h->sync));
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, h->devs[0].dev));
  memcpy(b.uuid, prop.uuid.bytes, sizeof b.uuid);
  memset(blob, 0, ISING_IPC_BLOB_BYTES);
  memcpy(blob, &b, sizeof b);
  return ISING_OK;
}

int ising_ipc_connect(ising_t h, const void* blobs, size_t len) {
  if (!h || !h->p2p || !blobs || len < (size_t)h->world * ISING_IPC_BLOB_BYTES) return ISING_ERR_ARG;
  if (h->connected) return ISING_OK;
  CU(cudaSetDevice(h->devs[0].dev));
  const int up = (h->rank + h->world - 1) % h->world, dn = (h->rank + 1) % h->world;
  std::vector<IpcBlob> all(h->world);
  for (int r = 0; r < h->world; ++r) {
    memcpy(&all[r], (const char*)blobs + (size_t)r * ISING_IPC_BLOB_BYTES, sizeof(IpcBlob));
    if (all[r].magic != kIpcMagic || all[r].rank != r || all[r].world != h->world ||
        all[r].R != h->slabs[0].R || all[r].W != h->W) {
      g_last_error = "ising_ipc_connect: blobs not from this lattice / rank order";
      return ISING_ERR_ARG;
    }
  }
  // Ranks of several processes on one GPU (testing; with MPS their kernels run concurrently):
  // no programmatic dependent launch, for the reason given in ising_p2p_connect_local.
  for (int r = 0; r < h->world; ++r)
    if (r != h->rank && memcmp(all[r].uuid, all[h->rank].uuid, sizeof all[r].uuid) == 0)
      h->pdl = false;
  for (int r = 0; r < h->world; ++r) {
    if (r == h->rank) {
      h->peer_sync[r] = h->sync;
      continue;
    }
    void* ptr = nullptr;
    CU(cudaIpcOpenMemHandle(&ptr, all[r].sync, cudaIpcMemLazyEnablePeerAccess));
    h->opened.push_back(ptr);
    h->peer_sync[r] = (unsigned long long*)ptr;
    if (r == up || r == dn) {
      for (int c = 0; c < 2; ++c) {
        CU(cudaIpcOpenMemHandle(&ptr, all[r].plane[c], cudaIpcMemLazyEnablePeerAccess));
        h->opened.push_back(ptr);
        if (r == up) h->up_plane[c] = (uint64_t*)ptr;
        if (r == dn) h->dn_plane[c] = (uint64_t*)ptr;
      }
    }
  }
  h->connected = true;
  return ISING_OK;
}

int ising_p2p_connect_local(const ising_t* handles, int n) {
  if (!handles || n < 1 || n > kMaxRanks) return ISING_ERR_ARG;
  for (int r = 0; r < n; ++r) {
    const ising_t h = handles[r];
    if (!h || !h->p2p || h->world != n || h->rank != r || h->N != handles[0]->N ||
        h->M != handles[0]->M || h->seed != handles[0]->seed) {
      g_last_error = "ising_p2p_connect_local: handles[r] must be rank r of one rank-p2p lattice";
      return ISING_ERR_ARG;
    }
  }
  if (n == 1) return ISING_OK;  // connected at creation
  // Ranks sharing a device: no programmatic dependent launch.  A PDL-launched half-sweep's
  // blocks become resident as soon as the previous one's have started and then wait for it
  // to finish; while that one spins on another rank's flags, the waiting grids of several
  // ranks can hold every SM slot, so the awaited rank's phase never gets resident (observed:
  // 4 ranks of 8192 x 32768 on one B200 deadlocked).  Ranks on separate GPUs keep PDL.
  bool shared = false;
  for (int r = 0; r < n; ++r)
    for (int q = 0; q < r; ++q) shared |= handles[r]->devs[0].dev == handles[q]->devs[0].dev;
  if (shared)
    for (int r = 0; r < n; ++r) handles[r]->pdl = false;
  for (int r = 0; r < n; ++r) {
    ising_t h = handles[r];
    if (h->connected) continue;
    const int up = (r + n - 1) % n, dn = (r + 1) % n;
    const int dev = h->devs[0].dev;
    CU(cudaSetDevice(dev));
    for (int q : {up, dn}) {  // direct peer access to the neighbours' memory (NVLink P2P)
      const int qd = handles[q]->devs[0].dev;
      if (qd == dev) continue;
      int can = 0;
      CU(cudaDeviceCanAccessPeer(&can, dev, qd));
      if (!can) {
        g_last_error = "ising_p2p_connect_local: no P2P access between neighbouring devices";
        return ISING_ERR_DEVICE;
      }
      cudaError_t e = cudaDeviceEnablePeerAccess(qd, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled)
        cudaGetLastError();
      else if (e != cudaSuccess)
        return fail_cuda(e, "cudaDeviceEnablePeerAccess", __LINE__);
    }
    for (int q = 0; q < n; ++q) h->peer_sync[q] = handles[q]->sync;
    for (int c = 0; c < 2; ++c) {
      h->up_plane[c] = handles[up]->slabs[0].plane[c];
      h->dn_plane[c] = handles[dn]->slabs[0].plane[c];
    }
    h->connected = true;
  }
  return ISING_OK;
}

int ising_destroy(ising_t h) {
  destroy_ctx(h);
  return ISING_OK;
}

int ising_set_rule(ising_t h, int rule) {
  if (!h || (rule != ISING_RULE_METROPOLIS && rule != ISING_RULE_HEATBATH)) return ISING_ERR_ARG;
  h->rule = rule;
  if (h->gexec) {  // the graph bakes the kernel variant and thresholds
    cudaGraphExecDestroy(h->gexec);
    h->gexec = nullptr;
  }
  if (h->gexec_meas) {
    cudaGraphExecDestroy(h->gexec_meas);
    h->gexec_meas = nullptr;
  }
  if (h->beta_set) return ising_set_beta(h, h->beta);
  return ISING_OK;
}

int ising_set_beta(ising_t h, double beta) {
  if (!h || std::isnan(beta) || beta < 0) return ISING_ERR_ARG;
  h->beta = beta;
  if (h->gexec) {
    cudaGraphExecDestroy(h->gexec);
    h->gexec = nullptr;
  }
  if (h->gexec_meas) {
    cudaGraphExecDestroy(h->gexec_meas);
    h->gexec_meas = nullptr;
  }
  compute_thresholds(beta, h->rule, h->T);
  h->acc = make_accept(h->T);
  h->beta_set = true;
  return ISING_OK;
}

int ising_init_random(ising_t h) {
  if (!h) return ISING_ERR_ARG;
  return h->basic ? basic_init(h, 0) : run_init(h, 0);
}
int ising_init_cold(ising_t h) {
  if (!h) return ISING_ERR_ARG;
  return h->basic ? basic_init(h, 1) : run_init(h, 1);
}

// Load the lattice from host memory: +-1 bytes (row_bytes = M) or the bit-packed format
// (bits: row_bytes = M / 8).  Rank mode takes either the full lattice (its rows and halo rows
// are packed straight from it) or exactly its own R rows (then the halo rows are exchanged on
// device).
static int write_impl(ising_t h, const int8_t* in, int64_t in_len, uint64_t t, bool bits) {
  if (!h || !in) return ISING_ERR_ARG;
  if (t > 0xffffffffull) return ISING_ERR_RANGE;
  if (h->basic) {
    if (bits) {
      g_last_error = "bit-packed lattice I/O is for the multi-spin layout";
      return ISING_ERR_ARG;
    }
    if (in_len < h->N * h->M) return ISING_ERR_RANGE;
    TRY(basic_convert(h, const_cast<int8_t*>(in), false));
    h->t = t;
    h->state_set = true;
    return ISING_OK;
  }
  const int64_t row_bytes = bits ? h->M / 8 : h->M;
  const bool slab_only = h->rank_mode && h->world > 1 && in_len == h->slabs[0].R * row_bytes;
  if (!slab_only && in_len < h->N * row_bytes) return ISING_ERR_RANGE;
  if (h->p2p && h->world > 1 && !h->connected) return ISING_ERR_STATE;
  if (p2p_flags(h)) {
    // wait (by polling the stream, not inside a copy) until the neighbours are done with
    // this slab's halo rows, before any possibly pageable host copy is issued (see the
    // rank-p2p branch of ising_sweep_measure)
    TRY(p2p_wait(h));
    TRY(wait_stream(h, h->devs[0].stream));
  }
  for (auto& s : h->slabs) {
    Device& d = h->devs[s.devi];
    CU(cudaSetDevice(d.dev));
    TRY(ensure_staging(d, row_bytes));
    CU(launch_zero_u64(d.stream, d.red, 4));  // a kernel, not a memset (see launch_zero_u64)
    ++h->launch_count;
    const int64_t rpc = staging_rows(d, row_bytes);
    const int64_t r_lo = slab_only ? 0 : -1, r_hi = slab_only ? s.R : s.R + 1;
    const int64_t nchunks = (r_hi - r_lo + rpc - 1) / rpc;
    auto span = [&](int64_t k, int64_t* ra, int64_t* rb) {
      *ra = r_lo + k * rpc;
      *rb = std::min<int64_t>(*ra + rpc, r_hi);
    };
    // H2D of chunk k + 1 overlaps the packing of chunk k (pipeline_in)
    auto copy = [&](int64_t k, int8_t* buf, cudaStream_t st) -> int {
      int64_t ra, rb;
      span(k, &ra, &rb);
      if (slab_only)
        CU(cudaMemcpyAsync(buf, in + ra * row_bytes, (size_t)((rb - ra) * row_bytes),
                           cudaMemcpyHostToDevice, st));
      else
        TRY(h2d_rows(h, buf, in, s.row0 + ra, rb - ra, st, row_bytes));
      return ISING_OK;
    };
    auto kern = [&](int64_t k, int8_t* buf, cudaStream_t st) -> int {
      int64_t ra, rb;
      span(k, &ra, &rb);
      if (bits) {  // every bit pattern is a valid lattice: nothing to validate
        PackBitsParams p;
        p.plane[0] = s.plane[0];
        p.plane[1] = s.plane[1];
        p.bits = reinterpret_cast<const uint32_t*>(buf);
        p.W = h->W;
        p.row0 = s.row0;
        p.N = h->N;
        p.ra = (int32_t)ra;
        p.rb = (int32_t)rb;
        const int64_t total = (rb - ra) * h->W;
        CU(launch_pack_bits((int)std::min<int64_t>((total + 255) / 256, (int64_t)d.sms * 64), st, p));
        ++h->launch_count;
        return ISING_OK;
      }
      PackParams p;
      p.plane[0] = s.plane[0];
      p.plane[1] = s.plane[1];
      p.full = buf;
      p.W = h->W;
      p.M = h->M;
      p.row0 = s.row0;
      p.N = h->N;
      p.ra = (int32_t)ra;
      p.rb = (int32_t)rb;
      p.bad = reinterpret_cast<unsigned int*>(d.red + 2);
      const int64_t total = 2 * (rb - ra) * h->W;
      const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)d.sms * 64);
      k_pack<<<grid, 256, 0, st>>>(p);
      CU(cudaGetLastError());
      ++h->launch_count;
      return ISING_OK;
    };
    TRY(pipeline_in(d, nchunks, copy, kern));
  }
  if (slab_only) TRY(exchange_halos(h));
  TRY(p2p_publish(h));
  TRY(sync_all(h));
  for (auto& s : h->slabs) {
    Device& d = h->devs[s.devi];
    CU(cudaSetDevice(d.dev));
    unsigned long long bad = 0;
    CU(cudaMemcpy(&bad, d.red + 2, sizeof bad, cudaMemcpyDeviceToHost));
    if (bad & 0xffffffffull) {
      g_last_error = "ising_write_lattice: values must be -1 or +1";
      return ISING_ERR_ARG;
    }
  }
  h->t = t;
  h->state_set = true;
  return ISING_OK;
}

int ising_write_lattice(ising_t h, const int8_t* in, int64_t in_len, uint64_t t) {
  return write_impl(h, in, in_len, t, false);
}

int ising_write_lattice_bits(ising_t h, const uint8_t* in, int64_t in_len, uint64_t t) {
  return write_impl(h, reinterpret_cast<const int8_t*>(in), in_len, t, true);
}

int ising_sweep(ising_t h, int64_t n) {
  if (!h || n < 0) return ISING_ERR_ARG;
  if (h->comm_aborted) return nccl_poll(h);
  if (!h->beta_set || !h->state_set) return ISING_ERR_STATE;
  if (h->p2p && h->world > 1 && !h->connected) return ISING_ERR_STATE;
  if (h->t + (uint64_t)n > 0xffffffffull) return ISING_ERR_RANGE;
  NvtxRange range("ising_sweep n=%lld t0=%lld", n, (long long)h->t);
  TRY(ensure_prof_events(h, n));
  h->kernel_launches = 0;
  for (auto& d : h->devs) {
    CU(cudaSetDevice(d.dev));
    CU(cudaEventRecord(d.ev_t0, d.stream));
  }
  h->prof_active = h->profiling;
  const int est = h->basic ? basic_enqueue_sweeps(h, n) : enqueue_sweeps(h, n);
  h->prof_active = false;
  TRY(est);
  for (auto& d : h->devs) {
    CU(cudaSetDevice(d.dev));
    CU(cudaEventRecord(d.ev_t1, d.stream));
  }
  TRY(sync_all(h));
  double mx = 0;
  for (auto& d : h->devs) {
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, d.ev_t0, d.ev_t1));
    mx = std::max(mx, (double)ms);
  }
  h->last_ms = mx;
  if (h->profiling) {
    double tot = 0;
    for (int64_t k = 0; k < h->kernel_launches; ++k) {
      float ms = 0;
      CU(cudaEventElapsedTime(&ms, h->prof_events[2 * k], h->prof_events[2 * k + 1]));
      tot += ms;
    }
    h->kernel_ms = tot;
  }
  return ISING_OK;
}

static int read_impl(ising_t h, int8_t* out, int64_t out_len, bool bits) {
  if (!h || !out) return ISING_ERR_ARG;
  if (bits && h->basic) {
    g_last_error = "bit-packed lattice I/O is for the multi-spin layout";
    return ISING_ERR_ARG;
  }
  const int64_t row_bytes = bits ? h->M / 8 : h->M;
  // rank mode: a buffer of exactly R rows receives this rank's rows at offset 0
  const bool slab_only = h->rank_mode && h->world > 1 && out_len == h->slabs[0].R * row_bytes;
  if (!slab_only && out_len < h->N * row_bytes) return ISING_ERR_RANGE;
  if (!h->state_set) return ISING_ERR_STATE;
  if (h->basic) return basic_convert(h, out, true);
  for (auto& s : h->slabs) {
    // local rows [0, R) of this slab -> host rows starting at its global row (or at 0)
    TRY(unpack_rows_to_host(h, s, 0, s.R, out + (slab_only ? 0 : s.row0) * row_bytes, bits));
  }
  TRY(sync_all(h));
  return ISING_OK;
}

int ising_read_lattice(ising_t h, int8_t* out, int64_t out_len) {
  return read_impl(h, out, out_len, false);
}

int ising_read_lattice_bits(ising_t h, uint8_t* out, int64_t out_len) {
  return read_impl(h, reinterpret_cast<int8_t*>(out), out_len, true);
}

int ising_read_rows(ising_t h, int64_t row_begin, int64_t nrows, int8_t* out, int64_t out_len) {
  if (!h || !out || row_begin < 0 || nrows < 0 || row_begin + nrows > h->N) return ISING_ERR_ARG;
  if (out_len < nrows * h->M) return ISING_ERR_RANGE;
  if (!h->state_set) return ISING_ERR_STATE;
  if (nrows == 0) return ISING_OK;
  if (h->basic) {
    Device& d = h->devs[0];
    CU(cudaSetDevice(d.dev));
    TRY(ensure_staging(d, h->M));
    const int64_t rpc = staging_rows(d, h->M);
    auto rows_of = [&](int64_t k) { return std::min<int64_t>(rpc, nrows - k * rpc); };
    auto kern = [&](int64_t k, int8_t* buf, cudaStream_t st) -> int {
      CU(launch_basic_convert(basic_grid(d, rows_of(k) * h->M), st, h->bplane[0], h->bplane[1],
                              buf, h->M / 2, row_begin + k * rpc, rows_of(k), 1, nullptr));
      ++h->launch_count;
      return ISING_OK;
    };
    auto copy = [&](int64_t k, int8_t* buf, cudaStream_t st) -> int {
      CU(cudaMemcpyAsync(out + k * rpc * h->M, buf, (size_t)(rows_of(k) * h->M),
                         cudaMemcpyDeviceToHost, st));
      return ISING_OK;
    };
    TRY(pipeline_out(d, (nrows + rpc - 1) / rpc, kern, copy));
    CU(cudaStreamSynchronize(d.stream));
    return ISING_OK;
  }
  int64_t covered = 0;
  for (auto& s : h->slabs) {
    const int64_t lo = std::max(row_begin, s.row0), hi = std::min(row_begin + nrows, s.row0 + s.R);
    if (lo >= hi) continue;
    covered += hi - lo;
    TRY(unpack_rows_to_host(h, s, lo - s.row0, hi - s.row0, out + (lo - row_begin) * h->M));
  }
  TRY(sync_all(h));
  if (covered != nrows) {
    g_last_error = "ising_read_rows: rows outside this process's slab";
    return ISING_ERR_ARG;
  }
  return ISING_OK;
}

int ising_observables(ising_t h, int64_t* up_count, int64_t* bond_energy) {
  if (!h || !up_count || !bond_energy) return ISING_ERR_ARG;
  if (h->comm_aborted) return nccl_poll(h);
  if (!h->state_set) return ISING_ERR_STATE;
  if (h->basic) return basic_observables(h, up_count, bond_energy);
  TRY(p2p_wait(h));  // the neighbours' last phase wrote this slab's white halo rows
  std::vector<unsigned long long*> outs;
  for (auto& d : h->devs) {
    CU(cudaSetDevice(d.dev));
    CU(launch_zero_u64(d.stream, d.red, 2));  // a kernel, not a memset (see launch_zero_u64)
    ++h->launch_count;
    outs.push_back(d.red);
  }
  TRY(enqueue_observables(h, outs));
  if (p2p_flags(h)) {
    // all-reduce of the two partials over peer memory
    Device& d = h->devs[0];
    GatherParams g{};
    g.local = d.red;
    for (int r = 0; r < h->world; ++r) g.slots[r] = h->peer_sync[r] + kGatherOffset;
    g.mine = h->sync + kGatherOffset;
    g.out = d.red;
    g.world = h->world;
    g.rank = h->rank;
    g.epoch = ++h->gather_epoch;
    CU(launch_gather(d.stream, g));
    ++h->launch_count;
  } else if (nccl_halos(h)) {
    Device& d = h->devs[0];
    NC(ncclAllReduce(d.red, d.red, 2, ncclUint64, ncclSum, h->comm, d.stream));
  }
  TRY(sync_all(h));
  unsigned long long up = 0, anti = 0;
  for (auto& d : h->devs) {
    unsigned long long v[2];
    CU(cudaSetDevice(d.dev));
    CU(cudaMemcpy(v, d.red, sizeof v, cudaMemcpyDeviceToHost));
    up += v[0];
    anti += v[1];
  }
  *up_count = (int64_t)up;
  *bond_energy = 2 * (int64_t)anti - 2 * h->N * h->M;
  return ISING_OK;
}

// Enqueue n_samples x `every` sweeps with the observables of every sample's white phase
// reduced into each device's meas buffer ([up, antiparallel] per sample), bracketed by the
// devices' ev_t0 / ev_t1 events.  Single-process handles (not rank mode); basic-layout
// handles with the SWAR kernel (basic_fused_obs).
static int measure_enqueue(ising_ctx* h, int64_t n_samples, int64_t every) {
  const size_t need = (size_t)std::max<int64_t>(n_samples, 1) * 2;
  const bool zero_slots =
      h->basic || (n_samples > 0 && persistent_eligible(h)) ||
      (graph_eligible(h) && every <= kGraphSweeps && n_samples >= std::max<int64_t>(1, kGraphSweeps / every));
  std::vector<unsigned long long*> base;
  for (auto& d : h->devs) {
    CU(cudaSetDevice(d.dev));
    if (d.meas_cap < need) {
      if (d.meas) CU(cudaFree(d.meas));
      d.meas = nullptr;
      d.meas_cap = 0;
      CU(cudaMalloc(&d.meas, need * sizeof(unsigned long long)));
      d.meas_cap = need;
    }
    // directly launched samples zero their own slot in their black phase (obs_clear); the
    // graph-replayed and persistent paths add into slots zeroed here
    if (zero_slots) CU(cudaMemsetAsync(d.meas, 0, need * sizeof(unsigned long long), d.stream));
    base.push_back(d.meas);
    CU(cudaEventRecord(d.ev_t0, d.stream));
  }
  std::vector<unsigned long long*> slot(base.size());
  if (h->basic) {  // byte layout: observables fused into each sample's last white phase
    for (int64_t k = 0; k < n_samples; ++k) TRY(basic_enqueue_sweeps(h, every, base[0] + 2 * k));
  } else if (n_samples > 0 && persistent_eligible(h)) {
    TRY(run_persistent(h, n_samples * every, base[0], every));  // the whole chain, one launch
  } else {
    int64_t k0 = 0;
    const int64_t S = std::max<int64_t>(1, kGraphSweeps / every);
    if (graph_eligible(h) && every <= kGraphSweeps && n_samples >= S) {
      if (!h->gexec_meas || h->meas_every != every || h->meas_base != base[0])
        TRY(build_measure_graph(h, every, base[0]));
      Device& d = h->devs[0];
      CU(launch_set_u32(d.stream, h->t_dev, (uint32_t)h->t, 0));
      CU(launch_set_u32(d.stream, h->t_dev + 1, 0u, 0));
      h->launch_count += 2;
      const int64_t reps = n_samples / S;
      for (int64_t r = 0; r < reps; ++r) {
        CU(cudaGraphLaunch(h->gexec_meas, d.stream));
        h->launch_count += h->meas_graph_launches;
      }
      h->t += (uint64_t)(reps * S * every);
      k0 = reps * S;
    }
    for (int64_t k = k0; k < n_samples; ++k) {
      for (size_t d = 0; d < base.size(); ++d) slot[d] = base[d] + 2 * k;
      TRY(enqueue_sweeps(h, every, &slot));  // observables fused into the last white phase
    }
  }
  for (auto& d : h->devs) {
    CU(cudaSetDevice(d.dev));
    CU(cudaEventRecord(d.ev_t1, d.stream));
  }
  return ISING_OK;
}

int ising_sweep_measure(ising_t h, int64_t n_samples, int64_t every, int64_t* up_counts,
                        int64_t* bond_energies) {
  if (!h || n_samples < 0 || every < 1 || (n_samples > 0 && (!up_counts || !bond_energies)))
    return ISING_ERR_ARG;
  if (!h->beta_set || !h->state_set) return ISING_ERR_STATE;
  if (h->t + (uint64_t)(n_samples * every) > 0xffffffffull) return ISING_ERR_RANGE;
  if (p2p_flags(h)) {
    // rank-p2p: the sample's observables are fused into its last white phase (this slab's
    // partials), then all-reduced over peer memory (k_gather) and read back; one host sync
    // per sample keeps consecutive gathers of the shared slots apart
    Device& d = h->devs[0];
    CU(cudaSetDevice(d.dev));
    double total = 0;
    std::vector<unsigned long long*> red{d.red};
    for (int64_t k = 0; k < n_samples; ++k) {
      // (no memset: the black phase of the sample's last sweep zeroes d.red, obs_clear)
      CU(cudaEventRecord(d.ev_t0, d.stream));
      TRY(enqueue_sweeps(h, every, &red));
      CU(cudaEventRecord(d.ev_t1, d.stream));
      GatherParams g{};
      g.local = d.red;
      for (int r = 0; r < h->world; ++r) g.slots[r] = h->peer_sync[r] + kGatherOffset;
      g.mine = h->sync + kGatherOffset;
      g.out = d.red;
      g.world = h->world;
      g.rank = h->rank;
      g.epoch = ++h->gather_epoch;
      CU(launch_gather(d.stream, g));
      ++h->launch_count;
      // Wait for the stream first: a copy to pageable memory issued while this stream still
      // waits on the other ranks blocks this thread inside the driver, where it can keep the
      // other ranks' threads of the same process (ising_p2p_connect_local) from launching
      // the phases it waits for.
      TRY(wait_stream(h, d.stream));
      unsigned long long v[2];
      CU(cudaMemcpy(v, d.red, sizeof v, cudaMemcpyDeviceToHost));
      float ms = 0;
      CU(cudaEventElapsedTime(&ms, d.ev_t0, d.ev_t1));
      total += ms;
      up_counts[k] = (int64_t)v[0];
      bond_energies[k] = 2 * (int64_t)v[1] - 2 * h->N * h->M;
    }
    h->last_ms = total;
    return ISING_OK;
  }
  if (nccl_halos(h) || (h->basic && !basic_fused_obs(h))) {
    // rank-NCCL / listing-shaped basic kernel: sweep, then the separate observables pass
    // (all-reduced over NCCL in rank mode) per sample
    double total = 0;
    for (int64_t k = 0; k < n_samples; ++k) {
      TRY(ising_sweep(h, every));
      total += h->last_ms;
      TRY(ising_observables(h, &up_counts[k], &bond_energies[k]));
    }
    h->last_ms = total;
    return ISING_OK;
  }
  TRY(measure_enqueue(h, n_samples, every));
  const size_t need = (size_t)std::max<int64_t>(n_samples, 1) * 2;
  TRY(sync_all(h));
  double mx = 0;
  std::vector<unsigned long long> host(need);
  for (int64_t k = 0; k < n_samples; ++k) up_counts[k] = bond_energies[k] = 0;
  for (auto& d : h->devs) {
    CU(cudaSetDevice(d.dev));
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, d.ev_t0, d.ev_t1));
    mx = std::max(mx, (double)ms);
    CU(cudaMemcpy(host.data(), d.meas, need * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    for (int64_t k = 0; k < n_samples; ++k) {
      up_counts[k] += (int64_t)host[2 * k];
      bond_energies[k] += (int64_t)host[2 * k + 1];  // antiparallel bonds for now
    }
  }
  for (int64_t k = 0; k < n_samples; ++k) bond_energies[k] = 2 * bond_energies[k] - 2 * h->N * h->M;
  h->last_ms = mx;
  return ISING_OK;
}

int ising_sweep_measure_async(ising_t h, int64_t n_samples, int64_t every, int64_t* up_counts,
                              int64_t* bond_energies, int64_t* ticket) {
  if (!h || !ticket || n_samples < 0 || every < 1 ||
      (n_samples > 0 && (!up_counts || !bond_energies)))
    return ISING_ERR_ARG;
  if (!h->beta_set || !h->state_set) return ISING_ERR_STATE;
  if (h->t + (uint64_t)(n_samples * every) > 0xffffffffull) return ISING_ERR_RANGE;
  PendingMeasure* pm = nullptr;
  for (auto& q : h->pending)
    if (q.ticket < 0) {
      pm = &q;
      break;
    }
  if (!pm) {
    g_last_error = "ising_sweep_measure_async: more than 8 calls pending";
    return ISING_ERR_STATE;
  }
  pm->up = up_counts;
  pm->energy = bond_energies;
  pm->n = n_samples;
  pm->ready = false;
  if (p2p_flags(h) || nccl_halos(h) || (h->basic && !basic_fused_obs(h)) || h->devs.size() > 1 ||
      n_samples == 0) {
    // cross-device reductions: the synchronous path, complete on return
    TRY(ising_sweep_measure(h, n_samples, every, up_counts, bond_energies));
    pm->ready = true;
    pm->ms = h->last_ms;
  } else {
    Device& d = h->devs[0];
    CU(cudaSetDevice(d.dev));
    for (cudaEvent_t* e : {&pm->t0, &pm->t1, &pm->done})
      if (!*e) CU(cudaEventCreate(e));
    CU(cudaEventRecord(pm->t0, d.stream));
    TRY(measure_enqueue(h, n_samples, every));
    CU(cudaEventRecord(pm->t1, d.stream));
    // one copy of the [up, antiparallel] pairs into this slot's pinned landing buffer; the
    // wait splits them into the caller's arrays
    if (pm->host_cap < (size_t)n_samples) {
      if (pm->host) CU(cudaFreeHost(pm->host));
      pm->host = nullptr;
      pm->host_cap = 0;
      CU(cudaHostAlloc(&pm->host, 2 * sizeof(unsigned long long) * (size_t)n_samples,
                       cudaHostAllocDefault));
      pm->host_cap = (size_t)n_samples;
    }
    CU(cudaMemcpyAsync(pm->host, d.meas, 2 * sizeof(unsigned long long) * (size_t)n_samples,
                       cudaMemcpyDeviceToHost, d.stream));
    CU(cudaEventRecord(pm->done, d.stream));
  }
  pm->ticket = h->next_ticket++;
  *ticket = pm->ticket;
  return ISING_OK;
}

int ising_measure_wait(ising_t h, int64_t ticket) {
  if (!h) return ISING_ERR_ARG;
  PendingMeasure* pm = nullptr;
  for (auto& q : h->pending)
    if (q.ticket >= 0 && q.ticket == ticket) pm = &q;
  if (!pm) return ISING_ERR_ARG;
  if (!pm->ready) {
    CU(cudaSetDevice(h->devs[0].dev));
    CU(cudaEventSynchronize(pm->done));
    for (int64_t k = 0; k < pm->n; ++k) {  // antiparallel bonds -> bond energy (Eq. 1, R11)
      pm->up[k] = (int64_t)pm->host[2 * k];
      pm->energy[k] = 2 * (int64_t)pm->host[2 * k + 1] - 2 * h->N * h->M;
    }
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, pm->t0, pm->t1));
    pm->ms = ms;
  }
  h->last_ms = pm->ms;
  pm->ticket = -1;
  return ISING_OK;
}

int ising_last_sweep_ms(ising_t h, double* device_ms) {
  if (!h || !device_ms) return ISING_ERR_ARG;
  *device_ms = h->last_ms;
  return ISING_OK;
}

int ising_set_profiling(ising_t h, int enable) {
  if (!h) return ISING_ERR_ARG;
  h->profiling = enable != 0;
  return ISING_OK;
}

int ising_kernel_stats(ising_t h, double* kernel_ms, int64_t* launches) {
  if (!h || !kernel_ms || !launches) return ISING_ERR_ARG;
  *kernel_ms = h->kernel_ms;
  *launches = h->kernel_launches;
  return ISING_OK;
}

int ising_get_sweep(ising_t h, uint64_t* t) {
  if (!h || !t) return ISING_ERR_ARG;
  *t = h->t;
  return ISING_OK;
}

int ising_slab_info(ising_t h, int64_t* row0, int64_t* rows) {
  if (!h || !row0 || !rows) return ISING_ERR_ARG;
  if (h->rank_mode) {
    *row0 = h->slabs[0].row0;
    *rows = h->slabs[0].R;
  } else {
    *row0 = 0;
    *rows = h->N;
  }
  return ISING_OK;
}

int ising_thresholds(ising_t h, uint64_t T[5]) {
  if (!h || !T) return ISING_ERR_ARG;
  if (!h->beta_set) return ISING_ERR_STATE;
  for (int a = 0; a < 5; ++a) T[a] = h->T[a];
  return ISING_OK;
}

int ising_launch_count(ising_t h, int64_t* launches) {
  if (!h || !launches) return ISING_ERR_ARG;
  *launches = h->launch_count;
  return ISING_OK;
}

int ising_kernel_variant(ising_t h, int* variant) {
  if (!h || !variant) return ISING_ERR_ARG;
  *variant = kernel_variant(h);
  return ISING_OK;
}

int ising_probe_philox(int device, double* draws_per_ns) {
  if (!draws_per_ns) return ISING_ERR_ARG;
  Device d;
  int st = setup_device(d, device);
  if (st != ISING_OK) return st;
  PhiloxKeys K;
  make_keys(0x0123456789abcdefull, &K);
  unsigned int* sink = nullptr;
  CU(cudaMalloc(&sink, sizeof(unsigned int)));
  const int grid = d.sms * 16;  // 2048 threads per SM
  const uint32_t per_thread = 2048;
  cudaEvent_t a, b;
  CU(cudaEventCreate(&a));
  CU(cudaEventCreate(&b));
  double best = 0;
  for (int rep = 0; rep < 4; ++rep) {
    CU(cudaEventRecord(a, d.stream));
    CU(launch_philox_probe(grid, d.stream, K, per_thread, sink));
    CU(cudaEventRecord(b, d.stream));
    CU(cudaEventSynchronize(b));
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, a, b));
    const double draws = 4.0 * grid * 128.0 * per_thread;
    if (rep > 0) best = std::max(best, draws / (ms * 1e6));
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  teardown_device(d);
  *draws_per_ns = best;
  return ISING_OK;
}

// ------------------------------------------------------------- lattice batches
// ising_batch_*: n independent L_rows x L_cols lattices on one device, each with its own seed
// and beta, one CTA per lattice holding it in shared memory for a chunk of sweeps
// (k_batch_sweeps).  SURVEY §8(f) row f2 (temperature scans / Binder analysis on small L).
struct ising_batch {
  int64_t N = 0, M = 0, W = 0;
  int n = 0;
  Device d;
  uint64_t* planes = nullptr;
  BatchLattice* lat_dev = nullptr;
  std::vector<BatchLattice> lat;
  int rule = ISING_RULE_METROPOLIS;
  int variant = 2;  // kernel variant every lattice shares (kernel_variant's numbering), 1: mixed HB
  bool beta_set = false, state_set = false;
  uint64_t t = 0;
  double last_ms = 0;
  int threads = 0;
  int cluster = 1;  // CTAs per lattice (1: k_batch_sweeps; > 1: k_batch_cluster_sweeps)
  size_t smem = 0;
  unsigned long long* obs = nullptr;
  size_t obs_cap = 0;  // u64 entries
  int8_t* full = nullptr;
  unsigned int* bad = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
};

namespace {
constexpr uint32_t kBatchSweepsPerLaunch = 4096;

void batch_free(ising_batch* b) {
  if (!b) return;
  if (b->d.dev >= 0) {
    cudaSetDevice(b->d.dev);
    if (b->d.stream) cudaStreamSynchronize(b->d.stream);  // this handle's work only
    for (void* p : {(void*)b->planes, (void*)b->lat_dev, (void*)b->obs, (void*)b->full, (void*)b->bad})
      if (p) cudaFree(p);
    if (b->e0) cudaEventDestroy(b->e0);
    if (b->e1) cudaEventDestroy(b->e1);
    teardown_device(b->d);
  }
  delete b;
}

BatchParams batch_params(const ising_batch* b) {
  BatchParams p{};
  p.planes = b->planes;
  p.lat = b->lat_dev;
  p.N = (int32_t)b->N;
  p.W = (int32_t)b->W;
  p.t0 = (uint32_t)b->t;
  return p;
}

int batch_ensure_obs(ising_batch* b, size_t entries) {
  if (b->obs_cap >= entries) return ISING_OK;
  if (b->obs) cudaFree(b->obs);
  b->obs = nullptr;
  b->obs_cap = 0;
  CU(cudaMalloc(&b->obs, entries * sizeof(unsigned long long)));
  b->obs_cap = entries;
  return ISING_OK;
}

// A lattice's kernel variant (kernel_variant's numbering, without the draw-free 4: batches
// always draw): 0 / 2 Metropolis, 7 / 3 / 5 / 6 heat bath.
int variant_of(int rule, const uint64_t T[5], const Accept& acc) {
  if (rule == ISING_RULE_METROPOLIS) return (acc.keep3 & acc.keep4) == 0xffffffffu ? 0 : 2;
  const uint64_t two32p1 = (uint64_t(1) << 32) + 1;
  if (!env_is_zero("ISING_HB_SYMMETRIC") && T[2] == (uint64_t(1) << 31) && T[0] + T[4] == two32p1 &&
      T[1] + T[3] == two32p1)
    return 7;
  switch (acc.always_mask) {
    case 0: return 3;
    case 1: return 5;
    case 3: return 6;
    default: return 1;
  }
}

cudaError_t batch_launch_sweeps(const ising_batch* b, int variant, const BatchParams& p) {
  if (b->cluster == 1) return launch_batch_sweeps(variant, b->n, b->threads, b->smem, b->d.stream, p);
  return launch_batch_cluster_sweeps(variant, b->n, b->cluster, b->threads, b->smem, b->d.stream, p);
}

// sweeps t + 1 .. t + n (every > 0: observables after every `every` sweeps into slot
// s / every - 1 of each lattice's n_samples), in launches of at most kBatchSweepsPerLaunch
int batch_run(ising_batch* b, int64_t n, int64_t every, int64_t n_samples) {
  NvtxRange r("ising_batch_sweeps %lld x %lld lattices", (long long)n, (long long)b->n);
  CU(cudaSetDevice(b->d.dev));
  CU(cudaEventRecord(b->e0, b->d.stream));
  int64_t done = 0;
  while (done < n) {
    const int64_t chunk = std::min<int64_t>(n - done, kBatchSweepsPerLaunch);
    BatchParams p = batch_params(b);
    p.t0 = (uint32_t)(b->t + done);
    p.sweeps = (uint32_t)chunk;
    if (every > 0) {
      p.every = (uint32_t)every;
      p.n_samples = (uint32_t)n_samples;
      p.s_base = (uint32_t)done;
      p.obs = b->obs;
    }
    CU(batch_launch_sweeps(b, b->variant, p));
    done += chunk;
  }
  CU(cudaEventRecord(b->e1, b->d.stream));
  CU(cudaEventSynchronize(b->e1));
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, b->e0, b->e1));
  b->last_ms = ms;
  b->t += (uint64_t)n;
  return ISING_OK;
}
}  // namespace

int ising_batch_create(ising_batch_t* out, int64_t L_rows, int64_t L_cols, int n_lattices,
                       const uint64_t* seeds, int device) {
  if (!out || !seeds) return ISING_ERR_ARG;
  *out = nullptr;
  // CTAs per lattice: one if both planes fit its shared memory, else the smallest cluster
  // (2 .. 16 CTAs, dividing L_rows) whose row bands plus halo rows fit
  int cluster = 0;
  // (a CTA has a thread per 128-bit column pair of a row: L_cols / 64 <= kBatchMaxThreads)
  if (L_rows >= 2 && L_cols >= 64 && L_cols % 64 == 0 && L_rows <= 65536 &&
      L_cols / 64 <= kBatchMaxThreads) {
    if (L_rows * L_cols / 2 <= (int64_t)kBatchMaxSmem) {
      cluster = 1;
    } else {
      for (int C = 2; C <= 16 && !cluster; C *= 2)
        if (L_rows % C == 0 && L_rows / C >= 2 &&
            (L_rows / C + 2) * (L_cols / 32) * 16 <= (int64_t)kBatchMaxSmem)
          cluster = C;
    }
  }
  if (cluster == 0 || (L_rows & 1) || n_lattices < 1 || n_lattices > 65535) {
    g_last_error = "ising_batch_create: need L_rows even, L_cols % 64 == 0, 1 <= n <= 65535, and "
                   "a lattice that fits one CTA's shared memory (L_rows * L_cols <= 409600) or a "
                   "cluster of up to 16 (L_rows / C + 2) * L_cols / 2 <= 204800 bytes, e.g. 2048^2";
    return ISING_ERR_ARG;
  }
  ising_batch* b = new (std::nothrow) ising_batch;
  if (!b) return ISING_ERR_OOM;
  b->N = L_rows;
  b->M = L_cols;
  b->W = L_cols / 32;
  b->n = n_lattices;
  int st = setup_device(b->d, device);
  if (st != ISING_OK) {
    batch_free(b);
    return st;
  }
  auto fail = [&](int s) {
    batch_free(b);
    return s;
  };
  try {
    b->lat.resize(n_lattices);
  } catch (const std::bad_alloc&) {
    return fail(ISING_ERR_OOM);
  }
  for (int k = 0; k < n_lattices; ++k) {
    make_keys(seeds[k], &b->lat[k].keys);
    b->lat[k].acc = Accept{};
  }
  const size_t words = (size_t)n_lattices * 2 * b->N * b->W;
  cudaError_t e = cudaMalloc(&b->planes, words * sizeof(uint64_t));
  if (e == cudaSuccess) e = cudaMalloc(&b->lat_dev, sizeof(BatchLattice) * n_lattices);
  if (e == cudaSuccess) e = cudaMalloc(&b->full, (size_t)(b->N * b->M));
  if (e == cudaSuccess) e = cudaEventCreate(&b->e0);
  if (e == cudaSuccess) e = cudaEventCreate(&b->e1);
  if (e != cudaSuccess) return fail(fail_cuda(e, "ising_batch_create", __LINE__));
  b->cluster = cluster;
  if (cluster == 1) {
    b->threads = batch_threads((int)b->N, (int)b->W);
    b->smem = (size_t)(2 * b->N * b->W) * sizeof(uint64_t);
  } else {
    const int R = (int)(b->N / cluster);
    b->threads = batch_threads(R, (int)b->W);
    b->smem = (size_t)(2 * (R + 2) * b->W) * sizeof(uint64_t);
  }
  *out = b;
  return ISING_OK;
}

int ising_batch_destroy(ising_batch_t b) {
  batch_free(b);
  return ISING_OK;
}

int ising_batch_set_beta(ising_batch_t b, const double* betas, int rule) {
  if (!b || !betas || (rule != ISING_RULE_METROPOLIS && rule != ISING_RULE_HEATBATH))
    return ISING_ERR_ARG;
  for (int k = 0; k < b->n; ++k)
    if (std::isnan(betas[k]) || betas[k] < 0) return ISING_ERR_ARG;
  int variant = -1;  // the lattices' common kernel variant, if they share one
  for (int k = 0; k < b->n; ++k) {
    uint64_t T[5];
    compute_thresholds(betas[k], rule, T);
    b->lat[k].acc = make_accept(T);
    const int v = variant_of(rule, T, b->lat[k].acc);
    variant = (k == 0 || v == variant) ? v : (rule == ISING_RULE_METROPOLIS ? 2 : 1);
  }
  b->variant = variant;
  CU(cudaSetDevice(b->d.dev));
  CU(cudaMemcpyAsync(b->lat_dev, b->lat.data(), sizeof(BatchLattice) * b->n,
                     cudaMemcpyHostToDevice, b->d.stream));
  CU(cudaStreamSynchronize(b->d.stream));
  b->rule = rule;
  b->beta_set = true;
  return ISING_OK;
}

static int batch_init(ising_batch_t b, int cold) {
  if (!b) return ISING_ERR_ARG;
  CU(cudaSetDevice(b->d.dev));
  if (!b->beta_set) {  // the keys must be on the device for the random start
    CU(cudaMemcpyAsync(b->lat_dev, b->lat.data(), sizeof(BatchLattice) * b->n,
                       cudaMemcpyHostToDevice, b->d.stream));
  }
  CU(launch_batch_init(b->n, cold, b->d.stream, batch_params(b)));
  CU(cudaStreamSynchronize(b->d.stream));
  b->t = 0;
  b->state_set = true;
  return ISING_OK;
}
int ising_batch_init_random(ising_batch_t b) { return batch_init(b, 0); }
int ising_batch_init_cold(ising_batch_t b) { return batch_init(b, 1); }

int ising_batch_sweep(ising_batch_t b, int64_t n) {
  if (!b || n < 0) return ISING_ERR_ARG;
  if (!b->beta_set || !b->state_set) return ISING_ERR_STATE;
  if (b->t + (uint64_t)n > 0xffffffffull) return ISING_ERR_RANGE;
  if (n == 0) return ISING_OK;
  return batch_run(b, n, 0, 0);
}

int ising_batch_sweep_measure(ising_batch_t b, int64_t n_samples, int64_t every,
                              int64_t* up_counts, int64_t* bond_energies) {
  if (!b || n_samples < 0 || every < 1 || !up_counts || !bond_energies) return ISING_ERR_ARG;
  if (!b->beta_set || !b->state_set) return ISING_ERR_STATE;
  if (n_samples > 0 && every > (int64_t)0xffffffff / n_samples) return ISING_ERR_RANGE;
  if (b->t + (uint64_t)(n_samples * every) > 0xffffffffull) return ISING_ERR_RANGE;
  if (n_samples == 0) return ISING_OK;
  const size_t entries = (size_t)b->n * n_samples * 2;
  TRY(batch_ensure_obs(b, entries));
  TRY(batch_run(b, n_samples * every, every, n_samples));
  // copy back in pieces through a bounded host buffer (no allocation of the whole series)
  std::vector<unsigned long long> host;
  try {
    host.resize(std::min<size_t>(entries, size_t(1) << 22));
  } catch (const std::bad_alloc&) {
    return ISING_ERR_OOM;
  }
  for (size_t q0 = 0; q0 < entries; q0 += host.size()) {
    const size_t m = std::min(host.size(), entries - q0);
    CU(cudaMemcpy(host.data(), b->obs + q0, m * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    for (size_t e = 0; e < m; e += 2) {
      const size_t q = (q0 + e) / 2;
      up_counts[q] = (int64_t)host[e];
      bond_energies[q] = 2 * (int64_t)host[e + 1] - 2 * b->N * b->M;
    }
  }
  return ISING_OK;
}

int ising_batch_observables(ising_batch_t b, int64_t* up_counts, int64_t* bond_energies) {
  if (!b || !up_counts || !bond_energies) return ISING_ERR_ARG;
  if (!b->state_set) return ISING_ERR_STATE;
  TRY(batch_ensure_obs(b, (size_t)b->n * 2));
  CU(cudaSetDevice(b->d.dev));
  BatchParams p = batch_params(b);
  p.measure_only = 1;
  p.n_samples = 1;
  p.obs = b->obs;
  CU(batch_launch_sweeps(b, 2, p));  // observables only: no acceptance
  std::vector<unsigned long long> host;
  try {
    host.resize((size_t)b->n * 2);
  } catch (const std::bad_alloc&) {
    return ISING_ERR_OOM;
  }
  CU(cudaMemcpyAsync(host.data(), b->obs, host.size() * sizeof(unsigned long long),
                     cudaMemcpyDeviceToHost, b->d.stream));
  CU(cudaStreamSynchronize(b->d.stream));
  for (int k = 0; k < b->n; ++k) {
    up_counts[k] = (int64_t)host[2 * k];
    bond_energies[k] = 2 * (int64_t)host[2 * k + 1] - 2 * b->N * b->M;
  }
  return ISING_OK;
}

int ising_batch_read_lattice(ising_batch_t b, int lattice, int8_t* out, int64_t out_len) {
  if (!b || !out || lattice < 0 || lattice >= b->n) return ISING_ERR_ARG;
  if (!b->state_set) return ISING_ERR_STATE;
  if (out_len < b->N * b->M) return ISING_ERR_RANGE;
  CU(cudaSetDevice(b->d.dev));
  CU(launch_batch_unpack(lattice, b->d.stream, batch_params(b), b->full));
  CU(cudaMemcpyAsync(out, b->full, (size_t)(b->N * b->M), cudaMemcpyDeviceToHost, b->d.stream));
  CU(cudaStreamSynchronize(b->d.stream));
  return ISING_OK;
}

int ising_batch_write_lattice(ising_batch_t b, int lattice, const int8_t* in, int64_t in_len,
                              uint64_t t) {
  if (!b || !in || lattice < 0 || lattice >= b->n) return ISING_ERR_ARG;
  if (in_len < b->N * b->M) return ISING_ERR_RANGE;
  if (t > 0xffffffffull) return ISING_ERR_RANGE;
  CU(cudaSetDevice(b->d.dev));
  if (!b->bad) CU(cudaMalloc(&b->bad, sizeof(unsigned int)));
  CU(cudaMemsetAsync(b->bad, 0, sizeof(unsigned int), b->d.stream));
  if (!b->beta_set) {  // the keys must be on the device before the first sweep
    CU(cudaMemcpyAsync(b->lat_dev, b->lat.data(), sizeof(BatchLattice) * b->n,
                       cudaMemcpyHostToDevice, b->d.stream));
  }
  if (!b->state_set) {  // the other lattices start cold until written
    CU(launch_batch_init(b->n, 1, b->d.stream, batch_params(b)));
    b->state_set = true;
  }
  CU(cudaMemcpyAsync(b->full, in, (size_t)(b->N * b->M), cudaMemcpyHostToDevice, b->d.stream));
  CU(launch_batch_pack(lattice, b->d.stream, batch_params(b), b->full, b->bad));
  unsigned int bad = 0;
  CU(cudaMemcpyAsync(&bad, b->bad, sizeof bad, cudaMemcpyDeviceToHost, b->d.stream));
  CU(cudaStreamSynchronize(b->d.stream));
  if (bad) {
    g_last_error = "ising_batch_write_lattice: values must be -1 or +1";
    return ISING_ERR_ARG;
  }
  b->t = t;
  return ISING_OK;
}

int ising_batch_last_sweep_ms(ising_batch_t b, double* device_ms) {
  if (!b || !device_ms) return ISING_ERR_ARG;
  *device_ms = b->last_ms;
  return ISING_OK;
}

int ising_batch_get_sweep(ising_batch_t b, uint64_t* t) {
  if (!b || !t) return ISING_ERR_ARG;
  *t = b->t;
  return ISING_OK;
}

const char* ising_strerror(int status) {
  switch (status) {
    case ISING_OK: return "ok";
    case ISING_ERR_ARG: return "invalid argument";
    case ISING_ERR_STATE: return "invalid call order (set_beta and init/write first)";
    case ISING_ERR_DEVICE: return "no suitable sm_100 device";
    case ISING_ERR_OOM: return "out of memory";
    case ISING_ERR_CUDA: return "CUDA error";
    case ISING_ERR_NCCL: return "NCCL error";
    case ISING_ERR_RANGE: return "out of range";
    default: return "unknown status";
  }
}

const char* ising_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"
