/*
 * include/ising.h — C ABI of the B200 checkerboard-Metropolis library (libising.so).
 *
 * The library runs the hot path of arXiv 1906.06297: the checkerboard
 * (red/black) Metropolis sweep of the 2D ferromagnetic Ising model on an
 * L_rows x L_cols periodic lattice, "update all the spins of one color in parallel,
 * keeping the other color constant, and then repeat the process with the opposite
 * color" (§2), with the multi-spin coding of §3.3:
 * the two colours live in separate arrays, four bits per spin, sixteen spins per
 * 64-bit word, and each half-sweep is one sm_100a kernel that forms the four
 * neighbour sums of a whole word with word-wide adds, draws an inline counter-based
 * Philox4x32-10 number per spin and accepts with an integer threshold.
 *
 * Conventions:
 *   - J = 1; beta = 1/T.  Site (i, J) is black iff i + J is even (R1).
 *   - Draw for plane site (i, j = J/2) of colour c (0 black, 1 white) in sweep t:
 *       r = Philox4x32-10(ctr = {t, j/4, c, i}, key = {lo32(seed), hi32(seed)})[j % 4] (R6).
 *   - Metropolis: with e = s*h (h = sum of the 4 neighbours),
 *     flip iff e <= 0 or r < T[e], T[e] = min(2^32, ceil(2^32 exp(-2 beta e))) (R5),
 *     computed on the host in IEEE double.  Heat bath:
 *     flip iff r < ceil(2^32 p/(1+p)), p = exp(-2 beta e), for every e.
 *   - One sweep = black half-sweep then white half-sweep; sweeps are numbered
 *     t = 1, 2, ...; t = 0 is the random initialisation (R7, R8).
 *
 * Status: every call returns ISING_OK (0) or a negative ising_status.  No C++
 * exception crosses the ABI.  A handle is not thread-safe.  The library owns the
 * handle and all device memory; the caller owns every host buffer it passes.
 * Calls that return data synchronise.  ising_sweep returns after the sweeps have
 * completed on every device of the handle.
 */
#ifndef ISING_H
#define ISING_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ising_ctx* ising_t;

enum ising_status {
  ISING_OK = 0,
  ISING_ERR_ARG = -1,    /* invalid argument (shape, beta, pointer, length) */
  ISING_ERR_STATE = -2,  /* call order: sweep before set_beta + init, etc.   */
  ISING_ERR_DEVICE = -3, /* no / too few sm_100 devices, bad device index    */
  ISING_ERR_OOM = -4,    /* device or pinned host allocation failed          */
  ISING_ERR_CUDA = -5,   /* CUDA runtime error (message via ising_last_error)*/
  ISING_ERR_NCCL = -6,   /* NCCL error                                       */
  ISING_ERR_RANGE = -7   /* sweep counter would exceed 2^32 - 1; short buffer*/
};

enum ising_rule {
  ISING_RULE_METROPOLIS = 0, /* PAPER.md:36-42 (the path)                    */
  ISING_RULE_HEATBATH = 1
};

/* ---------------------------------------------------------------- lifetime */

/* Create a lattice of L_rows x L_cols spins split into n_gpus row slabs on CUDA
 * devices 0..n_gpus-1 of this process (§4: "partitioned into
 * horizontal slabs and each GPU stores one slab").  Requirements: L_rows even,
 * L_rows % n_gpus == 0, L_rows / n_gpus >= 2, L_cols % 64 == 0, L_cols >= 64, and the
 * size limits L_rows <= 2^32, L_cols <= 2^35 (the draw counter of R6 holds the row and
 * the plane column / 4 in 32-bit words) and L_rows / n_gpus <= 2^30 (slab rows); every
 * constructor checks them before touching a device.
 * Neighbouring slabs exchange boundary rows by direct peer stores from the
 * half-sweep kernel (NVLink P2P).  *out receives the handle.
 * Errors: ARG (shape, NULL out), DEVICE (fewer than n_gpus sm_100 devices or no
 * P2P between neighbours), OOM, CUDA. */
int ising_create(ising_t* out, int64_t L_rows, int64_t L_cols, uint64_t seed, int n_gpus);

/* As ising_create, with an explicit device for each of n_slabs slabs
 * (devices[k] for global rows [k R, (k+1) R), R = L_rows / n_slabs).  Devices may
 * repeat: slabs on the same device exchange halos through that device's memory.
 * This is how slab decomposition is exercised on a single GPU. */
int ising_create_slabs(ising_t* out, int64_t L_rows, int64_t L_cols, uint64_t seed, int n_slabs,
                       const int* devices);

/* One process per GPU (torchrun): this process owns slab `rank` of `world` on CUDA
 * device `device`; halo rows move by ncclSend/ncclRecv (NCCL over NVLink) overlapped
 * with the interior update.  nccl_id points to id_len (= 128) bytes produced
 * by ising_nccl_unique_id on rank 0 and broadcast by the caller (e.g. torch.distributed).
 * With world == 1 nccl_id may be NULL; the handle then behaves as one slab, unless the
 * environment sets ISING_SELF_EXCHANGE=1: a one-rank communicator is created and every
 * half-sweep exchanges its halo rows with itself by ncclSend/ncclRecv (the transport's
 * per-GPU cost, measurable on one device).  Collective: all ranks must call it.
 * Failure detection: while a call waits for its streams it polls ncclCommGetAsyncError; on an
 * asynchronous error, or when the streams make no progress for ISING_NCCL_TIMEOUT_S seconds
 * (environment, default 300), the communicator is aborted and this and every later call on
 * the handle returns ISING_ERR_NCCL (destroy it). */
int ising_create_rank(ising_t* out, int64_t L_rows, int64_t L_cols, uint64_t seed, int rank,
                      int world, int device, const void* nccl_id, size_t id_len);

/* One process per GPU, halos moved by the half-sweep kernel itself: each rank maps its
 * neighbours' colour planes (CUDA IPC, NVLink P2P), stores its boundary rows straight
 * into their halo rows and raises a flag in their memory when the phase is done; the next
 * phase's kernel waits on the flags of both neighbours (the paper's
 * "read access to the memory of the two GPUs that handle the slabs on top and bottom",
 * PAPER.md:227).  After creation every rank exports ising_ipc_handle, the caller
 * all-gathers the blobs in rank order (e.g. torch.distributed) and passes them to
 * ising_ipc_connect.  world <= 8.  Ranks may share a device (for testing; the blobs carry the
 * device UUID and ranks that share one run without programmatic dependent launch, as in
 * ising_p2p_connect_local — under MPS their kernels run concurrently).  With world == 1
 * the rank is its own neighbour; ISING_SELF_EXCHANGE=1 in the environment makes it run the
 * whole flag protocol with itself (the protocol's per-GPU cost, measurable on one device). */
#define ISING_IPC_BLOB_BYTES 256
int ising_create_rank_p2p(ising_t* out, int64_t L_rows, int64_t L_cols, uint64_t seed, int rank,
                          int world, int device);
int ising_ipc_handle(ising_t h, void* blob, size_t len);            /* len >= 256 */
int ising_ipc_connect(ising_t h, const void* blobs, size_t len);    /* world * 256 bytes */

/* One process per GPU, the rank-p2p kernel protocol (fused peer stores + flags in peer
 * memory) over NCCL 2.28 symmetric memory instead of CUDA IPC (SURVEY §8(f) row f4's NCCL
 * device API): the planes and the flag area are allocated with ncclMemAlloc and registered as
 * symmetric windows (ncclCommWindowRegister, NCCL_WIN_COLL_SYMMETRIC), and the neighbours'
 * addresses come from ncclGetLsaPointer on the device.  Arguments as ising_create_rank (the
 * NCCL unique id from rank 0; world == 1: nccl_id may be NULL; ISING_SELF_EXCHANGE=1 as for
 * rank-p2p).  Every rank must be in the others' load/store-accessible (LSA) team — one
 * NVLink domain — else NCCL error.  world <= 8.  Collective: create and destroy. */
int ising_create_rank_lsa(ising_t* out, int64_t L_rows, int64_t L_cols, uint64_t seed, int rank,
                          int world, int device, const void* nccl_id, size_t id_len);

/* Connect the n rank-p2p handles of one lattice that live in THIS process (handles[r] =
 * rank r, all created with world = n) through their device pointers instead of CUDA IPC:
 * one process drives every rank, one host thread per handle (calls on different handles may
 * run concurrently; each handle alone stays single-threaded).  Devices may differ (peer
 * access is enabled between neighbours; DEVICE if unavailable) or repeat — then the ranks'
 * kernels run concurrently on one GPU, each on its own stream, and the flag protocol is
 * exercised under real concurrency (the multi-process same-GPU runs are time-sliced).
 * Sweeps, observables, init and write are collective across the n handles exactly as across
 * processes; destroy them together, after their last collective call.  Ranks that share a
 * device run without programmatic dependent launch (waiting dependent grids would otherwise
 * hold the SM slots a spinning neighbour waits for); with widths that are not a multiple of
 * 8192 columns (register-rolling kernel: every block waits for the neighbours) keep such
 * groups small enough that one rank's grid does not fill the device.
 * Errors: ARG (NULL, n outside 1..8, handles not ranks 0..n-1 of one lattice), DEVICE, CUDA. */
int ising_p2p_connect_local(const ising_t* handles, int n);

/* The paper's basic layout (§3.1, Fig. 2 listing) on one
 * device: one signed byte per spin in two colour planes, one Philox block per four sites,
 * same draw contract and thresholds (bit-identical results), 3 algorithmic bytes per
 * attempted flip instead of 1.5.  L_rows even, L_cols % 8 == 0, L_rows <= 2^32, L_cols <= 2^35.
 * Every other call works
 * on the handle as on a one-slab multi-spin handle. */
int ising_create_basic(ising_t* out, int64_t L_rows, int64_t L_cols, uint64_t seed, int device);

/* Writes an NCCL unique id (id_len >= 128 bytes) into id. */
int ising_nccl_unique_id(void* id, size_t id_len);

/* Releases all device memory, streams and communicators.  NULL is a no-op. */
int ising_destroy(ising_t h);

/* --------------------------------------------------------------- parameters */

/* beta = J/T in [0, +inf]; NaN or negative -> ARG.  Computes the integer
 * thresholds on the host (R5). */
int ising_set_beta(ising_t h, double beta);

/* ISING_RULE_METROPOLIS (default) or ISING_RULE_HEATBATH; takes effect at the
 * next set_beta.  Other values -> ARG. */
int ising_set_rule(ising_t h, int rule);

/* ------------------------------------------------------------------- state */

/* Random start: spin = +1 iff r(seed, t=0, c, i, j) < 2^31 (R8).  Sets t := 0. */
int ising_init_random(ising_t h);

/* Cold start: all spins +1.  Sets t := 0. */
int ising_init_cold(ising_t h);

/* Load a full lattice from host memory: in[i*L_cols + J] in {-1, +1}, row-major,
 * in_len >= L_rows*L_cols (else RANGE); any other value -> ARG.  Sets the sweep
 * counter to t (the next sweep is t+1) — with the counter-based draws this is an
 * exact resume (checkpoint/restart).  Rank mode (world > 1): either
 * the full lattice (every rank keeps its own rows and halo rows) or exactly this rank's
 * R x L_cols rows (in_len == R*L_cols; the halo rows are then exchanged on the device).
 * Collective in rank mode. */
int ising_write_lattice(ising_t h, const int8_t* in, int64_t in_len, uint64_t t);

/* The same two calls in the bit-packed host format: spin (i, J) is bit (J & 7) of byte
 * (i*L_cols + J) / 8, 1 for +1 (row-major, least significant bit first: numpy's
 * packbits(..., bitorder="little") of the +1 mask).  L_cols / 8 bytes per row, 8x less host
 * memory and PCIe traffic than the +-1 bytes (checkpoints of the 2^40-spin lattice: 128 GiB
 * instead of 1 TiB).  in_len / out_len >= L_rows*L_cols/8 (else RANGE); rank mode (world > 1)
 * also takes exactly this rank's R*L_cols/8 bytes, as for the byte format.  Every bit pattern
 * is a valid lattice.  Multi-spin handles only (ARG for ising_create_basic handles).
 * ising_write_lattice_bits is collective in rank mode. */
int ising_write_lattice_bits(ising_t h, const uint8_t* in, int64_t in_len, uint64_t t);
int ising_read_lattice_bits(ising_t h, uint8_t* out, int64_t out_len);

/* Run n >= 0 full sweeps (black then white), t += n.  STATE if set_beta or an
 * init/write has not happened; RANGE if t + n > 2^32 - 1.  Returns after
 * completion.  Collective in rank mode. */
int ising_sweep(ising_t h, int64_t n);

/* Unpack to host: out[i*L_cols + J] = spin (i, J) in {-1, +1}, row-major;
 * out_len >= L_rows*L_cols (else RANGE).  Rank mode (world > 1): only this rank's rows
 * are written — at their global offset, or at offset 0 when out_len == R*L_cols. */
int ising_read_lattice(ising_t h, int8_t* out, int64_t out_len);

/* Unpack global rows [row_begin, row_begin + nrows) to host: out[r*L_cols + J], r relative
 * to row_begin; out_len >= nrows*L_cols (else RANGE).  The rows must belong to this
 * process's slabs (rank mode: its own) — else ARG.  For lattices too large for one host
 * buffer (C4, C5) and for sampled checks. */
int ising_read_rows(ising_t h, int64_t row_begin, int64_t nrows, int8_t* out, int64_t out_len);

/* Integer observables of the whole lattice (Eq. 1):
 * *up_count = number of +1 spins; *bond_energy = -sum over the 2 N M torus bonds
 * of s s' (each bond once, R11), in [-2NM, 2NM].  STATE before an init.
 * Collective in rank mode (int64 all-reduce over NCCL). */
int ising_observables(ising_t h, int64_t* up_count, int64_t* bond_energy);

/* A measured chain (the Fig. 5 / Fig. 6 methodology): n_samples
 * times, run `every` sweeps and record the observables of the resulting state into
 * up_counts[k] / bond_energies[k] (caller-owned arrays of n_samples).  The samples are
 * reduced on the device into a device-side series and copied back once, so the chain
 * does not synchronise per sample.  t += n_samples * every.  Same errors as ising_sweep;
 * in rank mode every rank receives the global values. */
int ising_sweep_measure(ising_t h, int64_t n_samples, int64_t every, int64_t* up_counts,
                        int64_t* bond_energies);

/* Asynchronous measured chain: the same sweeps and fused observables as
 * ising_sweep_measure, but the call returns once the work and the device->host copy of the
 * results are enqueued on the handle's stream, so the host can enqueue the next chunk while
 * this one runs (the results land in a pinned buffer of the library).  up_counts /
 * bond_energies (n_samples entries each) stay owned by the caller, must stay valid, and are
 * written by ising_measure_wait(h, *ticket); the wait also sets
 * ising_last_sweep_ms to this call's device time.  At most 8 calls may be pending
 * (ISING_ERR_STATE beyond).  Rank-mode, multi-device and basic-layout handles run the
 * synchronous path (results final on return; the wait is then a no-op).  The sweep counter
 * advances at enqueue time, so calls compose with ising_sweep in stream order. */
int ising_sweep_measure_async(ising_t h, int64_t n_samples, int64_t every, int64_t* up_counts,
                              int64_t* bond_energies, int64_t* ticket);
int ising_measure_wait(ising_t h, int64_t ticket);

/* ------------------------------------------------------------ introspection */

/* CUDA-event time of the last ising_sweep on this process's devices (max over
 * devices), milliseconds. */
int ising_last_sweep_ms(ising_t h, double* device_ms);

/* Per-launch timing of the half-sweep kernels of the last ising_sweep when
 * profiling is enabled (ising_set_profiling(h, 1)): *kernel_ms = summed CUDA-event
 * duration of the half-sweep launches on the first device's stream, *launches = how
 * many (at most the first 4096 launches of the call are timed).  Profiling adds one
 * event pair per timed launch and disables graph replay. */
int ising_set_profiling(ising_t h, int enable);
int ising_kernel_stats(ising_t h, double* kernel_ms, int64_t* launches);

/* Current sweep counter t. */
int ising_get_sweep(ising_t h, uint64_t* t);

/* This process's slab: first global row and number of rows (all rows for
 * ising_create / ising_create_slabs handles). */
int ising_slab_info(ising_t h, int64_t* row0, int64_t* rows);

/* Thresholds the kernels use for the current beta and rule: T[k] for e = 2k - 4,
 * k = 0..4 (2^32 means "always").  Host-side; for tests and reports. */
int ising_thresholds(ising_t h, uint64_t T[5]);

/* Half-sweep kernel variant the next sweep runs (for tests and reports; the same numbering
 * for packed and ising_create_basic handles): 0 Metropolis (both thresholds < 2^32), 2 Metropolis with a threshold at 2^32,
 * 4 Metropolis draw-free (thresholds in {0, 2^32}: beta = 0 or inf); heat bath 3 / 5 / 6
 * (0 / 1 / 2 leading thresholds at 2^32, five compares per site), 7 (symmetric thresholds
 * T[0] + T[4] = T[1] + T[3] = 2^32 + 1 and T[2] = 2^31: two compares per site on |r|), 1 generic. */
int ising_kernel_variant(ising_t h, int* variant);

/* Number of kernel launches issued by this handle since creation. */
int ising_launch_count(ising_t h, int64_t* launches);

/* Diagnostic: Philox4x32-10-only draw throughput of CUDA device `device` (the same
 * device function the half-sweep uses, outputs XOR-folded), in draws per ns — the
 * measured ALU roofline of the path (every attempted flip consumes one draw). */
int ising_probe_philox(int device, double* draws_per_ns);

/* ----------------------------------------------------------- lattice batches
 * n independent L_rows x L_cols lattices on one device, each with its own seed and beta
 * (temperature scans and the Binder-cumulant analysis, PAPER.md:414-421,
 * run many small lattices, which one-lattice handles leave launch-bound).  One CTA per lattice
 * keeps both colour planes in shared memory for up to 4096 sweeps per launch (L_rows * L_cols
 * <= 409600, e.g. 640 x 640); larger lattices span a thread-block cluster of 2 to 16 CTAs
 * (the smallest that divides L_rows and fits (L_rows / C + 2) * L_cols / 2 bytes per CTA in
 * 200 KB — up to 2048 x 2048), halo rows moving through distributed shared memory.  Every
 * lattice follows exactly the contract of a one-lattice handle with the same seed and beta
 * (same draws, thresholds and update order): bit-identical results.  Limits: L_rows even,
 * L_cols % 64 == 0, L_cols <= 32768, a lattice that fits as above, 1 <= n <= 65535; else ARG.
 * The handle owns its device memory; calls synchronise before returning; not thread-safe. */
typedef struct ising_batch* ising_batch_t;
/* seeds: n values (lattice k draws with seeds[k]); device: CUDA device index. */
int ising_batch_create(ising_batch_t* out, int64_t L_rows, int64_t L_cols, int n_lattices,
                       const uint64_t* seeds, int device);
int ising_batch_destroy(ising_batch_t b);                 /* NULL is a no-op */
/* betas: n values (each as ising_set_beta: >= 0 or +inf, NaN -> ARG); rule:
 * ISING_RULE_METROPOLIS or ISING_RULE_HEATBATH for every lattice of the batch. */
int ising_batch_set_beta(ising_batch_t b, const double* betas, int rule);
int ising_batch_init_random(ising_batch_t b);             /* every lattice; t := 0 */
int ising_batch_init_cold(ising_batch_t b);
/* n >= 0 sweeps of every lattice; STATE / RANGE as ising_sweep. */
int ising_batch_sweep(ising_batch_t b, int64_t n);
/* n_samples x every sweeps; after every `every` sweeps each lattice's (up count, bond
 * energy) — as ising_observables — into up_counts / bond_energies[k * n_samples + s]
 * (n * n_samples entries each, caller-owned). */
int ising_batch_sweep_measure(ising_batch_t b, int64_t n_samples, int64_t every,
                              int64_t* up_counts, int64_t* bond_energies);
/* Current (up count, bond energy) of every lattice (n entries each); STATE before an init /
 * write. */
int ising_batch_observables(ising_batch_t b, int64_t* up_counts, int64_t* bond_energies);
/* Lattice `lattice` as +-1 bytes, row-major; out_len >= L_rows * L_cols (else RANGE); lattice
 * outside 0 .. n-1 -> ARG; STATE before an init / write. */
int ising_batch_read_lattice(ising_batch_t b, int lattice, int8_t* out, int64_t out_len);
/* Load lattice `lattice` from +-1 bytes (in_len >= L_rows * L_cols, else RANGE; other values
 * -> ARG) and set the batch's sweep counter to t (shared by all lattices: the next sweep is
 * t + 1) — checkpoint / exact resume of a batch, lattice by lattice.  Lattices never
 * initialised or written start cold. */
int ising_batch_write_lattice(ising_batch_t b, int lattice, const int8_t* in, int64_t in_len,
                              uint64_t t);
int ising_batch_last_sweep_ms(ising_batch_t b, double* device_ms);  /* last sweep call */
int ising_batch_get_sweep(ising_batch_t b, uint64_t* t);

const char* ising_strerror(int status);

/* Message of the last CUDA/NCCL error seen by this thread ("" if none). */
const char* ising_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* ISING_H */
