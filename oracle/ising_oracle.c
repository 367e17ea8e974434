/*
 * oracle/ising_oracle.c — CPU ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library.  The product path
 * (paper_1906_06297_b200/) never links, imports or executes anything here, and
 * this file includes nothing from the product (no shared headers, helpers,
 * tables or constants).
 *
 * What it computes: the checkerboard Metropolis sweep of the 2D ferromagnetic
 * Ising model with periodic boundaries, exactly as PAPER.md describes it, in
 * the plainest form:
 *   - one signed byte (+1/-1) per spin, two colour planes of nx x ny = N x M/2
 *     "each containing one color of spins compacted along the rows"
 *     (§3.1; Fig. 1 centre);
 *   - the per-spin stencil of the Fig. 2 CUDA C listing `update_lattice`
 *     (§3.1), with the `%` operators that LaTeX ate restored
 *     (reading R2);
 *   - Metropolis acceptance "accepted with probability e^(-beta dE)"
 *     (§2) as the listing writes it, rand < exp(-2 beta nn lij)
 *     (PAPER.md:155-156), with rand = r * 2^-32 for a uint32 Philox draw r,
 *     which is the same predicate as r < ceil(2^32 exp(-2 beta e)) (reading R5);
 *   - heat-bath acceptance P = e^(-beta dE)/(e^(-beta dE)+1) (§2);
 *   - Philox4x32-10 (§3.2, §3.3), written from the
 *     generator's published round function, keyed statelessly on
 *     (seed, sweep, colour, site) (reading R6, the analogue of the paper's
 *     curand_init(seed, sequence, offset) addressing);
 *   - observables straight from Eq. 1 (§2): the up-spin count
 *     and E = -sum over the 2NM torus bonds of s s' (reading R11).
 *
 * No blocking, packing, fusion or reordering: every site is visited in the
 * listing's tid order.  The only parallelism is an OpenMP split of the rows of
 * one colour phase, which cannot change the result because sites of one colour
 * read only the other colour (§2).
 *
 * Parity status: pinned (tests/test_oracle_*.py): Philox by the Random123
 * known-answer vectors; thresholds by closed forms at beta_c; the stencil by the
 * Fig. 3 caption's worked example and a brute-force torus
 * stencil; the update rule by beta = 0 / beta = inf special cases and a
 * brute-force full-lattice sweep; the chain by exact 4x4 enumeration and
 * Onsager.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- Philox */
/* Philox4x32-10: Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy
 * as 1, 2, 3" (SC'11).  Round: (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2;
 * c <- {hi1^c1^k0, lo1, hi0^c3^k1, lo0}; key bumped by (W0, W1) between rounds. */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += W0;
      k1 += W1;
    }
    uint64_t p0 = (uint64_t)M0 * (uint64_t)c0;
    uint64_t p1 = (uint64_t)M1 * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

/* The draw for plane site (i, j) of colour c in sweep t (t = 0: initialisation).
 * Reading R6: counter {t, j/4, c, i}, key {lo32(seed), hi32(seed)}, word j%4. */
uint32_t oracle_rand(uint64_t seed, uint32_t t, uint32_t c, uint32_t i, uint64_t j) {
  uint32_t ctr[4] = {t, (uint32_t)(j / 4), c, i};
  uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
  uint32_t out[4];
  oracle_philox4x32_10(ctr, key, out);
  return out[j % 4];
}

/* ------------------------------------------------------------ thresholds */
#define RULE_METROPOLIS 0
#define RULE_HEATBATH 1

/* Metropolis: accept with probability p = exp(-beta dE), dE = 2 e (J = 1, e = s*h,
 * reading R3).  u = r 2^-32 < p  <=>  r < ceil(2^32 p); capped at 2^32 ("always").
 * T[k] for e = 2k - 4, k = 0..4; for e <= 0 p >= 1 so T = 2^32. */
static uint64_t ceil_scaled(double p) {
  if (!(p > 0.0)) return 0;                          /* p == 0 (or NaN guard) */
  if (p >= 1.0) return (uint64_t)1 << 32;
  double x = ceil(ldexp(p, 32));                     /* ldexp is exact */
  if (x >= 4294967296.0) return (uint64_t)1 << 32;
  return (uint64_t)x;
}

void oracle_thresholds(double beta, int rule, uint64_t T[5]) {
  for (int k = 0; k < 5; ++k) {
    int e = 2 * k - 4;
    double P;
    if (rule == RULE_METROPOLIS) {
      if (e <= 0) {
        P = 1.0;
      } else if (isinf(beta)) {
        P = 0.0;
      } else {
        P = exp(-2.0 * beta * (double)e);
      }
    } else {                                         /* heat bath */
      if (isinf(beta)) {
        P = (e < 0) ? 1.0 : (e == 0 ? 0.5 : 0.0);
      } else {
        double p = exp(-2.0 * beta * (double)e);
        P = isinf(p) ? 1.0 : p / (p + 1.0);
      }
    }
    T[k] = ceil_scaled(P);
  }
}

/* ------------------------------------------------------------ the stencil */
/* Fig. 2 listing, restored:  j = tid % ny;
 * black: joff = (i % 2) ? jpp : jnn;  white: joff = (i % 2) ? jnn : jpp.
 * Returns nn_sum, the sum of the four opposite-colour neighbours of plane site
 * (i, j) of the target colour. */
int oracle_nn_sum(const int8_t* op_lattice, int is_black, int64_t nx, int64_t ny, int64_t i,
                  int64_t j) {
  int64_t ipp = (i + 1 < nx) ? i + 1 : 0;
  int64_t inn = (i - 1 >= 0) ? i - 1 : nx - 1;
  int64_t jpp = (j + 1 < ny) ? j + 1 : 0;
  int64_t jnn = (j - 1 >= 0) ? j - 1 : ny - 1;
  int64_t joff;
  if (is_black) {
    joff = (i % 2) ? jpp : jnn;
  } else {
    joff = (i % 2) ? jnn : jpp;
  }
  return op_lattice[inn * ny + j] + op_lattice[i * ny + j] + op_lattice[ipp * ny + j] +
         op_lattice[i * ny + joff];
}

/* One colour phase: the body of update_lattice<is_black> for every tid
 * (PAPER.md:121-159), with the float compare replaced by the integer one
 * (reading R5).  t is the sweep index (>= 1), colour c = is_black ? 0 : 1. */
void oracle_update_lattice(int8_t* lattice, const int8_t* op_lattice, int is_black, int64_t nx,
                           int64_t ny, uint64_t seed, uint32_t t, const uint64_t T[5], int rule) {
  const uint32_t colour = is_black ? 0u : 1u;
#pragma omp parallel for schedule(static) if (nx * ny >= 65536)
  for (int64_t i = 0; i < nx; ++i) {
    for (int64_t j = 0; j < ny; ++j) {
      int nn_sum = oracle_nn_sum(op_lattice, is_black, nx, ny, i, j);
      int8_t lij = lattice[i * ny + j];
      int e = nn_sum * lij;                          /* dE = 2 J e */
      uint32_t r = oracle_rand(seed, t, colour, (uint32_t)i, (uint64_t)j);
      int flip;
      if (rule == RULE_METROPOLIS)
        flip = (e <= 0) || ((uint64_t)r < T[(e + 4) / 2]);
      else
        flip = (uint64_t)r < T[(e + 4) / 2];
      if (flip) lattice[i * ny + j] = (int8_t)(-lij);
    }
  }
}

/* The same phase for one horizontal slab of a lattice split across GPUs
 * (§4: "partitioned into horizontal slabs ... each GPU needs only read
 * access to the memory of the two GPUs that handle the slabs on top and bottom").
 * lattice / op_lattice hold the slab's nrows rows (global rows row0 .. row0+nrows-1)
 * of the target / source colour; op_above / op_below are the source rows of the
 * neighbouring slabs (global rows row0-1 and row0+nrows, mod N).  Identical to
 * oracle_update_lattice except that the listing's inn / ipp rows at the slab edge
 * come from the neighbours, and parity and the draw use the global row (R19). */
void oracle_update_slab(int8_t* lattice, const int8_t* op_lattice, const int8_t* op_above,
                        const int8_t* op_below, int is_black, int64_t row0, int64_t nrows,
                        int64_t ny, uint64_t seed, uint32_t t, const uint64_t T[5], int rule) {
  const uint32_t colour = is_black ? 0u : 1u;
  for (int64_t i = 0; i < nrows; ++i) {
    const int64_t gi = row0 + i;
    const int8_t* up = (i == 0) ? op_above : op_lattice + (i - 1) * ny;
    const int8_t* dn = (i == nrows - 1) ? op_below : op_lattice + (i + 1) * ny;
    const int8_t* me = op_lattice + i * ny;
    for (int64_t j = 0; j < ny; ++j) {
      int64_t jpp = (j + 1 < ny) ? j + 1 : 0;
      int64_t jnn = (j - 1 >= 0) ? j - 1 : ny - 1;
      int64_t joff;
      if (is_black) {
        joff = (gi % 2) ? jpp : jnn;
      } else {
        joff = (gi % 2) ? jnn : jpp;
      }
      int nn_sum = up[j] + me[j] + dn[j] + me[joff];
      int8_t lij = lattice[i * ny + j];
      int e = nn_sum * lij;
      uint32_t r = oracle_rand(seed, t, colour, (uint32_t)gi, (uint64_t)j);
      int flip;
      if (rule == RULE_METROPOLIS)
        flip = (e <= 0) || ((uint64_t)r < T[(e + 4) / 2]);
      else
        flip = (uint64_t)r < T[(e + 4) / 2];
      if (flip) lattice[i * ny + j] = (int8_t)(-lij);
    }
  }
}

/* Sweeps t0+1 .. t0+nsweeps; each is black then white (reading R7). */
void oracle_sweep(int8_t* black, int8_t* white, int64_t nx, int64_t ny, uint64_t seed, uint32_t t0,
                  int64_t nsweeps, double beta, int rule) {
  uint64_t T[5];
  oracle_thresholds(beta, rule, T);
  for (int64_t s = 1; s <= nsweeps; ++s) {
    uint32_t t = (uint32_t)(t0 + s);
    oracle_update_lattice(black, white, 1, nx, ny, seed, t, T, rule);
    oracle_update_lattice(white, black, 0, nx, ny, seed, t, T, rule);
  }
}

/* ------------------------------------------------------------------ init */
/* Reading R8: random start sigma = +1 iff r(seed, 0, c, i, j) < 2^31; cold: all +1. */
void oracle_init_random(int8_t* black, int8_t* white, int64_t nx, int64_t ny, uint64_t seed) {
  for (int c = 0; c < 2; ++c) {
    int8_t* plane = c == 0 ? black : white;
#pragma omp parallel for schedule(static) if (nx * ny >= 65536)
    for (int64_t i = 0; i < nx; ++i)
      for (int64_t j = 0; j < ny; ++j)
        plane[i * ny + j] = oracle_rand(seed, 0, (uint32_t)c, (uint32_t)i, (uint64_t)j) < 0x80000000u
                                ? (int8_t)1
                                : (int8_t)-1;
  }
}

void oracle_init_cold(int8_t* black, int8_t* white, int64_t nx, int64_t ny) {
  for (int64_t k = 0; k < nx * ny; ++k) {
    black[k] = 1;
    white[k] = 1;
  }
}

/* ------------------------------------------------------ full-lattice view */
/* Reading R1: site (i, J) is black iff (i + J) is even; its plane column is J/2. */
void oracle_full_lattice(const int8_t* black, const int8_t* white, int64_t nx, int64_t ny,
                         int8_t* out) {
  int64_t M = 2 * ny;
#pragma omp parallel for schedule(static) if (nx * ny >= 65536)
  for (int64_t i = 0; i < nx; ++i)
    for (int64_t J = 0; J < M; ++J)
      out[i * M + J] = ((i + J) % 2 == 0) ? black[i * ny + J / 2] : white[i * ny + J / 2];
}

void oracle_from_full(const int8_t* full, int8_t* black, int8_t* white, int64_t nx, int64_t ny) {
  int64_t M = 2 * ny;
  for (int64_t i = 0; i < nx; ++i)
    for (int64_t J = 0; J < M; ++J) {
      if ((i + J) % 2 == 0)
        black[i * ny + J / 2] = full[i * M + J];
      else
        white[i * ny + J / 2] = full[i * M + J];
    }
}

/* ----------------------------------------------------------- observables */
/* Eq. 1 with J = 1, each nearest-neighbour bond of the torus
 * once (reading R11): the right and the down bond of every site. */
void oracle_observables(const int8_t* black, const int8_t* white, int64_t nx, int64_t ny,
                        int64_t* up, int64_t* energy) {
  int64_t M = 2 * ny;
  int64_t u = 0, E = 0;
#pragma omp parallel for schedule(static) reduction(+ : u, E) if (nx * ny >= 65536)
  for (int64_t i = 0; i < nx; ++i) {
    for (int64_t J = 0; J < M; ++J) {
      int64_t ir = i, Jr = (J + 1) % M, id = (i + 1) % nx, Jd = J;
      int s = ((i + J) % 2 == 0) ? black[i * ny + J / 2] : white[i * ny + J / 2];
      int sr = ((ir + Jr) % 2 == 0) ? black[ir * ny + Jr / 2] : white[ir * ny + Jr / 2];
      int sd = ((id + Jd) % 2 == 0) ? black[id * ny + Jd / 2] : white[id * ny + Jd / 2];
      if (s == 1) ++u;
      E -= s * sr + s * sd;
    }
  }
  *up = u;
  *energy = E;
}

/* A measured chain: after each of nsweeps sweeps record (up, E).  Driver loop
 * for the statistical pins (no arithmetic of its own). */
void oracle_chain(int8_t* black, int8_t* white, int64_t nx, int64_t ny, uint64_t seed, uint32_t t0,
                  int64_t nsweeps, double beta, int rule, int64_t* ups, int64_t* energies) {
  for (int64_t s = 0; s < nsweeps; ++s) {
    oracle_sweep(black, white, nx, ny, seed, (uint32_t)(t0 + s), 1, beta, rule);
    oracle_observables(black, white, nx, ny, &ups[s], &energies[s]);
  }
}

/* --------------------------------------------------- sampled single sites */
/* Value of full-lattice site (i, J) of an N x M torus after sweep 1 from the random start,
 * evaluated site by site without materialising the lattice (for lattices too large for
 * this oracle, BASELINE configs C4 / C5).  The black phase of sweep 1 reads the four white
 * neighbours at t = 0; the white phase reads the four black neighbours after the black
 * phase.  Same stencil (readings R1-R2) and acceptance (R5) as
 * oracle_update_lattice, same draws (R6, R8). */
static int init_spin(uint64_t seed, int c, int64_t i, int64_t j) {
  return oracle_rand(seed, 0, (uint32_t)c, (uint32_t)i, (uint64_t)j) < 0x80000000u ? 1 : -1;
}

static int accept(int rule, int e, uint32_t r, const uint64_t T[5]) {
  if (rule == RULE_METROPOLIS) return (e <= 0) || ((uint64_t)r < T[(e + 4) / 2]);
  return (uint64_t)r < T[(e + 4) / 2];
}

static int black_after_phase1(uint64_t seed, int64_t nx, int64_t ny, const uint64_t T[5], int rule,
                              int64_t i, int64_t j) {
  int64_t ipp = (i + 1 < nx) ? i + 1 : 0, inn = (i - 1 >= 0) ? i - 1 : nx - 1;
  int64_t jpp = (j + 1 < ny) ? j + 1 : 0, jnn = (j - 1 >= 0) ? j - 1 : ny - 1;
  int64_t joff = (i % 2) ? jpp : jnn;  /* black target */
  int nn = init_spin(seed, 1, inn, j) + init_spin(seed, 1, i, j) + init_spin(seed, 1, ipp, j) +
           init_spin(seed, 1, i, joff);
  int s = init_spin(seed, 0, i, j);
  return accept(rule, nn * s, oracle_rand(seed, 1, 0, (uint32_t)i, (uint64_t)j), T) ? -s : s;
}

int oracle_sample_after_one_sweep(uint64_t seed, int64_t N, int64_t M, double beta, int rule,
                                  int64_t i, int64_t J) {
  uint64_t T[5];
  oracle_thresholds(beta, rule, T);
  int64_t nx = N, ny = M / 2, j = J / 2;
  if ((i + J) % 2 == 0) return black_after_phase1(seed, nx, ny, T, rule, i, j);
  int64_t ipp = (i + 1 < nx) ? i + 1 : 0, inn = (i - 1 >= 0) ? i - 1 : nx - 1;
  int64_t jpp = (j + 1 < ny) ? j + 1 : 0, jnn = (j - 1 >= 0) ? j - 1 : ny - 1;
  int64_t joff = (i % 2) ? jnn : jpp;  /* white target */
  int nn = black_after_phase1(seed, nx, ny, T, rule, inn, j) +
           black_after_phase1(seed, nx, ny, T, rule, i, j) +
           black_after_phase1(seed, nx, ny, T, rule, ipp, j) +
           black_after_phase1(seed, nx, ny, T, rule, i, joff);
  int s = init_spin(seed, 1, i, j);
  return accept(rule, nn * s, oracle_rand(seed, 1, 1, (uint32_t)i, (uint64_t)j), T) ? -s : s;
}

/* Row i of the full lattice after sweep 1 (out: M bytes), site by site (OpenMP over J). */
void oracle_sample_row_after_one_sweep(uint64_t seed, int64_t N, int64_t M, double beta, int rule,
                                       int64_t i, int8_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t J = 0; J < M; ++J)
    out[J] = (int8_t)oracle_sample_after_one_sweep(seed, N, M, beta, rule, i, J);
}

/* ------------------------------------------------------------- threading */
void oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int oracle_get_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
