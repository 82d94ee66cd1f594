/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the MPDATA step (see
 * mpdata_oracle.h: provenance, scope, and "parity unpinned by the
 * reference"). Build: oracle/Makefile (-O3 -ffp-contract=off).
 */
#include "mpdata_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* Pinned constant of the MPDATA ratios. */
#define ORC_EPS 1e-15

double orc_eps(void) { return ORC_EPS; }

/* ---- counter-based seeded values (workload.hpp:61-63: pure function of
 * (seed, field, i, j, k)) ---- */
static uint64_t orc_splitmix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static double orc_uniform(uint64_t seed, uint64_t field, uint64_t i, uint64_t j, uint64_t k) {
  uint64_t z = orc_splitmix(seed);
  z = orc_splitmix(z ^ field);
  z = orc_splitmix(z ^ i);
  z = orc_splitmix(z ^ j);
  z = orc_splitmix(z ^ k);
  return (double)(z >> 11) * 0x1.0p-53;
}

typedef struct {
  int recipe;
  int64_t n, m, l;
  uint64_t seed;
  double ci, cj, ck;            /* grid centre in index space */
  double ax, ay, az;            /* rotation axis (unit) */
  double sx, sy, sz;            /* per-axis Courant scale */
  int64_t c0[3], c1[3];         /* cube [c0, c1) per axis */
} OrcRecipe;

static int orc_recipe_setup(OrcRecipe* r, int recipe, int64_t n, int64_t m, int64_t l,
                            uint64_t seed) {
  memset(r, 0, sizeof(*r));
  if (recipe < 0 || recipe > 2 || n < 1 || m < 1 || l < 1) return 1;
  r->recipe = recipe;
  r->n = n; r->m = m; r->l = l; r->seed = seed;
  r->ci = (double)(n - 1) / 2.0;
  r->cj = (double)(m - 1) / 2.0;
  r->ck = (double)(l - 1) / 2.0;
  if (recipe == 2) {
    /* Solid-body rotation about a seeded axis; max |C| = 0.3 per axis. */
    double a0 = 2.0 * orc_uniform(seed, 7, 0, 0, 0) - 1.0;
    double a1 = 2.0 * orc_uniform(seed, 7, 1, 0, 0) - 1.0;
    double a2 = 2.0 * orc_uniform(seed, 7, 2, 0, 0) - 1.0;
    double nrm = sqrt((a0 * a0 + a1 * a1) + a2 * a2);
    r->ax = a0 / nrm; r->ay = a1 / nrm; r->az = a2 / nrm;
    double dx = fabs(r->ay) * r->ck + fabs(r->az) * r->cj;
    double dy = fabs(r->az) * r->ci + fabs(r->ax) * r->ck;
    double dz = fabs(r->ax) * r->cj + fabs(r->ay) * r->ci;
    r->sx = dx > 0.0 ? 0.3 / dx : 0.0;
    r->sy = dy > 0.0 ? 0.3 / dy : 0.0;
    r->sz = dz > 0.0 ? 0.3 / dz : 0.0;
    /* 32^3 cube at C2's 256x256x64, scaled per axis to this grid. */
    int64_t ext[3] = {n, m, l}, ref[3] = {256, 256, 64};
    for (int a = 0; a < 3; ++a) {
      int64_t e = (32 * ext[a]) / ref[a];
      if (e < 1) e = 1;
      if (e > ext[a]) e = ext[a];
      r->c0[a] = (ext[a] - e) / 2;
      r->c1[a] = r->c0[a] + e;
    }
  }
  return 0;
}

/* vals = {x, u, v, w, h} at global cell (i, j, k). */
static void orc_recipe_cell(const OrcRecipe* r, int64_t i, int64_t j, int64_t k, double* vals) {
  uint64_t s = r->seed;
  uint64_t I = (uint64_t)i, J = (uint64_t)j, K = (uint64_t)k;
  if (r->recipe == 0) {
    vals[0] = 1.0 + orc_uniform(s, 0, I, J, K);
    vals[1] = -0.25 + 0.5 * orc_uniform(s, 1, I, J, K);
    vals[2] = -0.25 + 0.5 * orc_uniform(s, 2, I, J, K);
    vals[3] = -0.25 + 0.5 * orc_uniform(s, 3, I, J, K);
    vals[4] = 0.9 + 0.2 * orc_uniform(s, 4, I, J, K);
  } else if (r->recipe == 1) {
    double di = (double)i - r->ci, dj = (double)j - r->cj, dk = (double)k - r->ck;
    double r2 = (di * di + dj * dj) + dk * dk;
    double g = exp(-r2 / 128.0); /* sigma = 8 cells: 2 sigma^2 = 128 */
    vals[0] = (1.5 + 0.5 * g) + 0.01 * orc_uniform(s, 0, I, J, K);
    vals[1] = -0.25 + 0.5 * orc_uniform(s, 1, I, J, K);
    vals[2] = -0.25 + 0.5 * orc_uniform(s, 2, I, J, K);
    vals[3] = -0.25 + 0.5 * orc_uniform(s, 3, I, J, K);
    vals[4] = 1.0;
  } else {
    int in_cube = i >= r->c0[0] && i < r->c1[0] && j >= r->c0[1] && j < r->c1[1] &&
                  k >= r->c0[2] && k < r->c1[2];
    vals[0] = in_cube ? 3.0 : 1.0 + orc_uniform(s, 0, I, J, K);
    double di = (double)i - r->ci, dj = (double)j - r->cj, dk = (double)k - r->ck;
    vals[1] = r->sx * (r->ay * dk - r->az * dj);
    vals[2] = r->sy * (r->az * di - r->ax * dk);
    vals[3] = r->sz * (r->ax * dj - r->ay * di);
    vals[4] = 0.9 + 0.2 * orc_uniform(s, 4, I, J, K);
  }
}

#define REAL double
#define SFX f64
#include "mpdata_oracle_step.inc"
#undef REAL
#undef SFX

#define REAL float
#define SFX f32
#include "mpdata_oracle_step.inc"
#undef REAL
#undef SFX

/* ---- reference surrogate stage ops on the padded GridField layout ---- */
#define PIX(i, j, k) \
  ((size_t)((((i) + halo) * (m + 2 * halo) + ((j) + halo)) * (l + 2 * halo) + ((k) + halo)))

static int64_t orc_clamp(int64_t a, int64_t lo, int64_t hi) { return a < lo ? lo : a > hi ? hi : a; }

void orc_fill_halo_clamped(double* f, int64_t n, int64_t m, int64_t l, int64_t halo) {
  for (int64_t i = -halo; i < n + halo; ++i)
    for (int64_t j = -halo; j < m + halo; ++j)
      for (int64_t k = -halo; k < l + halo; ++k) {
        int interior = i >= 0 && i < n && j >= 0 && j < m && k >= 0 && k < l;
        if (interior) continue;
        f[PIX(i, j, k)] = f[PIX(orc_clamp(i, 0, n - 1), orc_clamp(j, 0, m - 1), orc_clamp(k, 0, l - 1))];
      }
}

static void orc_stage7(const double* in, double* out, int64_t n, int64_t m, int64_t l,
                       int64_t halo, int is_max) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < m; ++j)
      for (int64_t k = 0; k < l; ++k) {
        double nb[7] = {in[PIX(i, j, k)],     in[PIX(i - 1, j, k)], in[PIX(i + 1, j, k)],
                        in[PIX(i, j - 1, k)], in[PIX(i, j + 1, k)], in[PIX(i, j, k - 1)],
                        in[PIX(i, j, k + 1)]};
        double r = nb[0];
        for (int q = 1; q < 7; ++q) r = is_max ? (nb[q] > r ? nb[q] : r) : (nb[q] < r ? nb[q] : r);
        out[PIX(i, j, k)] = r;
      }
}

void orc_stage_max7(const double* in, double* out, int64_t n, int64_t m, int64_t l, int64_t halo) {
  orc_stage7(in, out, n, m, l, halo, 1);
}
void orc_stage_min7(const double* in, double* out, int64_t n, int64_t m, int64_t l, int64_t halo) {
  orc_stage7(in, out, n, m, l, halo, 0);
}
