// Seeded field recipes of the BASELINE configs, shared by the host
// (imb::init_fields) and the device init kernel. Every value is a pure
// function of (seed, field, global i, j, k) — the contract of
// /root/reference/proj/include/imbalance/workload.hpp:61-63 — so a slab of
// any decomposition regenerates bit-identical values, halos included.
//
// Compiled WITHOUT floating-point contraction on both sides (host:
// -ffp-contract=off, device: --fmad=false) so the non-transcendental
// recipes are bit-identical between CPU and GPU. The Gaussian recipe calls
// exp(), which may differ by an ulp between libm and CUDA; parity tests
// therefore upload host-generated fields for it.
#pragma once

#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define IMB_HD __host__ __device__ __forceinline__
#else
#define IMB_HD inline
#endif

namespace imb::recipe {

enum Kind : int { kUniform = 0, kGauss = 1, kRotCube = 2 };

IMB_HD std::uint64_t mix64(std::uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Uniform double in [0, 1) with 53 random bits, keyed by (seed, field, i, j, k).
IMB_HD double unit(std::uint64_t seed, std::uint64_t field, std::uint64_t i, std::uint64_t j,
                   std::uint64_t k) {
  std::uint64_t z = mix64(seed);
  z = mix64(z ^ field);
  z = mix64(z ^ i);
  z = mix64(z ^ j);
  z = mix64(z ^ k);
  return static_cast<double>(z >> 11) * (1.0 / 9007199254740992.0);
}

// Grid-level constants of a recipe, computed once on the host.
struct Params {
  int kind = kRotCube;
  std::int64_t n = 0, m = 0, l = 0;
  std::uint64_t seed = 42;
  double ci = 0, cj = 0, ck = 0;  // centre in index space
  double ax = 0, ay = 0, az = 0;  // unit rotation axis
  double sx = 0, sy = 0, sz = 0;  // Courant scale per axis (max |C| = 0.3)
  std::int64_t lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};  // step-discontinuity cube
};

inline Params make_params(int kind, std::int64_t n, std::int64_t m, std::int64_t l,
                          std::uint64_t seed) {
  Params p;
  p.kind = kind;
  p.n = n;
  p.m = m;
  p.l = l;
  p.seed = seed;
  p.ci = static_cast<double>(n - 1) / 2.0;
  p.cj = static_cast<double>(m - 1) / 2.0;
  p.ck = static_cast<double>(l - 1) / 2.0;
  if (kind == kRotCube) {
    const double a0 = 2.0 * unit(seed, 7, 0, 0, 0) - 1.0;
    const double a1 = 2.0 * unit(seed, 7, 1, 0, 0) - 1.0;
    const double a2 = 2.0 * unit(seed, 7, 2, 0, 0) - 1.0;
    const double len = std::sqrt((a0 * a0 + a1 * a1) + a2 * a2);
    p.ax = a0 / len;
    p.ay = a1 / len;
    p.az = a2 / len;
    const double reach_x = std::fabs(p.ay) * p.ck + std::fabs(p.az) * p.cj;
    const double reach_y = std::fabs(p.az) * p.ci + std::fabs(p.ax) * p.ck;
    const double reach_z = std::fabs(p.ax) * p.cj + std::fabs(p.ay) * p.ci;
    p.sx = reach_x > 0.0 ? 0.3 / reach_x : 0.0;
    p.sy = reach_y > 0.0 ? 0.3 / reach_y : 0.0;
    p.sz = reach_z > 0.0 ? 0.3 / reach_z : 0.0;
    // The 32^3 cube of config 2 (256x256x64), scaled per axis to this grid.
    const std::int64_t ext[3] = {n, m, l}, base[3] = {256, 256, 64};
    for (int a = 0; a < 3; ++a) {
      std::int64_t e = (32 * ext[a]) / base[a];
      e = e < 1 ? 1 : (e > ext[a] ? ext[a] : e);
      p.lo[a] = (ext[a] - e) / 2;
      p.hi[a] = p.lo[a] + e;
    }
  }
  return p;
}

// out = {x, u, v, w, h} at global cell (i, j, k), each index in [0, extent).
IMB_HD void cell(const Params& p, std::int64_t i, std::int64_t j, std::int64_t k, double* out) {
  const std::uint64_t s = p.seed, I = static_cast<std::uint64_t>(i),
                      J = static_cast<std::uint64_t>(j), K = static_cast<std::uint64_t>(k);
  if (p.kind == kRotCube) {
    const bool cube = i >= p.lo[0] && i < p.hi[0] && j >= p.lo[1] && j < p.hi[1] &&
                      k >= p.lo[2] && k < p.hi[2];
    out[0] = cube ? 3.0 : 1.0 + unit(s, 0, I, J, K);
    const double di = static_cast<double>(i) - p.ci;
    const double dj = static_cast<double>(j) - p.cj;
    const double dk = static_cast<double>(k) - p.ck;
    // Face velocities of the rigid rotation a x (r - c): u depends on (j,k)
    // only, v on (i,k), w on (i,j) -> discretely divergence-free.
    out[1] = p.sx * (p.ay * dk - p.az * dj);
    out[2] = p.sy * (p.az * di - p.ax * dk);
    out[3] = p.sz * (p.ax * dj - p.ay * di);
    out[4] = 0.9 + 0.2 * unit(s, 4, I, J, K);
    return;
  }
  if (p.kind == kGauss) {
    const double di = static_cast<double>(i) - p.ci;
    const double dj = static_cast<double>(j) - p.cj;
    const double dk = static_cast<double>(k) - p.ck;
    const double r2 = (di * di + dj * dj) + dk * dk;
    out[0] = (1.5 + 0.5 * exp(-r2 / 128.0)) + 0.01 * unit(s, 0, I, J, K);
    out[4] = 1.0;
  } else {
    out[0] = 1.0 + unit(s, 0, I, J, K);
    out[4] = 0.9 + 0.2 * unit(s, 4, I, J, K);
  }
  out[1] = -0.25 + 0.5 * unit(s, 1, I, J, K);
  out[2] = -0.25 + 0.5 * unit(s, 2, I, J, K);
  out[3] = -0.25 + 0.5 * unit(s, 3, I, J, K);
}

}  // namespace imb::recipe
