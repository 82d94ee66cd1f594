// Fused streaming MPDATA step (IORD = 2, optional nonoscillatory limiter):
// one kernel reads psi^n, u, v, w, h and writes psi^{n+1}; every
// intermediate (psi^(1), pseudo-velocities, beta bounds, limited velocities,
// fluxes) lives in shared memory or registers.
//
// Geometry (B200-first):
//  * A warp owns whole rows: each lane holds KPT = l/32 CONSECUTIVE k values
//    of a row (l in {32, 64, 128}), so every global/shared access is a
//    16/32-byte vector per lane and a warp moves a whole contiguous row; the
//    k +- 1 neighbours are in-register or one warp shuffle away, with the
//    periodic k wrap closing inside the warp (no k halo, no k-neighbour loads).
//  * A block owns a j-tile of TJ output rows plus a recomputed halo of 2 rows
//    (limiter) or 1 row (plain) on each side: RR = NW*RW region rows.
//  * The block streams along i (the slab axis) over a segment of planes. The
//    stages run one plane apart, so along i nothing is recomputed except a
//    two-plane warm-up per segment. Shared memory holds 3 planes of psi^(1),
//    2 of the y/z pseudo-velocities and 2 of each beta; same-column
//    dependencies along i (x-face velocity, x-flux, the psi^n star extrema)
//    are register carries.
//  * Divisions: fp64 folds the four divisions of a pseudo-velocity into one
//    reciprocal of hb*dA*dB*dC and the two beta divisions into one, with a
//    MUFU seed + 2 Newton steps; fp32 uses MUFU.RCP. Both stay inside the
//    parity tolerance (1e-12 / 1e-5).
// The per-cell arithmetic follows SURVEY.md Appendix A (see mpdata_math.cuh).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>

#include "mpdata_kernels.cuh"
#include "mpdata_math.cuh"

namespace imb::dev {

namespace {

constexpr unsigned kFull = 0xffffffffu;

template <class T, int L, int RW, int NW, bool NONOS>
struct Cfg {
  static constexpr int KPT = L / 32;              // consecutive k per lane
  static constexpr int RR = NW * RW;              // region rows
  static constexpr int HALO = NONOS ? 2 : 1;      // recomputed rows on each side
  static constexpr int TJ = RR - 2 * HALO;        // output rows per tile
  static constexpr int NT = NW * 32;
  static constexpr int PLANE = RR * L;            // cells of one smem plane
  static constexpr int NSLOT = NONOS ? 11 : 5;
  static constexpr std::size_t SMEM = sizeof(T) * PLANE * NSLOT;
};

template <class T>
struct Args {
  const T* __restrict__ x;
  const T* __restrict__ u;
  const T* __restrict__ v;
  const T* __restrict__ w;
  const T* __restrict__ h;
  T* __restrict__ out;
  int m;            // rows (j extent)
  int R;            // halo planes of the padded slab
  int ntj;          // j tiles
  int nseg;         // i segments
  int o0, o1;       // output plane range (interior coordinates)
  long long plane;  // m * l
};

// ---- per-lane vectors of K consecutive k values ---------------------------
template <class T, int K>
struct Vec {
  T e[K];
};

template <class T, int K>
__device__ __forceinline__ Vec<T, K> vload(const T* p) {  // global, read-only path
  Vec<T, K> r;
  if constexpr (sizeof(T) == 8 && K == 4) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    r.e[0] = a.x; r.e[1] = a.y; r.e[2] = b.x; r.e[3] = b.y;
  } else if constexpr (sizeof(T) == 8 && K == 2) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    r.e[0] = a.x; r.e[1] = a.y;
  } else if constexpr (sizeof(T) == 4 && K == 4) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    r.e[0] = a.x; r.e[1] = a.y; r.e[2] = a.z; r.e[3] = a.w;
  } else if constexpr (sizeof(T) == 4 && K == 2) {
    const float2 a = __ldg(reinterpret_cast<const float2*>(p));
    r.e[0] = a.x; r.e[1] = a.y;
  } else {
    r.e[0] = __ldg(p);
  }
  return r;
}

template <class T, int K>
__device__ __forceinline__ Vec<T, K> sload(const T* p) {  // shared
  Vec<T, K> r;
  if constexpr (sizeof(T) == 8 && K == 4) {
    const double2 a = reinterpret_cast<const double2*>(p)[0];
    const double2 b = reinterpret_cast<const double2*>(p)[1];
    r.e[0] = a.x; r.e[1] = a.y; r.e[2] = b.x; r.e[3] = b.y;
  } else if constexpr (sizeof(T) == 8 && K == 2) {
    const double2 a = reinterpret_cast<const double2*>(p)[0];
    r.e[0] = a.x; r.e[1] = a.y;
  } else if constexpr (sizeof(T) == 4 && K == 4) {
    const float4 a = reinterpret_cast<const float4*>(p)[0];
    r.e[0] = a.x; r.e[1] = a.y; r.e[2] = a.z; r.e[3] = a.w;
  } else if constexpr (sizeof(T) == 4 && K == 2) {
    const float2 a = reinterpret_cast<const float2*>(p)[0];
    r.e[0] = a.x; r.e[1] = a.y;
  } else {
    r.e[0] = p[0];
  }
  return r;
}

template <class T, int K>
__device__ __forceinline__ void vstore(T* p, const Vec<T, K>& v) {  // shared or global
  if constexpr (sizeof(T) == 8 && K == 4) {
    reinterpret_cast<double2*>(p)[0] = make_double2(v.e[0], v.e[1]);
    reinterpret_cast<double2*>(p)[1] = make_double2(v.e[2], v.e[3]);
  } else if constexpr (sizeof(T) == 8 && K == 2) {
    reinterpret_cast<double2*>(p)[0] = make_double2(v.e[0], v.e[1]);
  } else if constexpr (sizeof(T) == 4 && K == 4) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v.e[0], v.e[1], v.e[2], v.e[3]);
  } else if constexpr (sizeof(T) == 4 && K == 2) {
    reinterpret_cast<float2*>(p)[0] = make_float2(v.e[0], v.e[1]);
  } else {
    p[0] = v.e[0];
  }
}

// Value at k-1 / k+1 (periodic in k: the warp holds the whole row).
template <class T, int K>
__device__ __forceinline__ Vec<T, K> kminus(const Vec<T, K>& a, int lane) {
  Vec<T, K> r;
  r.e[0] = __shfl_sync(kFull, a.e[K - 1], (lane + 31) & 31);
#pragma unroll
  for (int e = 1; e < K; ++e) r.e[e] = a.e[e - 1];
  return r;
}
template <class T, int K>
__device__ __forceinline__ Vec<T, K> kplus(const Vec<T, K>& a, int lane) {
  Vec<T, K> r;
  r.e[K - 1] = __shfl_sync(kFull, a.e[0], (lane + 1) & 31);
#pragma unroll
  for (int e = 0; e + 1 < K; ++e) r.e[e] = a.e[e + 1];
  return r;
}
template <class T, int K>
__device__ __forceinline__ Vec<T, K> vabs(const Vec<T, K>& a) {
  Vec<T, K> r;
#pragma unroll
  for (int e = 0; e < K; ++e) r.e[e] = fabs(a.e[e]);
  return r;
}

// Reciprocals without the IEEE-division slow path: fp64 = MUFU.RCP64H seed +
// two Newton steps (error ~2^-80 before the final rounding, i.e. within an
// ulp); fp32 = MUFU.RCP (~1 ulp). Arguments are positive and normal here
// (denominators carry +eps, densities are positive).
__device__ __forceinline__ double rcp(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double e = fma(-d, y, 1.0);
  y = fma(y, e, y);
  e = fma(-d, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ float rcp(float d) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(d));
  return y;
}
__device__ __forceinline__ double qdiv(double a, double b) { return a * rcp(b); }
__device__ __forceinline__ float qdiv(float a, float b) { return a * rcp(b); }

// Upwind flux c * (c > 0 ? a : b): equal to pos(c) a + neg(c) b exactly.
template <class T>
__device__ __forceinline__ T upflux(T a, T b, T c) {
  return c * (c > T(0) ? a : b);
}
// Limited velocity: vel * min(1, bdL, buR) for vel > 0, else
// vel * min(1, buL, bdR) — equal to dev::limit exactly.
template <class T>
__device__ __forceinline__ T limit_sel(T vel, T bdL, T buR, T buL, T bdR) {
  const bool right = vel > T(0);
  const T a = right ? bdL : buL;
  const T b = right ? buR : bdR;
  return vel * tmin(tmin(T(1), a), b);
}

// Pseudo-velocity at one face with a single reciprocal:
//   ((|U| hb - U^2) nA dB dC - 0.125 U (S1 nB dC + S2 nC dB) dA) / (hb dA dB dC)
// where nX/dX are the numerator / (denominator incl. eps) of the ratios.
template <class T>
__device__ __forceinline__ T pseudo_face(T Un, T hL, T hR, T aR, T aL, T bp, T bm, T S1, T cp,
                                         T cm, T S2) {
  const T eps = Eps<T>::value;
  const T hb = T(0.5) * (hL + hR);
  const T nA = aR - aL, dA = (aR + aL) + eps;
  const T nB = bp - bm, dB = (bp + bm) + eps;
  const T nC = cp - cm, dC = (cp + cm) + eps;
  if constexpr (sizeof(T) == 8) {
    const T dBC = dB * dC;
    const T r = rcp(hb * dA * dBC);
    const T t1 = (fabs(Un) * hb - Un * Un) * nA * dBC;
    const T cr = (S1 * nB) * dC + (S2 * nC) * dB;
    const T t2 = (T(0.125) * Un) * cr * dA;
    return (t1 - t2) * r;
  } else {
    const T rhb = rcp(hb);
    const T A = qdiv(nA, dA), B = qdiv(nB, dB), C = qdiv(nC, dC);
    const T t1 = (fabs(Un) - Un * Un * rhb) * A;
    const T cr = S1 * B + S2 * C;
    return t1 - (T(0.125) * Un) * cr * rhb;
  }
}

template <class T, int L, int RW, int NW, bool NONOS>
__global__ void __launch_bounds__(NW * 32, 1) k_fused(Args<T> a) {
  using C = Cfg<T, L, RW, NW, NONOS>;
  constexpr int K = C::KPT, RR = C::RR, PL = C::PLANE;
  using V = Vec<T, K>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  T* s_x1 = sm;                          // 3 slots of psi^(1), by plane mod 3
  T* s_v = sm + 3 * PL;                  // y-face pseudo-velocities
  T* s_w = s_v + (NONOS ? 2 : 1) * PL;   // z-face pseudo-velocities
  T* s_bu = s_w + (NONOS ? 2 : 1) * PL;  // beta up,   2 slots (NONOS)
  T* s_bd = s_bu + 2 * PL;               // beta down, 2 slots (NONOS)

  const int tile = blockIdx.x % a.ntj;
  const int seg = blockIdx.x / a.ntj;
  const int span = a.o1 - a.o0;
  const int ib = a.o0 + static_cast<int>((static_cast<long long>(span) * seg) / a.nseg);
  const int ie = a.o0 + static_cast<int>((static_cast<long long>(span) * (seg + 1)) / a.nseg);
  if (ib >= ie) return;
  const int j0 = tile * C::TJ;
  const int m = a.m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kl = lane * K;  // first k of this lane

  // Rows of this warp: region row r = warp*RW + rr; global offsets of the
  // row (j wraps periodically) and of its j-1 / j+1 neighbours.
  int gj[RW], gjm[RW], gjp[RW];
#pragma unroll
  for (int rr = 0; rr < RW; ++rr) {
    int j = j0 - C::HALO + warp * RW + rr;
    j = ((j % m) + m) % m;
    gj[rr] = j * L + kl;
    gjm[rr] = (j == 0 ? m - 1 : j - 1) * L + kl;
    gjp[rr] = (j == m - 1 ? 0 : j + 1) * L + kl;
  }
  auto slot3 = [](int p) { return (p + 6) % 3; };  // p >= -3
  auto pl = [&](int p) { return static_cast<long long>(p + a.R) * a.plane; };
  auto srow = [&](int r) { return r * L + kl; };  // smem offset of a row vector

  V nmx_new[RW], nmn_new[RW], nmx[RW], nmn[RW];  // psi^n star extrema (NONOS)

  // P1: psi^(1) at plane p (donor cell) for all region rows.
  auto stage_donor = [&](int p) {
    const T* X = a.x + pl(p);
    const T* Xm = a.x + pl(p - 1);
    const T* Xp = a.x + pl(p + 1);
    const T* U = a.u + pl(p);
    const T* Up = a.u + pl(p + 1);
    const T* Vv = a.v + pl(p);
    const T* W = a.w + pl(p);
    const T* H = a.h + pl(p);
    T* dst = s_x1 + slot3(p) * PL;
#pragma unroll
    for (int rr = 0; rr < RW; ++rr) {
      const int r = warp * RW + rr;
      const V xc = vload<T, K>(X + gj[rr]);
      const V xm = vload<T, K>(Xm + gj[rr]), xp = vload<T, K>(Xp + gj[rr]);
      const V ym = vload<T, K>(X + gjm[rr]), yp = vload<T, K>(X + gjp[rr]);
      const V zm = kminus(xc, lane), zp = kplus(xc, lane);
      const V uc = vload<T, K>(U + gj[rr]), up = vload<T, K>(Up + gj[rr]);
      const V vc = vload<T, K>(Vv + gj[rr]), vp = vload<T, K>(Vv + gjp[rr]);
      const V wc = vload<T, K>(W + gj[rr]);
      const V wp = kplus(wc, lane);
      const V hc = vload<T, K>(H + gj[rr]);
      V res;
#pragma unroll
      for (int e = 0; e < K; ++e) {
        const T c = xc.e[e];
        const T fxl = upflux(xm.e[e], c, uc.e[e]);
        const T fxr = upflux(c, xp.e[e], up.e[e]);
        const T fyl = upflux(ym.e[e], c, vc.e[e]);
        const T fyr = upflux(c, yp.e[e], vp.e[e]);
        const T fzl = upflux(zm.e[e], c, wc.e[e]);
        const T fzr = upflux(c, zp.e[e], wp.e[e]);
        const T div = ((fxr - fxl) + (fyr - fyl)) + (fzr - fzl);
        res.e[e] = c - qdiv(div, hc.e[e]);
        if constexpr (NONOS) {
          nmx_new[rr].e[e] = tmax(tmax(tmax(c, xm.e[e]), tmax(xp.e[e], ym.e[e])),
                                  tmax(tmax(yp.e[e], zm.e[e]), zp.e[e]));
          nmn_new[rr].e[e] = tmin(tmin(tmin(c, xm.e[e]), tmin(xp.e[e], ym.e[e])),
                                  tmin(tmin(yp.e[e], zm.e[e]), zp.e[e]));
        }
      }
      vstore(dst + srow(r), res);
    }
  };

  // P2: pseudo-velocities around base plane pb: x-face pb+1 (into ut), y and
  // z faces of plane pb (into smem).
  auto stage_pseudo = [&](int pb, bool only_u, V* ut, T* vdst, T* wdst) {
    const T* s0 = s_x1 + slot3(pb - 1) * PL;
    const T* s1 = s_x1 + slot3(pb) * PL;
    const T* s2 = s_x1 + slot3(pb + 1) * PL;
    const T* U1 = a.u + pl(pb);
    const T* U2 = a.u + pl(pb + 1);
    const T* V1 = a.v + pl(pb);
    const T* V2 = a.v + pl(pb + 1);
    const T* W1 = a.w + pl(pb);
    const T* W2 = a.w + pl(pb + 1);
    const T* H1 = a.h + pl(pb);
    const T* H2 = a.h + pl(pb + 1);
#pragma unroll
    for (int rr = 0; rr < RW; ++rr) {
      const int r = warp * RW + rr;
      if (r < 1) continue;  // warp-uniform
      const bool row_u = r < RR - 1;  // x/z faces (y faces: every r >= 1)
      const V a1 = vabs(sload<T, K>(s1 + srow(r)));
      const V a1m = vabs(sload<T, K>(s1 + srow(r - 1)));
      const V u2c = vload<T, K>(U2 + gj[rr]);
      const V h1c = vload<T, K>(H1 + gj[rr]);
      const V a1km = kminus(a1, lane);
      if (row_u) {  // x-face between planes pb and pb+1 of this column
        const V a2 = vabs(sload<T, K>(s2 + srow(r)));
        const V a1p = vabs(sload<T, K>(s1 + srow(r + 1)));
        const V a2p = vabs(sload<T, K>(s2 + srow(r + 1)));
        const V a2m = vabs(sload<T, K>(s2 + srow(r - 1)));
        const V a1kp = kplus(a1, lane), a2kp = kplus(a2, lane), a2km = kminus(a2, lane);
        const V v1 = vload<T, K>(V1 + gj[rr]), v2 = vload<T, K>(V2 + gj[rr]);
        const V v1p = vload<T, K>(V1 + gjp[rr]), v2p = vload<T, K>(V2 + gjp[rr]);
        const V w1 = vload<T, K>(W1 + gj[rr]), w2 = vload<T, K>(W2 + gj[rr]);
        const V w1p = kplus(w1, lane), w2p = kplus(w2, lane);
        const V h2 = vload<T, K>(H2 + gj[rr]);
#pragma unroll
        for (int e = 0; e < K; ++e) {
          const T Vs = (v1.e[e] + v2.e[e]) + (v1p.e[e] + v2p.e[e]);
          const T Ws = (w1.e[e] + w2.e[e]) + (w1p.e[e] + w2p.e[e]);
          ut[rr].e[e] = pseudo_face<T>(u2c.e[e], h1c.e[e], h2.e[e], a2.e[e], a1.e[e],
                                       a1p.e[e] + a2p.e[e], a1m.e[e] + a2m.e[e], Vs,
                                       a1kp.e[e] + a2kp.e[e], a1km.e[e] + a2km.e[e], Ws);
        }
      }
      if (only_u) continue;
      const V a0 = vabs(sload<T, K>(s0 + srow(r)));
      const V a2 = vabs(sload<T, K>(s2 + srow(r)));
      const V u1c = vload<T, K>(U1 + gj[rr]);
      const V w1 = vload<T, K>(W1 + gj[rr]);
      {  // y-face between rows r-1 and r of plane pb
        const V a0m = vabs(sload<T, K>(s0 + srow(r - 1)));
        const V a2m = vabs(sload<T, K>(s2 + srow(r - 1)));
        const V a1mkp = kplus(a1m, lane), a1mkm = kminus(a1m, lane), a1kp = kplus(a1, lane);
        const V u1m = vload<T, K>(U1 + gjm[rr]), u2m = vload<T, K>(U2 + gjm[rr]);
        const V w1m = vload<T, K>(W1 + gjm[rr]);
        const V w1mkp = kplus(w1m, lane), w1kp = kplus(w1, lane);
        const V v1 = vload<T, K>(V1 + gj[rr]);
        const V h1m = vload<T, K>(H1 + gjm[rr]);
        V res;
#pragma unroll
        for (int e = 0; e < K; ++e) {
          const T Us = (u1m.e[e] + u1c.e[e]) + (u2m.e[e] + u2c.e[e]);
          const T Ws = (w1m.e[e] + w1.e[e]) + (w1mkp.e[e] + w1kp.e[e]);
          res.e[e] = pseudo_face<T>(v1.e[e], h1m.e[e], h1c.e[e], a1.e[e], a1m.e[e],
                                    a2m.e[e] + a2.e[e], a0m.e[e] + a0.e[e], Us,
                                    a1mkp.e[e] + a1kp.e[e], a1mkm.e[e] + a1km.e[e], Ws);
        }
        vstore(vdst + srow(r), res);
      }
      if (row_u) {  // z-face between k-1 and k
        const V a1p = vabs(sload<T, K>(s1 + srow(r + 1)));
        const V a1pkm = kminus(a1p, lane), a1mkm = kminus(a1m, lane);
        const V a2km = kminus(a2, lane), a0km = kminus(a0, lane);
        const V u2km = kminus(u2c, lane), u1km = kminus(u1c, lane);
        const V v1 = vload<T, K>(V1 + gj[rr]), v1p = vload<T, K>(V1 + gjp[rr]);
        const V v1km = kminus(v1, lane), v1pkm = kminus(v1p, lane);
        const V h1km = kminus(h1c, lane);
        V res;
#pragma unroll
        for (int e = 0; e < K; ++e) {
          const T Us = (u1km.e[e] + u1c.e[e]) + (u2km.e[e] + u2c.e[e]);
          const T Vs = (v1km.e[e] + v1.e[e]) + (v1pkm.e[e] + v1p.e[e]);
          res.e[e] = pseudo_face<T>(w1.e[e], h1km.e[e], h1c.e[e], a1.e[e], a1km.e[e],
                                    a2km.e[e] + a2.e[e], a0km.e[e] + a0.e[e], Us,
                                    a1pkm.e[e] + a1p.e[e], a1mkm.e[e] + a1m.e[e], Vs);
        }
        vstore(wdst + srow(r), res);
      }
    }
  };

  // ---- register carries along i (same (j,k) column) -------------------------
  V ucar[RW], ufresh[RW], fxc[RW];
#pragma unroll
  for (int rr = 0; rr < RW; ++rr)
#pragma unroll
    for (int e = 0; e < K; ++e) {
      ucar[rr].e[e] = ufresh[rr].e[e] = fxc[rr].e[e] = T(0);
      nmx[rr].e[e] = nmn[rr].e[e] = nmx_new[rr].e[e] = nmn_new[rr].e[e] = T(0);
    }

  const int lag = NONOS ? 2 : 1;  // psi^(1) planes ahead of the output plane
  // warm-up: psi^(1) on the first two planes of the window, then the x-face
  // pseudo-velocity between them.
  stage_donor(ib - lag);
  stage_donor(ib - lag + 1);
  if constexpr (NONOS) {
#pragma unroll
    for (int rr = 0; rr < RW; ++rr) {
      nmx[rr] = nmx_new[rr];
      nmn[rr] = nmn_new[rr];
    }
  }
  __syncthreads();
  stage_pseudo(ib - lag, true, ucar, nullptr, nullptr);

  const int tstart = NONOS ? ib - 2 : ib;
  for (int t = tstart; t < ie; ++t) {
    const bool emit = t >= ib;
    stage_donor(t + lag);  // psi^(1) of the newest plane
    __syncthreads();
    if constexpr (NONOS) {
      const int p1 = t + 1;
      T* vA = s_v + (p1 & 1) * PL;              // y-face velocities, plane t+1
      T* wA = s_w + (p1 & 1) * PL;
      const T* vB = s_v + ((p1 + 1) & 1) * PL;  // limited, plane t
      const T* wB = s_w + ((p1 + 1) & 1) * PL;
      T* buA = s_bu + (p1 & 1) * PL;            // beta, plane t+1
      T* bdA = s_bd + (p1 & 1) * PL;
      const T* buB = s_bu + ((p1 + 1) & 1) * PL;  // beta, plane t
      const T* bdB = s_bd + ((p1 + 1) & 1) * PL;
      stage_pseudo(p1, false, ufresh, vA, wA);
      __syncthreads();
      // P3: 7-point bounds and beta of plane t+1.
      {
        const T* s0 = s_x1 + slot3(t) * PL;
        const T* s1 = s_x1 + slot3(t + 1) * PL;
        const T* s2 = s_x1 + slot3(t + 2) * PL;
        const T* H1 = a.h + pl(p1);
#pragma unroll
        for (int rr = 0; rr < RW; ++rr) {
          const int r = warp * RW + rr;
          if (r < 1 || r >= RR - 1) continue;
          const V xc = sload<T, K>(s1 + srow(r));
          const V xm = sload<T, K>(s0 + srow(r)), xp = sload<T, K>(s2 + srow(r));
          const V ym = sload<T, K>(s1 + srow(r - 1)), yp = sload<T, K>(s1 + srow(r + 1));
          const V zm = kminus(xc, lane), zp = kplus(xc, lane);
          const V va = sload<T, K>(vA + srow(r)), vap = sload<T, K>(vA + srow(r + 1));
          const V wa = sload<T, K>(wA + srow(r));
          const V wap = kplus(wa, lane);
          const V hc = vload<T, K>(H1 + gj[rr]);
          V bu, bd;
#pragma unroll
          for (int e = 0; e < K; ++e) {
            const T c = xc.e[e];
            const T mx = tmax(tmax(tmax(nmx[rr].e[e], c), tmax(xm.e[e], xp.e[e])),
                              tmax(tmax(ym.e[e], yp.e[e]), tmax(zm.e[e], zp.e[e])));
            const T mn = tmin(tmin(tmin(nmn[rr].e[e], c), tmin(xm.e[e], xp.e[e])),
                              tmin(tmin(ym.e[e], yp.e[e]), tmin(zm.e[e], zp.e[e])));
            const T axl = upflux(xm.e[e], c, ucar[rr].e[e]);
            const T axr = upflux(c, xp.e[e], ufresh[rr].e[e]);
            const T ayl = upflux(ym.e[e], c, va.e[e]);
            const T ayr = upflux(c, yp.e[e], vap.e[e]);
            const T azl = upflux(zm.e[e], c, wa.e[e]);
            const T azr = upflux(c, zp.e[e], wap.e[e]);
            // 2*pos(f) = f + |f| and -2*neg(f) = |f| - f are exact, so these
            // are the oracle's inflow/outflow sums scaled by exactly 2.
            const T fin2 = (((axl + fabs(axl)) + (fabs(axr) - axr)) +
                            ((ayl + fabs(ayl)) + (fabs(ayr) - ayr))) +
                           ((azl + fabs(azl)) + (fabs(azr) - azr));
            const T fout2 = (((axr + fabs(axr)) + (fabs(axl) - axl)) +
                             ((ayr + fabs(ayr)) + (fabs(ayl) - ayl))) +
                            ((azr + fabs(azr)) + (fabs(azl) - azl));
            const T di = T(0.5) * fin2 + Eps<T>::value, dou = T(0.5) * fout2 + Eps<T>::value;
            if constexpr (sizeof(T) == 8) {
              const T rr2 = rcp(di * dou);
              bu.e[e] = ((mx - c) * hc.e[e]) * dou * rr2;
              bd.e[e] = ((c - mn) * hc.e[e]) * di * rr2;
            } else {
              bu.e[e] = qdiv((mx - c) * hc.e[e], di);
              bd.e[e] = qdiv((c - mn) * hc.e[e], dou);
            }
          }
          vstore(buA + srow(r), bu);
          vstore(bdA + srow(r), bd);
        }
      }
      __syncthreads();
      // P4: limit plane t+1 velocities; P5: final update of plane t.
      {
        const T* s0 = s_x1 + slot3(t) * PL;
        const T* s1 = s_x1 + slot3(t + 1) * PL;
        const T* H0 = a.h + pl(t);
        T* O = a.out + pl(t);
#pragma unroll
        for (int rr = 0; rr < RW; ++rr) {
          const int r = warp * RW + rr;
          if (r < 2 || r >= RR - 1) continue;
          const V bu = sload<T, K>(buA + srow(r)), bd = sload<T, K>(bdA + srow(r));
          {
            const V va = sload<T, K>(vA + srow(r));
            const V bum = sload<T, K>(buA + srow(r - 1)), bdm = sload<T, K>(bdA + srow(r - 1));
            V res;
#pragma unroll
            for (int e = 0; e < K; ++e)
              res.e[e] = limit_sel(va.e[e], bdm.e[e], bu.e[e], bum.e[e], bd.e[e]);
            vstore(vA + srow(r), res);
          }
          if (r >= RR - 2) continue;
          const V wa = sload<T, K>(wA + srow(r));
          const V bukm = kminus(bu, lane), bdkm = kminus(bd, lane);
          const V buo = sload<T, K>(buB + srow(r)), bdo = sload<T, K>(bdB + srow(r));
          const V xc = sload<T, K>(s0 + srow(r));
          const V x1 = sload<T, K>(s1 + srow(r));
          V wres, fxr;
#pragma unroll
          for (int e = 0; e < K; ++e) {
            wres.e[e] = limit_sel(wa.e[e], bdkm.e[e], bu.e[e], bukm.e[e], bd.e[e]);
            const T ul = limit_sel(ucar[rr].e[e], bdo.e[e], bu.e[e], buo.e[e], bd.e[e]);
            fxr.e[e] = upflux(xc.e[e], x1.e[e], ul);
          }
          vstore(wA + srow(r), wres);
          if (emit) {
            const V ym = sload<T, K>(s0 + srow(r - 1)), yp = sload<T, K>(s0 + srow(r + 1));
            const V zm = kminus(xc, lane), zp = kplus(xc, lane);
            const V vb = sload<T, K>(vB + srow(r)), vbp = sload<T, K>(vB + srow(r + 1));
            const V wb = sload<T, K>(wB + srow(r));
            const V wbp = kplus(wb, lane);
            const V hc = vload<T, K>(H0 + gj[rr]);
            V res;
#pragma unroll
            for (int e = 0; e < K; ++e) {
              const T c = xc.e[e];
              const T fyl = upflux(ym.e[e], c, vb.e[e]);
              const T fyr = upflux(c, yp.e[e], vbp.e[e]);
              const T fzl = upflux(zm.e[e], c, wb.e[e]);
              const T fzr = upflux(c, zp.e[e], wbp.e[e]);
              const T div = ((fxr.e[e] - fxc[rr].e[e]) + (fyr - fyl)) + (fzr - fzl);
              res.e[e] = c - qdiv(div, hc.e[e]);
            }
            const int j = j0 + r - 2;
            if (j < m) vstore(O + gj[rr], res);
          }
          fxc[rr] = fxr;
        }
      }
#pragma unroll
      for (int rr = 0; rr < RW; ++rr) {
        ucar[rr] = ufresh[rr];
        nmx[rr] = nmx_new[rr];
        nmn[rr] = nmn_new[rr];
      }
      __syncthreads();
    } else {
      // Plain IORD=2: pseudo-velocities of plane t, then the final update.
      stage_pseudo(t, false, ufresh, s_v, s_w);
      __syncthreads();
      const T* sm1 = s_x1 + slot3(t - 1) * PL;
      const T* s0 = s_x1 + slot3(t) * PL;
      const T* s1 = s_x1 + slot3(t + 1) * PL;
      const T* H0 = a.h + pl(t);
      T* O = a.out + pl(t);
#pragma unroll
      for (int rr = 0; rr < RW; ++rr) {
        const int r = warp * RW + rr;
        if (r < 1 || r >= RR - 1) continue;
        const V xc = sload<T, K>(s0 + srow(r));
        const V xm = sload<T, K>(sm1 + srow(r)), xp = sload<T, K>(s1 + srow(r));
        const V ym = sload<T, K>(s0 + srow(r - 1)), yp = sload<T, K>(s0 + srow(r + 1));
        const V zm = kminus(xc, lane), zp = kplus(xc, lane);
        const V vv = sload<T, K>(s_v + srow(r)), vvp = sload<T, K>(s_v + srow(r + 1));
        const V ww = sload<T, K>(s_w + srow(r));
        const V wwp = kplus(ww, lane);
        const V hc = vload<T, K>(H0 + gj[rr]);
        V res;
#pragma unroll
        for (int e = 0; e < K; ++e) {
          const T c = xc.e[e];
          const T fxl = upflux(xm.e[e], c, ucar[rr].e[e]);
          const T fxr = upflux(c, xp.e[e], ufresh[rr].e[e]);
          const T fyl = upflux(ym.e[e], c, vv.e[e]);
          const T fyr = upflux(c, yp.e[e], vvp.e[e]);
          const T fzl = upflux(zm.e[e], c, ww.e[e]);
          const T fzr = upflux(c, zp.e[e], wwp.e[e]);
          const T div = ((fxr - fxl) + (fyr - fyl)) + (fzr - fzl);
          res.e[e] = c - qdiv(div, hc.e[e]);
        }
        const int j = j0 + r - 1;
        if (j < m) vstore(O + gj[rr], res);
        ucar[rr] = ufresh[rr];
      }
      __syncthreads();
    }
  }
}

struct Plan {
  int ntj, nseg;
};

// Choose the i-segmentation: minimise waves x (planes per segment + warm-up).
Plan plan_grid(std::int64_t m, int tj, std::int64_t planes, int resident, int warm) {
  Plan best{static_cast<int>((m + tj - 1) / tj), 1};
  double best_cost = 1e300;
  for (int nseg = 1; nseg <= planes; ++nseg) {
    const long long blocks = static_cast<long long>(best.ntj) * nseg;
    if (blocks > INT_MAX / 2) break;
    const long long waves = (blocks + resident - 1) / resident;
    const long long seg = (planes + nseg - 1) / nseg;
    const double cost = static_cast<double>(waves) * static_cast<double>(seg + warm);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best.nseg = nseg;
    }
  }
  return best;
}

template <class T, int L, int RW, int NW, bool NONOS>
int launch_cfg(const FusedShape& fs, const T* x, const T* u, const T* v, const T* w, const T* h,
               T* out, int num_sms, cudaStream_t st) {
  using C = Cfg<T, L, RW, NW, NONOS>;
  static bool configured = false;
  static int per_sm = 1;
  if (!configured) {
    cudaFuncSetAttribute(k_fused<T, L, RW, NW, NONOS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(C::SMEM));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fused<T, L, RW, NW, NONOS>, C::NT,
                                                  C::SMEM);
    if (per_sm < 1) per_sm = 1;
    configured = true;
  }
  const Plan p = plan_grid(fs.m, C::TJ, fs.o1 - fs.o0, per_sm * num_sms, NONOS ? 4 : 2);
  Args<T> a{x, u, v, w, h, out, static_cast<int>(fs.m), static_cast<int>(fs.R), p.ntj, p.nseg,
            static_cast<int>(fs.o0), static_cast<int>(fs.o1), fs.m * fs.l};
  k_fused<T, L, RW, NW, NONOS><<<p.ntj * p.nseg, C::NT, C::SMEM, st>>>(a);
  return 1;
}

template <class T, bool NONOS>
int dispatch_l(const FusedShape& fs, const T* x, const T* u, const T* v, const T* w, const T* h,
               T* out, int num_sms, cudaStream_t st) {
  switch (fs.l) {
    case 128: return launch_cfg<T, 128, 1, 16, NONOS>(fs, x, u, v, w, h, out, num_sms, st);
    case 64: return launch_cfg<T, 64, 2, 16, NONOS>(fs, x, u, v, w, h, out, num_sms, st);
    case 32: return launch_cfg<T, 32, 4, 16, NONOS>(fs, x, u, v, w, h, out, num_sms, st);
    default: return 0;
  }
}

}  // namespace

bool fused_supported(int iord, int nonos, std::int64_t m, std::int64_t l, bool) {
  (void)nonos;
  return iord == 2 && (l == 32 || l == 64 || l == 128) && m >= 3 && m < (1 << 20);
}

template <class T>
int launch_fused(const FusedShape& fs, int iord, int nonos, const T* x, const T* u, const T* v,
                 const T* w, const T* h, T* out, int num_sms, cudaStream_t st) {
  if (iord != 2) return 0;
  return nonos ? dispatch_l<T, true>(fs, x, u, v, w, h, out, num_sms, st)
               : dispatch_l<T, false>(fs, x, u, v, w, h, out, num_sms, st);
}
template int launch_fused<double>(const FusedShape&, int, int, const double*, const double*,
                                  const double*, const double*, const double*, double*, int,
                                  cudaStream_t);
template int launch_fused<float>(const FusedShape&, int, int, const float*, const float*,
                                 const float*, const float*, const float*, float*, int,
                                 cudaStream_t);

}  // namespace imb::dev
