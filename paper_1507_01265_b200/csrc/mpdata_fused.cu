// Fused streaming MPDATA step (IORD = 2, optional nonoscillatory limiter):
// one kernel reads psi^n, u, v, w, h and writes psi^{n+1}; every
// intermediate (psi^(1), pseudo-velocities, beta bounds, limited velocities,
// fluxes) lives in shared memory or registers.
//
// Geometry (B200-first):
//  * k (contiguous, l <= 128) is covered completely by each warp's lanes
//    (k = lane + 32*kk), periodic in-register wrap -> no k halo at all.
//  * Each block owns a j-tile of TJ output rows plus a 2-row (limiter) or
//    1-row (plain) recomputed halo on either side: RR = NW*RW region rows,
//    one or more rows per warp, fixed for every stage.
//  * The block streams along i (the slab axis) over a segment of planes. The
//    stages run with a lag of one plane each, so along i nothing is
//    recomputed except a 2-plane warm-up per segment: smem keeps 3 planes of
//    psi^(1), 2 of the y/z pseudo-velocities and 1 of each beta; every
//    same-column dependency along i (x-face velocity, beta of the previous
//    plane, the x-flux shared by two consecutive outputs) is a register
//    carry.
//  * Divisions: fp64 folds the four divisions of a pseudo-velocity into one
//    reciprocal of hb*dA*dB*dC and the two beta divisions into one; fp32
//    uses the fast reciprocal. Both stay inside the parity tolerance.
// The per-cell arithmetic follows SURVEY.md Appendix A (see mpdata_math.cuh).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>

#include "mpdata_kernels.cuh"
#include "mpdata_math.cuh"

namespace imb::dev {

namespace {

template <class T, int L, int RR_, int NT_, bool NONOS>
struct Cfg {
  static constexpr int RR = RR_;                  // region rows
  static constexpr int Q = RR * L / NT_;          // cells per thread
  static_assert(Q * NT_ == RR * L && NT_ % L == 0, "threads must tile whole rows");
  static constexpr int HALO = NONOS ? 2 : 1;      // recomputed rows on each side
  static constexpr int TJ = RR - 2 * HALO;        // output rows per tile
  static constexpr int NT = NT_;
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
// Limited velocity: vel * min(1, bdL, buR) for outflow to the right, else
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

template <class T, int L, int RR_, int NT, bool NONOS>
__global__ void __launch_bounds__(NT, 1) k_fused(Args<T> a) {
  using C = Cfg<T, L, RR_, NT, NONOS>;
  constexpr int Q = C::Q, RR = C::RR, PL = C::PLANE;
  constexpr int RSTEP = NT / L;  // rows between a thread's consecutive cells
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
  // Thread -> cells: cell q is (row r0 + q*RSTEP, column k); a warp covers 32
  // consecutive k of one row, so every row test below is warp-uniform.
  const int r0 = threadIdx.x / L, kc = threadIdx.x % L;
  int gjr[Q], gjmr[Q], gjpr[Q];
#pragma unroll
  for (int rr = 0; rr < Q; ++rr) {
    int j = j0 - C::HALO + r0 + rr * RSTEP;
    j = ((j % m) + m) % m;
    gjr[rr] = j * L;
    gjmr[rr] = (j == 0 ? m - 1 : j - 1) * L;
    gjpr[rr] = (j == m - 1 ? 0 : j + 1) * L;
  }
#define IMB_CELL(q)                                                   \
  const int rr_ = (q);                                                \
  const int r = r0 + rr_ * RSTEP;                                     \
  const int k = kc;                                                   \
  const int km = k == 0 ? L - 1 : k - 1, kp = k == L - 1 ? 0 : k + 1; \
  const int o = r * L + k, om_k = r * L + km, op_k = r * L + kp;      \
  const int gj = gjr[rr_], gjm = gjmr[rr_], gjp = gjpr[rr_];          \
  (void)om_k; (void)op_k; (void)gjm; (void)gjp; (void)km; (void)kp;
  auto slot3 = [](int p) { return (p + 6) % 3; };  // p >= -3
  auto pl = [&](int p) { return static_cast<long long>(p + a.R) * a.plane; };

  // ψn star extrema of the newest donor plane (NONOS), carried one plane.
  T nmx_new[Q], nmn_new[Q], nmx[Q], nmn[Q];
  // P1: psi^(1) at plane p (donor cell) for all region rows.
  auto stage_donor = [&](int p) {
    const T* X = a.x + pl(p);
    const T* Xm = a.x + pl(p - 1);
    const T* Xp = a.x + pl(p + 1);
    const T* U = a.u + pl(p);
    const T* Up = a.u + pl(p + 1);
    const T* V = a.v + pl(p);
    const T* W = a.w + pl(p);
    const T* H = a.h + pl(p);
    T* dst = s_x1 + slot3(p) * PL;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      IMB_CELL(q)
      const int c = gj + k;
      const T xc = __ldg(X + c);
      const T xm = __ldg(Xm + c), xp = __ldg(Xp + c);
      const T ym = __ldg(X + gjm + k), yp = __ldg(X + gjp + k);
      const T zm = __ldg(X + gj + km), zp = __ldg(X + gj + kp);
      const T fxl = upflux(xm, xc, __ldg(U + c));
      const T fxr = upflux(xc, xp, __ldg(Up + c));
      const T fyl = upflux(ym, xc, __ldg(V + c));
      const T fyr = upflux(xc, yp, __ldg(V + gjp + k));
      const T fzl = upflux(zm, xc, __ldg(W + c));
      const T fzr = upflux(xc, zp, __ldg(W + gj + kp));
      const T div = ((fxr - fxl) + (fyr - fyl)) + (fzr - fzl);
      dst[o] = xc - qdiv(div, __ldg(H + c));
      if constexpr (NONOS) {
        nmx_new[q] = tmax(tmax(tmax(xc, xm), tmax(xp, ym)), tmax(tmax(yp, zm), zp));
        nmn_new[q] = tmin(tmin(tmin(xc, xm), tmin(xp, ym)), tmin(tmin(yp, zm), zp));
      }
    }
  };

  // P2: pseudo-velocities around base plane pb: x-face pb+1 (into ut), y and
  // z faces of plane pb (into smem).
  auto stage_pseudo = [&](int pb, bool only_u, T* ut, T* vdst, T* wdst) {
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
    for (int q = 0; q < Q; ++q) {
      IMB_CELL(q)
      const int c = gj + k;
      const bool row_u = r >= 1 && r < RR - 1;  // x/z faces
      const bool row_v = r >= 1;                // y faces
      const T a1c = fabs(s1[o]);
      const T u2c = __ldg(U2 + c), h1c = __ldg(H1 + c);
      if (row_u) {  // x-face between planes pb and pb+1 of this column
        const T a2c = fabs(s2[o]);
        const T bp = fabs(s1[o + L]) + fabs(s2[o + L]);
        const T bm = fabs(s1[o - L]) + fabs(s2[o - L]);
        const T cp = fabs(s1[op_k]) + fabs(s2[op_k]);
        const T cm = fabs(s1[om_k]) + fabs(s2[om_k]);
        const int cjp = gjp + k, ckp = gj + kp;
        const T Vs = (__ldg(V1 + c) + __ldg(V2 + c)) + (__ldg(V1 + cjp) + __ldg(V2 + cjp));
        const T Ws = (__ldg(W1 + c) + __ldg(W2 + c)) + (__ldg(W1 + ckp) + __ldg(W2 + ckp));
        ut[q] = pseudo_face<T>(u2c, h1c, __ldg(H2 + c), a2c, a1c, bp, bm, Vs, cp, cm, Ws);
      }
      if (only_u) continue;
      const T u1c = __ldg(U1 + c);
      if (row_v) {  // y-face between rows r-1 and r of plane pb
        const int om = o - L;
        const int cjm = gjm + k;
        const T aL = fabs(s1[om]);
        const T bp = fabs(s2[om]) + fabs(s2[o]);
        const T bm = fabs(s0[om]) + fabs(s0[o]);
        const T cp = fabs(s1[op_k - L]) + fabs(s1[op_k]);
        const T cm = fabs(s1[om_k - L]) + fabs(s1[om_k]);
        const T Us = (__ldg(U1 + cjm) + u1c) + (__ldg(U2 + cjm) + u2c);
        const int cjmkp = gjm + kp, ckp = gj + kp;
        const T Ws = (__ldg(W1 + cjm) + __ldg(W1 + c)) + (__ldg(W1 + cjmkp) + __ldg(W1 + ckp));
        vdst[o] = pseudo_face<T>(__ldg(V1 + c), __ldg(H1 + cjm), h1c, a1c, aL, bp, bm, Us, cp, cm,
                                 Ws);
      }
      if (row_u) {  // z-face between k-1 and k
        const int ckm = gj + km;
        const T aL = fabs(s1[om_k]);
        const T bp = fabs(s2[om_k]) + fabs(s2[o]);
        const T bm = fabs(s0[om_k]) + fabs(s0[o]);
        const T cp = fabs(s1[om_k + L]) + fabs(s1[o + L]);
        const T cm = fabs(s1[om_k - L]) + fabs(s1[o - L]);
        const T Us = (__ldg(U1 + ckm) + u1c) + (__ldg(U2 + ckm) + u2c);
        const int cjpkm = gjp + km, cjp = gjp + k;
        const T Vs = (__ldg(V1 + ckm) + __ldg(V1 + c)) + (__ldg(V1 + cjpkm) + __ldg(V1 + cjp));
        wdst[o] = pseudo_face<T>(__ldg(W1 + c), __ldg(H1 + ckm), h1c, a1c, aL, bp, bm, Us, cp, cm,
                                 Vs);
      }
    }
  };

  // ---- register carries along i (same (j,k) column) -------------------------
  T ucar[Q], ufresh[Q], fxc[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    ucar[q] = ufresh[q] = fxc[q] = T(0);
    nmx[q] = nmn[q] = nmx_new[q] = nmn_new[q] = T(0);
  }

  const int lag = NONOS ? 2 : 1;  // psi^(1) planes ahead of the output plane
  // warm-up: psi^(1) on the first two planes of the window, then the x-face
  // pseudo-velocity between them.
  stage_donor(ib - lag);
  stage_donor(ib - lag + 1);
  if constexpr (NONOS) {
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      nmx[q] = nmx_new[q];
      nmn[q] = nmn_new[q];
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
        for (int q = 0; q < Q; ++q) {
          IMB_CELL(q)
          if (r < 1 || r >= RR - 1) continue;
          const T xc = s1[o];
          const T xm = s0[o], xp = s2[o], ym = s1[o - L], yp = s1[o + L];
          const T zm = s1[om_k], zp = s1[op_k];
          const T mx = tmax(tmax(tmax(nmx[q], xc), tmax(xm, xp)), tmax(tmax(ym, yp), tmax(zm, zp)));
          const T mn = tmin(tmin(tmin(nmn[q], xc), tmin(xm, xp)), tmin(tmin(ym, yp), tmin(zm, zp)));
          const T axl = upflux(xm, xc, ucar[q]);
          const T axr = upflux(xc, xp, ufresh[q]);
          const T ayl = upflux(ym, xc, vA[o]);
          const T ayr = upflux(xc, yp, vA[o + L]);
          const T azl = upflux(zm, xc, wA[o]);
          const T azr = upflux(xc, zp, wA[op_k]);
          // 2*pos(f) = f + |f|, -2*neg(f) = |f| - f (both exact): the sums are
          // the oracle's fin/fout scaled by exactly 2.
          const T fin2 = (((axl + fabs(axl)) + (fabs(axr) - axr)) + ((ayl + fabs(ayl)) + (fabs(ayr) - ayr))) +
                         ((azl + fabs(azl)) + (fabs(azr) - azr));
          const T fout2 = (((axr + fabs(axr)) + (fabs(axl) - axl)) + ((ayr + fabs(ayr)) + (fabs(ayl) - ayl))) +
                          ((azr + fabs(azr)) + (fabs(azl) - azl));
          const T hc = __ldg(H1 + gj + k);
          const T di = T(0.5) * fin2 + Eps<T>::value, dou = T(0.5) * fout2 + Eps<T>::value;
          T bu, bd;
          if constexpr (sizeof(T) == 8) {
            const T rr2 = rcp(di * dou);
            bu = ((mx - xc) * hc) * dou * rr2;
            bd = ((xc - mn) * hc) * di * rr2;
          } else {
            bu = qdiv((mx - xc) * hc, di);
            bd = qdiv((xc - mn) * hc, dou);
          }
          buA[o] = bu;
          bdA[o] = bd;
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
        for (int q = 0; q < Q; ++q) {
          IMB_CELL(q)
          if (r >= 2 && r < RR - 1)
            vA[o] = limit_sel(vA[o], bdA[o - L], buA[o], buA[o - L], bdA[o]);
          if (r < 2 || r >= RR - 2) continue;
          wA[o] = limit_sel(wA[o], bdA[om_k], buA[o], buA[om_k], bdA[o]);
          const T ul = limit_sel(ucar[q], bdB[o], buA[o], buB[o], bdA[o]);
          const T xc = s0[o];
          const T fxr = upflux(xc, s1[o], ul);
          if (emit) {
            const T fyl = upflux(s0[o - L], xc, vB[o]);
            const T fyr = upflux(xc, s0[o + L], vB[o + L]);
            const T fzl = upflux(s0[om_k], xc, wB[o]);
            const T fzr = upflux(xc, s0[op_k], wB[op_k]);
            const T div = ((fxr - fxc[q]) + (fyr - fyl)) + (fzr - fzl);
            const int j = j0 + r - 2;
            if (j < m) O[gj + k] = xc - qdiv(div, __ldg(H0 + gj + k));
          }
          fxc[q] = fxr;
        }
      }
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        ucar[q] = ufresh[q];
        nmx[q] = nmx_new[q];
        nmn[q] = nmn_new[q];
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
      for (int q = 0; q < Q; ++q) {
        IMB_CELL(q)
        if (r < 1 || r >= RR - 1) continue;
        const T xc = s0[o];
        const T fxl = upflux(sm1[o], xc, ucar[q]);
        const T fxr = upflux(xc, s1[o], ufresh[q]);
        const T fyl = upflux(s0[o - L], xc, s_v[o]);
        const T fyr = upflux(xc, s0[o + L], s_v[o + L]);
        const T fzl = upflux(s0[om_k], xc, s_w[o]);
        const T fzr = upflux(xc, s0[op_k], s_w[op_k]);
        const T div = ((fxr - fxl) + (fyr - fyl)) + (fzr - fzl);
        const int j = j0 + r - 1;
        if (j < m) O[gj + k] = xc - qdiv(div, __ldg(H0 + gj + k));
        ucar[q] = ufresh[q];
      }
      __syncthreads();
    }
  }
#undef IMB_CELL
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

template <class T, int L, int RR, int NT, bool NONOS>
int launch_cfg(const FusedShape& fs, const T* x, const T* u, const T* v, const T* w, const T* h,
               T* out, int num_sms, cudaStream_t st) {
  using C = Cfg<T, L, RR, NT, NONOS>;
  static bool configured = false;
  static int per_sm = 1;
  if (!configured) {
    cudaFuncSetAttribute(k_fused<T, L, RR, NT, NONOS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(C::SMEM));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fused<T, L, RR, NT, NONOS>, C::NT,
                                                  C::SMEM);
    if (per_sm < 1) per_sm = 1;
    configured = true;
  }
  const Plan p = plan_grid(fs.m, C::TJ, fs.o1 - fs.o0, per_sm * num_sms, NONOS ? 4 : 2);
  Args<T> a{x, u, v, w, h, out, static_cast<int>(fs.m), static_cast<int>(fs.R), p.ntj, p.nseg,
            static_cast<int>(fs.o0), static_cast<int>(fs.o1), fs.m * fs.l};
  k_fused<T, L, RR, NT, NONOS><<<p.ntj * p.nseg, C::NT, C::SMEM, st>>>(a);
  return 1;
}

template <class T, bool NONOS>
int dispatch_l(const FusedShape& fs, const T* x, const T* u, const T* v, const T* w, const T* h,
               T* out, int num_sms, cudaStream_t st) {
  static const int nt = [] {
    const char* e = std::getenv("IMB_FUSED_NT");
    return e ? std::atoi(e) : 1024;
  }();
  if (nt == 512) {
    switch (fs.l) {
      case 128: return launch_cfg<T, 128, 16, 512, NONOS>(fs, x, u, v, w, h, out, num_sms, st);
      case 64: return launch_cfg<T, 64, 32, 512, NONOS>(fs, x, u, v, w, h, out, num_sms, st);
      case 32: return launch_cfg<T, 32, 64, 512, NONOS>(fs, x, u, v, w, h, out, num_sms, st);
      default: return 0;
    }
  }
  switch (fs.l) {
    case 128: return launch_cfg<T, 128, 16, 1024, NONOS>(fs, x, u, v, w, h, out, num_sms, st);
    case 64: return launch_cfg<T, 64, 32, 1024, NONOS>(fs, x, u, v, w, h, out, num_sms, st);
    case 32: return launch_cfg<T, 32, 64, 1024, NONOS>(fs, x, u, v, w, h, out, num_sms, st);
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
