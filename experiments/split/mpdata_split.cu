// EXPERIMENT (not built into the product; measured slower).
// Built against paper_1507_01265_b200/csrc headers with launch_split /
// split_supported declared as in the original mpdata_kernels.cuh patch.
//
// Split IORD=2 + limiter step: two streaming kernels instead of one.
//
//  k_split_a: donor psi^(1) and all antidiffusive pseudo-velocities, written
//             to HBM (psi1, ut, vt, wt). A j-tile of 16 output rows needs only
//             one recomputed donor row on each side, and the donor of plane
//             p+2 shares a barrier phase with the pseudo-velocities of plane p
//             (one barrier per plane).
//  k_split_b: 7-point bounds, beta, limiter and the final update, reading the
//             four intermediates; a j-tile of 14 output rows recomputes beta
//             on one row on each side.
//
// Against the single fused kernel (mpdata_fused.cu) this trades 64 B/cell of
// extra HBM traffic (the step is far from HBM-bound) for less j-halo
// recompute (pseudo-velocities 1.0x instead of 1.25x) and a smaller live
// state per thread in each kernel. The per-cell arithmetic is the same
// (mpdata_math.cuh), so results stay within the parity tolerance; the
// decomposition tests require bit-identity only within one path.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>

#include "mpdata_kernels.cuh"
#include "mpdata_math.cuh"
#include "mpdata_vec.cuh"

namespace imb::dev {

namespace {

template <class T>
struct ArgsA {
  const T* __restrict__ x;
  const T* __restrict__ u;
  const T* __restrict__ v;
  const T* __restrict__ w;
  const T* __restrict__ h;
  T* __restrict__ x1;  // psi^(1)
  T* __restrict__ ut;  // pseudo-velocity at x-face i-1/2 (index i)
  T* __restrict__ vt;  // y-face j-1/2
  T* __restrict__ wt;  // z-face k-1/2
  int m, R, ntj, kseg, lseg;
  int p0, p1;  // pseudo-velocity planes [p0, p1); psi1 is written on [p0-1, p1]
  long long plane;
  int pf;
};

template <class T>
struct ArgsB {
  const T* __restrict__ x;  // psi^n
  const T* __restrict__ h;
  const T* __restrict__ x1;
  const T* __restrict__ ut;
  const T* __restrict__ vt;
  const T* __restrict__ wt;
  T* __restrict__ out;
  int m, R, ntj, kseg, lseg;
  int o0, o1;
  long long plane;
  T* push_lo;
  T* push_hi;
  int lo_ni;
  int ni;
};

// ---- kernel A ------------------------------------------------------------
template <class T, int L, int NW, int NS>
__global__ void __launch_bounds__(NW * 32, 1) k_split_a(ArgsA<T> a) {
  constexpr int K = L / (32 * NS), RR = NW, SR = RR + 2, PL = SR * L;
  using V = Vec<T, K>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // 4 psi^(1) planes (by plane mod 4) of SR rows; region row r (-1 .. RR) at (r+1)*L
  T* const sx = reinterpret_cast<T*>(smem_raw) + L;

  const int span = a.p1 - a.p0;
  const int nbig = a.ntj * a.kseg;
  const bool big = static_cast<int>(blockIdx.x) < nbig;
  const int tile = big ? blockIdx.x % a.ntj : blockIdx.x - nbig;
  const int pa = a.p0 + (big ? static_cast<int>(blockIdx.x / a.ntj) * a.lseg : a.kseg * a.lseg);
  const int pb = big ? pa + a.lseg : a.p1;
  if (pa >= pb) return;
  (void)span;
  const int m = a.m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j0 = tile * RR;
  auto wrapj = [&](int j) { return ((j % m) + m) % m; };
  // own row (r = warp) and, for warps 0 / NW-1, the halo donor row -1 / RR
  const int jr = wrapj(j0 + warp);
  const int gj = jr * L, gjm = (jr == 0 ? m - 1 : jr - 1) * L, gjp = (jr == m - 1 ? 0 : jr + 1) * L;
  const int hr = warp == 0 ? -1 : RR;  // halo row of warps 0 / NW-1
  const int jh = wrapj(j0 + hr);
  const int hj = jh * L, hjm = (jh == 0 ? m - 1 : jh - 1) * L, hjp = (jh == m - 1 ? 0 : jh + 1) * L;
  const bool has_halo = warp == 0 || warp == NW - 1;
  const bool own_row = j0 + warp < m;  // rows past m (last tile) are computed, not stored
  auto pl = [&](int p) { return static_cast<long long>(p + a.R) * a.plane; };
  auto slot = [&](int p) { return sx + ((p + 8) & 3) * PL; };
  auto k0of = [&](int c) { return c * 32 * K + lane * K; };
#define KMG(vec, row, k0) kminus<L, NS, true>(vec, row, k0, lane)
#define KPG(vec, row, k0) kplus<L, NS, true>(vec, row, k0, lane)
#define KMS(vec, row, k0) kminus<L, NS, false>(vec, row, k0, lane)
#define KPS(vec, row, k0) kplus<L, NS, false>(vec, row, k0, lane)

  // donor cell group: row r with offsets (g_, gm_, gp_) of plane p
  auto donor = [&](int p, int r, int g_, int gm_, int gp_, bool store) {
    const T* X = a.x + pl(p);
    const T* Xm = a.x + pl(p - 1);
    const T* Xp = a.x + pl(p + 1);
    const T* U = a.u + pl(p);
    const T* Up = a.u + pl(p + 1);
    const T* Vv = a.v + pl(p);
    const T* W = a.w + pl(p);
    const T* H = a.h + pl(p);
    T* dst = slot(p);
#pragma unroll
    for (int c = 0; c < NS; ++c) {
      const int k0 = k0of(c);
      const int g = g_ + k0;
      const V xc = vload<T, K>(X + g);
      const V xm = vload<T, K>(Xm + g), xp = vload<T, K>(Xp + g);
      const V ym = vload<T, K>(X + gm_ + k0), yp = vload<T, K>(X + gp_ + k0);
      const V zm = KMG(xc, X + g_, k0), zp = KPG(xc, X + g_, k0);
      const V uc = vload<T, K>(U + g), up = vload<T, K>(Up + g);
      const V vc = vload<T, K>(Vv + g), vp = vload<T, K>(Vv + gp_ + k0);
      const V wc = vload<T, K>(W + g);
      const V wp = KPG(wc, W + g_, k0);
      const V hc = vload<T, K>(H + g);
      V res;
#pragma unroll
      for (int e = 0; e < K; ++e) {
        const T x0 = xc.e[e];
        const T fxl = upflux(xm.e[e], x0, uc.e[e]);
        const T fxr = upflux(x0, xp.e[e], up.e[e]);
        const T fyl = upflux(ym.e[e], x0, vc.e[e]);
        const T fyr = upflux(x0, yp.e[e], vp.e[e]);
        const T fzl = upflux(zm.e[e], x0, wc.e[e]);
        const T fzr = upflux(x0, zp.e[e], wp.e[e]);
        const T div = ((fxr - fxl) + (fyr - fyl)) + (fzr - fzl);
        res.e[e] = x0 - qdiv(div, hc.e[e]);
      }
      vstore(dst + r * L + k0, res);
      if (store) vstore(a.x1 + pl(p) + g, res);
    }
  };
  auto stage_donor = [&](int p) {
    donor(p, warp, gj, gjm, gjp, own_row);
    if (has_halo) donor(p, hr, hj, hjm, hjp, false);
  };

  // pseudo-velocities of plane pb for this warp's row: x-face pb+1/2 (index
  // pb+1), y-face between rows r-1 and r, z-face between k-1 and k.
  auto stage_pseudo = [&](int pb, bool only_u) {
    const int r = warp;
    const T* s0 = slot(pb - 1);
    const T* s1 = slot(pb);
    const T* s2 = slot(pb + 1);
    const T* U1 = a.u + pl(pb);
    const T* U2 = a.u + pl(pb + 1);
    const T* V1 = a.v + pl(pb);
    const T* V2 = a.v + pl(pb + 1);
    const T* W1 = a.w + pl(pb);
    const T* W2 = a.w + pl(pb + 1);
    const T* H1 = a.h + pl(pb);
    const T* H2 = a.h + pl(pb + 1);
#pragma unroll
    for (int c = 0; c < NS; ++c) {
      const int k0 = k0of(c);
      const int g = gj + k0;
      const int so = r * L + k0;
      const V x1 = sload<T, K>(s1 + so);
      const V a1 = vabs(x1);
      const V a1m = vabs(sload<T, K>(s1 + so - L));
      const V u2c = vload<T, K>(U2 + g);
      const V h1c = vload<T, K>(H1 + g);
      const V a1km = vabs(KMS(x1, s1 + r * L, k0));
      {  // x-face between planes pb and pb+1 of this column
        const V x2 = sload<T, K>(s2 + so);
        const V a2 = vabs(x2);
        const V a1kp = vabs(KPS(x1, s1 + r * L, k0));
        const V a2kp = vabs(KPS(x2, s2 + r * L, k0)), a2km = vabs(KMS(x2, s2 + r * L, k0));
        V bp, bm, cp, cm, Vs, Ws;
        {
          const V a1p = vabs(sload<T, K>(s1 + so + L)), a2p = vabs(sload<T, K>(s2 + so + L));
          const V a2m = vabs(sload<T, K>(s2 + so - L));
#pragma unroll
          for (int e = 0; e < K; ++e) {
            bp.e[e] = a1p.e[e] + a2p.e[e];
            bm.e[e] = a1m.e[e] + a2m.e[e];
            cp.e[e] = a1kp.e[e] + a2kp.e[e];
            cm.e[e] = a1km.e[e] + a2km.e[e];
          }
        }
        {
          const V v1 = vload<T, K>(V1 + g), v2 = vload<T, K>(V2 + g);
          const V v1p = vload<T, K>(V1 + gjp + k0), v2p = vload<T, K>(V2 + gjp + k0);
#pragma unroll
          for (int e = 0; e < K; ++e) Vs.e[e] = (v1.e[e] + v2.e[e]) + (v1p.e[e] + v2p.e[e]);
        }
        {
          const V w1 = vload<T, K>(W1 + g), w2 = vload<T, K>(W2 + g);
          const V w1p = KPG(w1, W1 + gj, k0), w2p = KPG(w2, W2 + gj, k0);
#pragma unroll
          for (int e = 0; e < K; ++e) Ws.e[e] = (w1.e[e] + w2.e[e]) + (w1p.e[e] + w2p.e[e]);
        }
        const V h2 = vload<T, K>(H2 + g);
        V res;
#pragma unroll
        for (int e = 0; e < K; ++e)
          res.e[e] = pseudo_face<T>(u2c.e[e], h1c.e[e], h2.e[e], a2.e[e], a1.e[e], bp.e[e],
                                    bm.e[e], Vs.e[e], cp.e[e], cm.e[e], Ws.e[e]);
        if (own_row) vstore(a.ut + pl(pb + 1) + g, res);
      }
      if (only_u) continue;
      const V x0 = sload<T, K>(s0 + so);
      const V x2 = sload<T, K>(s2 + so);
      const V u1c = vload<T, K>(U1 + g);
      const V w1 = vload<T, K>(W1 + g);
      {  // y-face between rows r-1 and r of plane pb
        const V x1m = sload<T, K>(s1 + so - L);
        V bp, bm, cp, cm, Us, Ws;
        {
          const V a0m = vabs(sload<T, K>(s0 + so - L)), a2m = vabs(sload<T, K>(s2 + so - L));
          const V a1mkp = vabs(KPS(x1m, s1 + (r - 1) * L, k0));
          const V a1mkm = vabs(KMS(x1m, s1 + (r - 1) * L, k0));
          const V a1kp = vabs(KPS(x1, s1 + r * L, k0));
#pragma unroll
          for (int e = 0; e < K; ++e) {
            bp.e[e] = a2m.e[e] + fabs(x2.e[e]);
            bm.e[e] = a0m.e[e] + fabs(x0.e[e]);
            cp.e[e] = a1mkp.e[e] + a1kp.e[e];
            cm.e[e] = a1mkm.e[e] + a1km.e[e];
          }
        }
        {
          const V u1m = vload<T, K>(U1 + gjm + k0), u2m = vload<T, K>(U2 + gjm + k0);
#pragma unroll
          for (int e = 0; e < K; ++e) Us.e[e] = (u1m.e[e] + u1c.e[e]) + (u2m.e[e] + u2c.e[e]);
        }
        {
          const V w1m = vload<T, K>(W1 + gjm + k0);
          const V w1mkp = KPG(w1m, W1 + gjm, k0), w1kp = KPG(w1, W1 + gj, k0);
#pragma unroll
          for (int e = 0; e < K; ++e) Ws.e[e] = (w1m.e[e] + w1.e[e]) + (w1mkp.e[e] + w1kp.e[e]);
        }
        const V v1 = vload<T, K>(V1 + g);
        const V h1m = vload<T, K>(H1 + gjm + k0);
        V res;
#pragma unroll
        for (int e = 0; e < K; ++e)
          res.e[e] = pseudo_face<T>(v1.e[e], h1m.e[e], h1c.e[e], a1.e[e], a1m.e[e], bp.e[e],
                                    bm.e[e], Us.e[e], cp.e[e], cm.e[e], Ws.e[e]);
        if (own_row) vstore(a.vt + pl(pb) + g, res);
      }
      {  // z-face between k-1 and k
        V bp, bm, cp, cm, Us, Vs;
        {
          const V x1p = sload<T, K>(s1 + so + L);
          const V x1m = sload<T, K>(s1 + so - L);
          const V a1pkm = vabs(KMS(x1p, s1 + (r + 1) * L, k0));
          const V a1mkm = vabs(KMS(x1m, s1 + (r - 1) * L, k0));
          const V a2km = vabs(KMS(x2, s2 + r * L, k0)), a0km = vabs(KMS(x0, s0 + r * L, k0));
#pragma unroll
          for (int e = 0; e < K; ++e) {
            bp.e[e] = a2km.e[e] + fabs(x2.e[e]);
            bm.e[e] = a0km.e[e] + fabs(x0.e[e]);
            cp.e[e] = a1pkm.e[e] + fabs(x1p.e[e]);
            cm.e[e] = a1mkm.e[e] + a1m.e[e];
          }
        }
        {
          const V u2km = KMG(u2c, U2 + gj, k0), u1km = KMG(u1c, U1 + gj, k0);
#pragma unroll
          for (int e = 0; e < K; ++e) Us.e[e] = (u1km.e[e] + u1c.e[e]) + (u2km.e[e] + u2c.e[e]);
        }
        {
          const V v1 = vload<T, K>(V1 + g), v1p = vload<T, K>(V1 + gjp + k0);
          const V v1km = KMG(v1, V1 + gj, k0), v1pkm = KMG(v1p, V1 + gjp, k0);
#pragma unroll
          for (int e = 0; e < K; ++e) Vs.e[e] = (v1km.e[e] + v1.e[e]) + (v1pkm.e[e] + v1p.e[e]);
        }
        const V h1km = KMG(h1c, H1 + gj, k0);
        V res;
#pragma unroll
        for (int e = 0; e < K; ++e)
          res.e[e] = pseudo_face<T>(w1.e[e], h1km.e[e], h1c.e[e], a1.e[e], a1km.e[e], bp.e[e],
                                    bm.e[e], Us.e[e], cp.e[e], cm.e[e], Vs.e[e]);
        if (own_row) vstore(a.wt + pl(pb) + g, res);
      }
    }
  };

  // warm-up: psi^(1) of planes pa-1 .. pa+1, then the x-face pa-1/2
  stage_donor(pa - 1);
  stage_donor(pa);
  stage_donor(pa + 1);
  __syncthreads();
  stage_pseudo(pa - 1, true);
  for (int p = pa; p < pb; ++p) {
    if (a.pf > 0 && warp == 0 && lane < 5) {  // one-plane-ahead L2 prefetch of the inputs
      const int q = p + 3;
      if (q <= a.p1 + 1) {  // the last plane kernel A reads
        const T* f = lane == 0 ? a.x : lane == 1 ? a.u : lane == 2 ? a.v : lane == 3 ? a.w : a.h;
        const int rows = (RR + 4 < m ? RR + 4 : m);
        const int jj = wrapj(j0 - 2);
        const int first = (jj + rows <= m) ? rows : m - jj;
        l2_prefetch(f + pl(q) + static_cast<long long>(jj) * L, static_cast<unsigned>(first * L * sizeof(T)));
        if (first < rows)
          l2_prefetch(f + pl(q), static_cast<unsigned>((rows - first) * L * sizeof(T)));
      }
    }
    stage_pseudo(p, false);
    if (p + 2 <= pb) stage_donor(p + 2);
    __syncthreads();
  }
#undef KMG
#undef KPG
#undef KMS
#undef KPS
}

// ---- kernel B ------------------------------------------------------------
template <class T, int L, int NW, int NS>
__global__ void __launch_bounds__(NW * 32, 1) k_split_b(ArgsB<T> a) {
  constexpr int K = L / (32 * NS), RR = NW, PL = RR * L, TJ = RR - 2;
  using V = Vec<T, K>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* const sm = reinterpret_cast<T*>(smem_raw);
  T* const s_bu = sm;           // beta up,   2 planes
  T* const s_bd = sm + 2 * PL;  // beta down, 2 planes
  T* const s_vl = sm + 4 * PL;  // limited y-face velocity, 2 planes
  T* const s_wl = sm + 6 * PL;  // limited z-face velocity, 2 planes

  const int nbig = a.ntj * a.kseg;
  const bool big = static_cast<int>(blockIdx.x) < nbig;
  const int tile = big ? blockIdx.x % a.ntj : blockIdx.x - nbig;
  const int ib = a.o0 + (big ? static_cast<int>(blockIdx.x / a.ntj) * a.lseg : a.kseg * a.lseg);
  const int ie = big ? ib + a.lseg : a.o1;
  if (ib >= ie) return;
  const int m = a.m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = warp;  // region row; j = j0 - 1 + r, output rows 1 .. RR-2
  const int j0 = tile * TJ;
  const int jr = ((j0 - 1 + r) % m + m) % m;
  const int gj = jr * L, gjm = (jr == 0 ? m - 1 : jr - 1) * L, gjp = (jr == m - 1 ? 0 : jr + 1) * L;
  const bool out_row = r >= 1 && r < RR - 1 && j0 - 1 + r < m;
  auto pl = [&](int p) { return static_cast<long long>(p + a.R) * a.plane; };
  auto k0of = [&](int c) { return c * 32 * K + lane * K; };
#define KMG(vec, row, k0) kminus<L, NS, true>(vec, row, k0, lane)
#define KPG(vec, row, k0) kplus<L, NS, true>(vec, row, k0, lane)
#define KMS(vec, row, k0) kminus<L, NS, false>(vec, row, k0, lane)
#define KPS(vec, row, k0) kplus<L, NS, false>(vec, row, k0, lane)

  V fxc[NS];
#pragma unroll
  for (int c = 0; c < NS; ++c)
#pragma unroll
    for (int e = 0; e < K; ++e) fxc[c].e[e] = T(0);

  for (int t = ib - 2; t < ie; ++t) {
    const int p1 = t + 1;
    T* buA = s_bu + (p1 & 1) * PL;
    T* bdA = s_bd + (p1 & 1) * PL;
    // ---- phase 1: 7-point bounds and beta of plane t+1 (every region row)
    {
      const T* X1c = a.x1 + pl(p1);
      const T* X10 = a.x1 + pl(t);
      const T* X12 = a.x1 + pl(t + 2);
      const T* Xn1 = a.x + pl(p1);
      const T* Xn0 = a.x + pl(t);
      const T* Xn2 = a.x + pl(t + 2);
      const T* Ul = a.ut + pl(p1);      // x-face t+1/2
      const T* Ur = a.ut + pl(t + 2);   // x-face t+3/2
      const T* Vt = a.vt + pl(p1);
      const T* Wt = a.wt + pl(p1);
      const T* H1 = a.h + pl(p1);
#pragma unroll
      for (int c = 0; c < NS; ++c) {
        const int k0 = k0of(c);
        const int g = gj + k0;
        const V xc = vload<T, K>(X1c + g);
        const V xm = vload<T, K>(X10 + g), xp = vload<T, K>(X12 + g);
        const V ym = vload<T, K>(X1c + gjm + k0), yp = vload<T, K>(X1c + gjp + k0);
        const V zm = KMG(xc, X1c + gj, k0), zp = KPG(xc, X1c + gj, k0);
        V mx, mn;
        {
          const V nc = vload<T, K>(Xn1 + g);
          const V n0 = vload<T, K>(Xn0 + g), n2 = vload<T, K>(Xn2 + g);
          const V nym = vload<T, K>(Xn1 + gjm + k0), nyp = vload<T, K>(Xn1 + gjp + k0);
          const V nzm = KMG(nc, Xn1 + gj, k0), nzp = KPG(nc, Xn1 + gj, k0);
#pragma unroll
          for (int e = 0; e < K; ++e) {
            mx.e[e] = tmax(tmax(tmax(nc.e[e], n0.e[e]), tmax(n2.e[e], nym.e[e])),
                           tmax(tmax(nyp.e[e], nzm.e[e]), nzp.e[e]));
            mn.e[e] = tmin(tmin(tmin(nc.e[e], n0.e[e]), tmin(n2.e[e], nym.e[e])),
                           tmin(tmin(nyp.e[e], nzm.e[e]), nzp.e[e]));
          }
        }
        const V ul = vload<T, K>(Ul + g), ur = vload<T, K>(Ur + g);
        const V va = vload<T, K>(Vt + g), vap = vload<T, K>(Vt + gjp + k0);
        const V wa = vload<T, K>(Wt + g);
        const V wap = KPG(wa, Wt + gj, k0);
        const V hc = vload<T, K>(H1 + g);
        V bu, bd;
#pragma unroll
        for (int e = 0; e < K; ++e) {
          const T x0 = xc.e[e];
          const T hi = tmax(tmax(tmax(mx.e[e], x0), tmax(xm.e[e], xp.e[e])),
                            tmax(tmax(ym.e[e], yp.e[e]), tmax(zm.e[e], zp.e[e])));
          const T lo = tmin(tmin(tmin(mn.e[e], x0), tmin(xm.e[e], xp.e[e])),
                            tmin(tmin(ym.e[e], yp.e[e]), tmin(zm.e[e], zp.e[e])));
          const T axl = upflux(xm.e[e], x0, ul.e[e]);
          const T axr = upflux(x0, xp.e[e], ur.e[e]);
          const T ayl = upflux(ym.e[e], x0, va.e[e]);
          const T ayr = upflux(x0, yp.e[e], vap.e[e]);
          const T azl = upflux(zm.e[e], x0, wa.e[e]);
          const T azr = upflux(x0, zp.e[e], wap.e[e]);
          const T fin2 = (((axl + fabs(axl)) + (fabs(axr) - axr)) +
                          ((ayl + fabs(ayl)) + (fabs(ayr) - ayr))) +
                         ((azl + fabs(azl)) + (fabs(azr) - azr));
          const T fout2 = (((axr + fabs(axr)) + (fabs(axl) - axl)) +
                           ((ayr + fabs(ayr)) + (fabs(ayl) - ayl))) +
                          ((azr + fabs(azr)) + (fabs(azl) - azl));
          const T di = T(0.5) * fin2 + Eps<T>::value, dou = T(0.5) * fout2 + Eps<T>::value;
          if constexpr (sizeof(T) == 8) {
            const T rr2 = rcp(di * dou);
            bu.e[e] = ((hi - x0) * hc.e[e]) * dou * rr2;
            bd.e[e] = ((x0 - lo) * hc.e[e]) * di * rr2;
          } else {
            bu.e[e] = qdiv((hi - x0) * hc.e[e], di);
            bd.e[e] = qdiv((x0 - lo) * hc.e[e], dou);
          }
        }
        vstore(buA + r * L + k0, bu);
        vstore(bdA + r * L + k0, bd);
      }
    }
    __syncthreads();
    // ---- phase 2: limit plane t+1 velocities; final update of plane t
    if (r >= 1) {
      const T* buB = s_bu + (t & 1) * PL;  // beta, plane t
      const T* bdB = s_bd + (t & 1) * PL;
      T* vlA = s_vl + (p1 & 1) * PL;
      T* wlA = s_wl + (p1 & 1) * PL;
      const T* vlB = s_vl + (t & 1) * PL;  // limited, plane t
      const T* wlB = s_wl + (t & 1) * PL;
      const T* Vt = a.vt + pl(p1);
      const T* Wt = a.wt + pl(p1);
      const T* Ul = a.ut + pl(p1);
      const T* X10 = a.x1 + pl(t);
      const T* X11 = a.x1 + pl(p1);
      const T* H0 = a.h + pl(t);
      T* O = a.out + pl(t);
#pragma unroll
      for (int c = 0; c < NS; ++c) {
        const int k0 = k0of(c);
        const int g = gj + k0;
        const int so = r * L + k0;
        const V bu = sload<T, K>(buA + so), bd = sload<T, K>(bdA + so);
        {
          const V va = vload<T, K>(Vt + g);
          const V bum = sload<T, K>(buA + so - L), bdm = sload<T, K>(bdA + so - L);
          V res;
#pragma unroll
          for (int e = 0; e < K; ++e)
            res.e[e] = limit_sel(va.e[e], bdm.e[e], bu.e[e], bum.e[e], bd.e[e]);
          vstore(vlA + so, res);
        }
        if (r >= RR - 1) continue;
        V fxr;
        {
          const V wa = vload<T, K>(Wt + g);
          const V bukm = KMS(bu, buA + r * L, k0), bdkm = KMS(bd, bdA + r * L, k0);
          const V buo = sload<T, K>(buB + so), bdo = sload<T, K>(bdB + so);
          const V ul = vload<T, K>(Ul + g);
          const V xc = vload<T, K>(X10 + g);
          const V x1 = vload<T, K>(X11 + g);
          V wres;
#pragma unroll
          for (int e = 0; e < K; ++e) {
            wres.e[e] = limit_sel(wa.e[e], bdkm.e[e], bu.e[e], bukm.e[e], bd.e[e]);
            const T ulim = limit_sel(ul.e[e], bdo.e[e], bu.e[e], buo.e[e], bd.e[e]);
            fxr.e[e] = upflux(xc.e[e], x1.e[e], ulim);
          }
          vstore(wlA + so, wres);
        }
        if (t >= ib) {
          const V xc = vload<T, K>(X10 + g);
          const V ym = vload<T, K>(X10 + gjm + k0), yp = vload<T, K>(X10 + gjp + k0);
          const V zm = KMG(xc, X10 + gj, k0), zp = KPG(xc, X10 + gj, k0);
          const V vb = sload<T, K>(vlB + so), vbp = sload<T, K>(vlB + so + L);
          const V wb = sload<T, K>(wlB + so);
          const V wbp = KPS(wb, wlB + r * L, k0);
          const V hc = vload<T, K>(H0 + g);
          V res;
#pragma unroll
          for (int e = 0; e < K; ++e) {
            const T x0 = xc.e[e];
            const T fyl = upflux(ym.e[e], x0, vb.e[e]);
            const T fyr = upflux(x0, yp.e[e], vbp.e[e]);
            const T fzl = upflux(zm.e[e], x0, wb.e[e]);
            const T fzr = upflux(x0, zp.e[e], wbp.e[e]);
            const T div = ((fxr.e[e] - fxc[c].e[e]) + (fyr - fyl)) + (fzr - fzl);
            res.e[e] = x0 - qdiv(div, hc.e[e]);
          }
          if (out_row) vstore(O + g, res);
        }
        fxc[c] = fxr;
      }
    }
    __syncthreads();
  }
  // halo push epilogue (as in k_fused): output planes t < R and t >= ni - R
  if (a.push_lo != nullptr || a.push_hi != nullptr) {
    const int tl = (ib > 0 ? ib : 0), th = (ie < a.R ? ie : a.R);
    const int ul = (ib > a.ni - a.R ? ib : a.ni - a.R), uh = ie;
    for (int pass = 0; pass < 2; ++pass) {
      const int q0 = pass == 0 ? tl : ul, q1 = pass == 0 ? th : uh;
      T* dstb = pass == 0 ? a.push_lo : a.push_hi;
      if (dstb == nullptr || !out_row) continue;
      for (int t = q0; t < q1; ++t) {
        const long long dplane = pass == 0 ? static_cast<long long>(a.R + a.lo_ni + t)
                                           : static_cast<long long>(a.R + t - a.ni);
#pragma unroll
        for (int c = 0; c < NS; ++c) {
          const int g = gj + k0of(c);
          vstore(dstb + dplane * a.plane + g, vload<T, K>(a.out + pl(t) + g));
        }
      }
    }
  }
#undef KMG
#undef KPG
#undef KMS
#undef KPS
}

template <class T, int L, int NW, int NS>
int launch_split_cfg(const FusedShape& fs, const T* x, const T* u, const T* v, const T* w,
                     const T* h, T* x1, T* ut, T* vt, T* wt, T* out, int num_sms,
                     cudaStream_t st, const HaloPush<T>& push) {
  auto ka = k_split_a<T, L, NW, NS>;
  auto kb = k_split_b<T, L, NW, NS>;
  constexpr std::size_t smem_a = sizeof(T) * 4 * (NW + 2) * L;
  constexpr std::size_t smem_b = sizeof(T) * 8 * NW * L;
  static bool configured = false;
  static int per_a = 1, per_b = 1;
  if (!configured) {
    cudaFuncSetAttribute(ka, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_a));
    cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_b));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_a, ka, NW * 32, smem_a);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_b, kb, NW * 32, smem_b);
    per_a = std::max(per_a, 1);
    per_b = std::max(per_b, 1);
    configured = true;
  }
  // kernel A: pseudo-velocities on [o0-1, o1+1), psi1 on [o0-2, o1+1]
  ArgsA<T> aa{x, u, v, w, h, x1, ut, vt, wt, static_cast<int>(fs.m), static_cast<int>(fs.R),
              0, 0, 0, static_cast<int>(fs.o0 - 1), static_cast<int>(fs.o1 + 1), fs.m * fs.l, 1};
  const Plan pa = plan_grid(fs.m, NW, aa.p1 - aa.p0, per_a * num_sms, 3);
  aa.ntj = pa.ntj;
  aa.kseg = pa.kseg;
  aa.lseg = pa.lseg;
  ka<<<pa.blocks, NW * 32, smem_a, st>>>(aa);
  ArgsB<T> ab{x, h, x1, ut, vt, wt, out, static_cast<int>(fs.m), static_cast<int>(fs.R), 0, 0, 0,
              static_cast<int>(fs.o0), static_cast<int>(fs.o1), fs.m * fs.l, push.lo, push.hi,
              static_cast<int>(push.lo_ni), static_cast<int>(fs.ni)};
  const Plan pb = plan_grid(fs.m, NW - 2, fs.o1 - fs.o0, per_b * num_sms, 2);
  ab.ntj = pb.ntj;
  ab.kseg = pb.kseg;
  ab.lseg = pb.lseg;
  kb<<<pb.blocks, NW * 32, smem_b, st>>>(ab);
  return 2;
}

}  // namespace

bool split_supported(int iord, int nonos, std::int64_t m, std::int64_t l) {
  return iord == 2 && nonos && l == 128 && m >= 3 && m < (1 << 20);
}

template <class T>
int launch_split(const FusedShape& fs, const T* x, const T* u, const T* v, const T* w,
                 const T* h, T* x1, T* ut, T* vt, T* wt, T* out, int num_sms, cudaStream_t st,
                 const HaloPush<T>& push) {
  if (fs.l != 128) return 0;
  constexpr int NS = sizeof(T) == 8 ? 2 : 1;
  return launch_split_cfg<T, 128, 16, NS>(fs, x, u, v, w, h, x1, ut, vt, wt, out, num_sms, st,
                                          push);
}

template int launch_split<double>(const FusedShape&, const double*, const double*, const double*,
                                  const double*, const double*, double*, double*, double*,
                                  double*, double*, int, cudaStream_t, const HaloPush<double>&);
template int launch_split<float>(const FusedShape&, const float*, const float*, const float*,
                                 const float*, const float*, float*, float*, float*, float*,
                                 float*, int, cudaStream_t, const HaloPush<float>&);

}  // namespace imb::dev
