// Staged MPDATA kernels: one launch per stage group, every intermediate in
// HBM. They are the general path (any IORD — config 5's IORD=3 — and any
// plane extent l), and the structural cross-check of the fused kernel.
//
// Device layout of every field (a "padded slab"): planes p in [0, ni + 2R),
// local i = p - R, each plane m*l values with k contiguous — the interior
// order of GridField::index (workload.hpp:40-43) with halos only along the
// slab axis. j and k are periodic and wrap by index arithmetic. The per-cell
// arithmetic is the fused kernel's (mpdata_math.cuh): exact select forms,
// one reciprocal per pseudo-velocity and per beta pair.
#include <cuda_runtime.h>

#include "mpdata_kernels.cuh"
#include "mpdata_math.cuh"

namespace imb::dev {

namespace {

// A cell of the launch span: plane base offset (64-bit) and in-plane offsets
// of the cell and its periodic j/k neighbours (32-bit).
struct Cell {
  long long base;  // p * plane
  long long plane;
  int o, ojm, ojp, okm, okp;
};

__device__ __forceinline__ bool locate(const Span& s, Cell& c) {
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int m = static_cast<int>(s.m), l = static_cast<int>(s.l);
  const long long plane = static_cast<long long>(m) * l;
  if (t >= (s.p1 - s.p0) * plane) return false;
  const long long p = s.p0 + t / plane;
  const int r = static_cast<int>(t - (p - s.p0) * plane);
  const int j = r / l, k = r - j * l;
  c.base = p * plane;
  c.plane = plane;
  c.o = r;
  c.ojm = (j == 0 ? r + (m - 1) * l : r - l);
  c.ojp = (j == m - 1 ? r - (m - 1) * l : r + l);
  c.okm = (k == 0 ? r + l - 1 : r - 1);
  c.okp = (k == l - 1 ? r - (l - 1) : r + 1);
  return true;
}

// out = x - div F(x, (U,V,W)) / h   (donor cell, and every corrective update)
template <class T>
__global__ void __launch_bounds__(256) k_update(Span s, const T* __restrict__ x,
                                                const T* __restrict__ U,
                                                const T* __restrict__ V,
                                                const T* __restrict__ W,
                                                const T* __restrict__ h, T* __restrict__ out) {
  Cell c;
  if (!locate(s, c)) return;
  const T* X = x + c.base;
  const T* Ub = U + c.base;
  const T* Vb = V + c.base;
  const T* Wb = W + c.base;
  const T xc = X[c.o];
  const T fxl = upflux(X[c.o - c.plane], xc, Ub[c.o]);
  const T fxr = upflux(xc, X[c.o + c.plane], Ub[c.o + c.plane]);
  const T fyl = upflux(X[c.ojm], xc, Vb[c.o]);
  const T fyr = upflux(xc, X[c.ojp], Vb[c.ojp]);
  const T fzl = upflux(X[c.okm], xc, Wb[c.o]);
  const T fzr = upflux(xc, X[c.okp], Wb[c.okp]);
  const T div = ((fxr - fxl) + (fyr - fyl)) + (fzr - fzl);
  out[c.base + c.o] = xc - qdiv(div, h[c.base + c.o]);
}

// Antidiffusive pseudo-velocities on all three face families.
template <class T>
__global__ void __launch_bounds__(256) k_pseudo(Span s, const T* __restrict__ x,
                                                const T* __restrict__ U,
                                                const T* __restrict__ V,
                                                const T* __restrict__ W,
                                                const T* __restrict__ h, T* __restrict__ ut,
                                                T* __restrict__ vt, T* __restrict__ wt) {
  Cell c;
  if (!locate(s, c)) return;
  const long long P = c.plane;
  const T* X = x + c.base;  // plane p; X - P is p-1, X + P is p+1
  const T* Ub = U + c.base;
  const T* Vb = V + c.base;
  const T* Wb = W + c.base;
  const T* Hb = h + c.base;
  const int o = c.o;
  // in-plane offsets of the diagonal neighbours
  const int ojmkp = c.ojm + (c.okp - o), ojmkm = c.ojm + (c.okm - o);
  const int ojpkm = c.ojp + (c.okm - o);
  auto A = [&](long long off) { return fabs(X[off]); };
  const T ac = A(o);
  const T hc = Hb[o];
  {  // x-face (i-1/2)
    const T Vs = (Vb[o - P] + Vb[o]) + (Vb[c.ojp - P] + Vb[c.ojp]);
    const T Ws = (Wb[o - P] + Wb[o]) + (Wb[c.okp - P] + Wb[c.okp]);
    ut[c.base + o] = pseudo_face<T>(Ub[o], Hb[o - P], hc, ac, A(o - P), A(c.ojp - P) + A(c.ojp),
                                    A(c.ojm - P) + A(c.ojm), Vs, A(c.okp - P) + A(c.okp),
                                    A(c.okm - P) + A(c.okm), Ws);
  }
  {  // y-face (j-1/2)
    const T Us = (Ub[c.ojm] + Ub[o]) + (Ub[c.ojm + P] + Ub[o + P]);
    const T Ws = (Wb[c.ojm] + Wb[o]) + (Wb[ojmkp] + Wb[c.okp]);
    vt[c.base + o] = pseudo_face<T>(Vb[o], Hb[c.ojm], hc, ac, A(c.ojm), A(c.ojm + P) + A(o + P),
                                    A(c.ojm - P) + A(o - P), Us, A(ojmkp) + A(c.okp),
                                    A(ojmkm) + A(c.okm), Ws);
  }
  {  // z-face (k-1/2)
    const T Us = (Ub[c.okm] + Ub[o]) + (Ub[c.okm + P] + Ub[o + P]);
    const T Vs = (Vb[c.okm] + Vb[o]) + (Vb[ojpkm] + Vb[c.ojp]);
    wt[c.base + o] = pseudo_face<T>(Wb[o], Hb[c.okm], hc, ac, A(c.okm), A(c.okm + P) + A(o + P),
                                    A(c.okm - P) + A(o - P), Us, A(ojpkm) + A(c.ojp),
                                    A(ojmkm) + A(c.ojm), Vs);
  }
}

template <class T>
__device__ __forceinline__ void ext7(const T* X, long long P, const Cell& c, T& hi, T& lo) {
  const T v[7] = {X[c.o], X[c.o - P], X[c.o + P], X[c.ojm], X[c.ojp], X[c.okm], X[c.okp]};
  hi = v[0];
  lo = v[0];
#pragma unroll
  for (int q = 1; q < 7; ++q) {
    hi = tmax(hi, v[q]);
    lo = tmin(lo, v[q]);
  }
}

// Nonoscillatory bounds; `first` folds in psi^n (first corrective pass).
template <class T>
__global__ void __launch_bounds__(256) k_bounds(Span s, const T* __restrict__ x,
                                                const T* __restrict__ xn, int first,
                                                T* __restrict__ mx, T* __restrict__ mn) {
  Cell c;
  if (!locate(s, c)) return;
  const long long o = c.base + c.o;
  T hi, lo;
  ext7(x + c.base, c.plane, c, hi, lo);
  if (first) {
    T h2, l2;
    ext7(xn + c.base, c.plane, c, h2, l2);
    hi = tmax(hi, h2);
    lo = tmin(lo, l2);
  } else {
    hi = tmax(hi, mx[o]);
    lo = tmin(lo, mn[o]);
  }
  mx[o] = hi;
  mn[o] = lo;
}

template <class T>
__global__ void __launch_bounds__(256) k_beta(Span s, const T* __restrict__ x,
                                              const T* __restrict__ ut,
                                              const T* __restrict__ vt,
                                              const T* __restrict__ wt,
                                              const T* __restrict__ h,
                                              const T* __restrict__ mx,
                                              const T* __restrict__ mn, T* __restrict__ bu,
                                              T* __restrict__ bd) {
  Cell c;
  if (!locate(s, c)) return;
  const long long P = c.plane;
  const T* X = x + c.base;
  const T* Ut = ut + c.base;
  const T* Vt = vt + c.base;
  const T* Wt = wt + c.base;
  const int o = c.o;
  const T xc = X[o];
  const T axl = upflux(X[o - P], xc, Ut[o]);
  const T axr = upflux(xc, X[o + P], Ut[o + P]);
  const T ayl = upflux(X[c.ojm], xc, Vt[o]);
  const T ayr = upflux(xc, X[c.ojp], Vt[c.ojp]);
  const T azl = upflux(X[c.okm], xc, Wt[o]);
  const T azr = upflux(xc, X[c.okp], Wt[c.okp]);
  // 2*pos(f) = f + |f|, -2*neg(f) = |f| - f: exact, so these are 2*fin, 2*fout.
  const T fin2 = (((axl + fabs(axl)) + (fabs(axr) - axr)) + ((ayl + fabs(ayl)) + (fabs(ayr) - ayr))) +
                 ((azl + fabs(azl)) + (fabs(azr) - azr));
  const T fout2 = (((axr + fabs(axr)) + (fabs(axl) - axl)) + ((ayr + fabs(ayr)) + (fabs(ayl) - ayl))) +
                  ((azr + fabs(azr)) + (fabs(azl) - azl));
  const long long g = c.base + o;
  const T hc = h[g];
  const T di = T(0.5) * fin2 + Eps<T>::value, dou = T(0.5) * fout2 + Eps<T>::value;
  if constexpr (sizeof(T) == 8) {
    const T r = rcp(di * dou);
    bu[g] = ((mx[g] - xc) * hc) * dou * r;
    bd[g] = ((xc - mn[g]) * hc) * di * r;
  } else {
    bu[g] = qdiv((mx[g] - xc) * hc, di);
    bd[g] = qdiv((xc - mn[g]) * hc, dou);
  }
}

// Limit the pseudo-velocities in place.
template <class T>
__global__ void __launch_bounds__(256) k_limit(Span s, T* __restrict__ ut, T* __restrict__ vt,
                                               T* __restrict__ wt, const T* __restrict__ bu,
                                               const T* __restrict__ bd) {
  Cell c;
  if (!locate(s, c)) return;
  const long long P = c.plane;
  const T* Bu = bu + c.base;
  const T* Bd = bd + c.base;
  const int o = c.o;
  const long long g = c.base + o;
  const T buc = Bu[o], bdc = Bd[o];
  ut[g] = limit_sel(ut[g], Bd[o - P], buc, Bu[o - P], bdc);
  vt[g] = limit_sel(vt[g], Bd[c.ojm], buc, Bu[c.ojm], bdc);
  wt[g] = limit_sel(wt[g], Bd[c.okm], buc, Bu[c.okm], bdc);
}

unsigned blocks_for(const Span& s) {
  const std::int64_t cells = (s.p1 - s.p0) * s.m * s.l;
  return static_cast<unsigned>((cells + 255) / 256);
}

}  // namespace

template <class T>
int launch_update(const Span& s, const T* x, const T* U, const T* V, const T* W, const T* h,
                  T* out, cudaStream_t st) {
  if (s.p1 <= s.p0) return 0;
  k_update<T><<<blocks_for(s), 256, 0, st>>>(s, x, U, V, W, h, out);
  return 1;
}

template <class T>
int launch_pseudo(const Span& s, const T* x, const T* U, const T* V, const T* W, const T* h,
                  T* ut, T* vt, T* wt, cudaStream_t st) {
  if (s.p1 <= s.p0) return 0;
  k_pseudo<T><<<blocks_for(s), 256, 0, st>>>(s, x, U, V, W, h, ut, vt, wt);
  return 1;
}

template <class T>
int launch_bounds(const Span& s, const T* x, const T* xn, int first, T* mx, T* mn,
                  cudaStream_t st) {
  if (s.p1 <= s.p0) return 0;
  k_bounds<T><<<blocks_for(s), 256, 0, st>>>(s, x, xn, first, mx, mn);
  return 1;
}

template <class T>
int launch_beta(const Span& s, const T* x, const T* ut, const T* vt, const T* wt, const T* h,
                const T* mx, const T* mn, T* bu, T* bd, cudaStream_t st) {
  if (s.p1 <= s.p0) return 0;
  k_beta<T><<<blocks_for(s), 256, 0, st>>>(s, x, ut, vt, wt, h, mx, mn, bu, bd);
  return 1;
}

template <class T>
int launch_limit(const Span& s, T* ut, T* vt, T* wt, const T* bu, const T* bd, cudaStream_t st) {
  if (s.p1 <= s.p0) return 0;
  k_limit<T><<<blocks_for(s), 256, 0, st>>>(s, ut, vt, wt, bu, bd);
  return 1;
}

#define IMB_INSTANTIATE(T)                                                                        \
  template int launch_update<T>(const Span&, const T*, const T*, const T*, const T*, const T*,   \
                                T*, cudaStream_t);                                               \
  template int launch_pseudo<T>(const Span&, const T*, const T*, const T*, const T*, const T*,   \
                                T*, T*, T*, cudaStream_t);                                       \
  template int launch_bounds<T>(const Span&, const T*, const T*, int, T*, T*, cudaStream_t);     \
  template int launch_beta<T>(const Span&, const T*, const T*, const T*, const T*, const T*,     \
                              const T*, const T*, T*, T*, cudaStream_t);                         \
  template int launch_limit<T>(const Span&, T*, T*, T*, const T*, const T*, cudaStream_t);
// Each precision is its own object (Makefile): fp32 is built with
// --fmad=false so it rounds exactly like the oracle (mpdata_math.cuh).
#ifndef IMB_ONLY_F32
IMB_INSTANTIATE(double)
#endif
#ifndef IMB_ONLY_F64
IMB_INSTANTIATE(float)
#endif
#undef IMB_INSTANTIATE

}  // namespace imb::dev
