// Staged MPDATA kernels: one launch per stage group, every intermediate in
// HBM. They are the general-purpose path (any grid, any plane range) used
// for slab boundary planes, grids too thin for the fused streaming kernel,
// and as the structural cross-check of the fused kernel in tests.
//
// Device layout of every field (a "padded slab"): planes p in [0, ni + 2R),
// local i = p - R, each plane m*l values with k contiguous — the interior
// order of GridField::index (workload.hpp:40-43) with halos only along the
// slab axis. j and k are periodic and wrap by index arithmetic.
#include <cuda_runtime.h>

#include "mpdata_kernels.cuh"
#include "mpdata_math.cuh"

namespace imb::dev {

namespace {

struct Cell {
  std::int64_t p, j, k, jm, jp, km, kp;
};

__device__ __forceinline__ bool locate(const Span& s, Cell& c) {
  const std::int64_t t = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const std::int64_t plane = s.m * s.l;
  if (t >= (s.p1 - s.p0) * plane) return false;
  c.p = s.p0 + t / plane;
  const std::int64_t r = t % plane;
  c.j = r / s.l;
  c.k = r % s.l;
  c.jm = c.j == 0 ? s.m - 1 : c.j - 1;
  c.jp = c.j == s.m - 1 ? 0 : c.j + 1;
  c.km = c.k == 0 ? s.l - 1 : c.k - 1;
  c.kp = c.k == s.l - 1 ? 0 : c.k + 1;
  return true;
}

__device__ __forceinline__ std::int64_t at(const Span& s, std::int64_t p, std::int64_t j,
                                           std::int64_t k) {
  return (p * s.m + j) * s.l + k;
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
  const std::int64_t o = at(s, c.p, c.j, c.k);
  const T xc = x[o];
  const std::int64_t ox = at(s, c.p + 1, c.j, c.k), oy = at(s, c.p, c.jp, c.k),
                     oz = at(s, c.p, c.j, c.kp);
  const T fxl = flux(x[at(s, c.p - 1, c.j, c.k)], xc, U[o]);
  const T fxr = flux(xc, x[ox], U[ox]);
  const T fyl = flux(x[at(s, c.p, c.jm, c.k)], xc, V[o]);
  const T fyr = flux(xc, x[oy], V[oy]);
  const T fzl = flux(x[at(s, c.p, c.j, c.km)], xc, W[o]);
  const T fzr = flux(xc, x[oz], W[oz]);
  const T div = ((fxr - fxl) + (fyr - fyl)) + (fzr - fzl);
  out[o] = xc - div / h[o];
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
  const std::int64_t p = c.p, j = c.j, k = c.k, pm = p - 1, pp = p + 1;
  const std::int64_t o = at(s, p, j, k);
  auto ax = [&](std::int64_t a, std::int64_t b, std::int64_t d) { return fabs(x[at(s, a, b, d)]); };
  const T ac = fabs(x[o]);
  const T hc = h[o];
  {  // x-face (i-1/2)
    const T Un = U[o];
    const T hb = T(0.5) * (h[at(s, pm, j, k)] + hc);
    const T A = ratio(ac, ax(pm, j, k));
    const T B = ratio(ax(pm, c.jp, k) + ax(p, c.jp, k), ax(pm, c.jm, k) + ax(p, c.jm, k));
    const T C = ratio(ax(pm, j, c.kp) + ax(p, j, c.kp), ax(pm, j, c.km) + ax(p, j, c.km));
    const T Vs = (V[at(s, pm, j, k)] + V[o]) + (V[at(s, pm, c.jp, k)] + V[at(s, p, c.jp, k)]);
    const T Ws = (W[at(s, pm, j, k)] + W[o]) + (W[at(s, pm, j, c.kp)] + W[at(s, p, j, c.kp)]);
    ut[o] = pseudo(Un, hb, A, Vs, B, Ws, C);
  }
  {  // y-face (j-1/2)
    const T Vn = V[o];
    const T hb = T(0.5) * (h[at(s, p, c.jm, k)] + hc);
    const T A = ratio(ac, ax(p, c.jm, k));
    const T B = ratio(ax(pp, c.jm, k) + ax(pp, j, k), ax(pm, c.jm, k) + ax(pm, j, k));
    const T C = ratio(ax(p, c.jm, c.kp) + ax(p, j, c.kp), ax(p, c.jm, c.km) + ax(p, j, c.km));
    const T Us = (U[at(s, p, c.jm, k)] + U[o]) + (U[at(s, pp, c.jm, k)] + U[at(s, pp, j, k)]);
    const T Ws = (W[at(s, p, c.jm, k)] + W[o]) + (W[at(s, p, c.jm, c.kp)] + W[at(s, p, j, c.kp)]);
    vt[o] = pseudo(Vn, hb, A, Us, B, Ws, C);
  }
  {  // z-face (k-1/2)
    const T Wn = W[o];
    const T hb = T(0.5) * (h[at(s, p, j, c.km)] + hc);
    const T A = ratio(ac, ax(p, j, c.km));
    const T B = ratio(ax(pp, j, c.km) + ax(pp, j, k), ax(pm, j, c.km) + ax(pm, j, k));
    const T C = ratio(ax(p, c.jp, c.km) + ax(p, c.jp, k), ax(p, c.jm, c.km) + ax(p, c.jm, k));
    const T Us = (U[at(s, p, j, c.km)] + U[o]) + (U[at(s, pp, j, c.km)] + U[at(s, pp, j, k)]);
    const T Vs = (V[at(s, p, j, c.km)] + V[o]) + (V[at(s, p, c.jp, c.km)] + V[at(s, p, c.jp, k)]);
    wt[o] = pseudo(Wn, hb, A, Us, B, Vs, C);
  }
}

template <class T>
__device__ __forceinline__ void ext7(const Span& s, const T* __restrict__ x, const Cell& c,
                                     T& hi, T& lo) {
  const T v[7] = {x[at(s, c.p, c.j, c.k)],  x[at(s, c.p - 1, c.j, c.k)], x[at(s, c.p + 1, c.j, c.k)],
                  x[at(s, c.p, c.jm, c.k)], x[at(s, c.p, c.jp, c.k)],    x[at(s, c.p, c.j, c.km)],
                  x[at(s, c.p, c.j, c.kp)]};
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
  const std::int64_t o = at(s, c.p, c.j, c.k);
  T hi, lo;
  ext7(s, x, c, hi, lo);
  if (first) {
    T h2, l2;
    ext7(s, xn, c, h2, l2);
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
  const std::int64_t o = at(s, c.p, c.j, c.k);
  const std::int64_t ox = at(s, c.p + 1, c.j, c.k), oy = at(s, c.p, c.jp, c.k),
                     oz = at(s, c.p, c.j, c.kp);
  const T xc = x[o];
  const T axl = flux(x[at(s, c.p - 1, c.j, c.k)], xc, ut[o]);
  const T axr = flux(xc, x[ox], ut[ox]);
  const T ayl = flux(x[at(s, c.p, c.jm, c.k)], xc, vt[o]);
  const T ayr = flux(xc, x[oy], vt[oy]);
  const T azl = flux(x[at(s, c.p, c.j, c.km)], xc, wt[o]);
  const T azr = flux(xc, x[oz], wt[oz]);
  const T fin = ((pos(axl) - neg(axr)) + (pos(ayl) - neg(ayr))) + (pos(azl) - neg(azr));
  const T fout = ((pos(axr) - neg(axl)) + (pos(ayr) - neg(ayl))) + (pos(azr) - neg(azl));
  const T hc = h[o];
  bu[o] = ((mx[o] - xc) * hc) / (fin + Eps<T>::value);
  bd[o] = ((xc - mn[o]) * hc) / (fout + Eps<T>::value);
}

// Limit the pseudo-velocities in place.
template <class T>
__global__ void __launch_bounds__(256) k_limit(Span s, T* __restrict__ ut, T* __restrict__ vt,
                                               T* __restrict__ wt, const T* __restrict__ bu,
                                               const T* __restrict__ bd) {
  Cell c;
  if (!locate(s, c)) return;
  const std::int64_t o = at(s, c.p, c.j, c.k);
  const T buc = bu[o], bdc = bd[o];
  std::int64_t L = at(s, c.p - 1, c.j, c.k);
  ut[o] = limit(ut[o], bd[L], buc, bu[L], bdc);
  L = at(s, c.p, c.jm, c.k);
  vt[o] = limit(vt[o], bd[L], buc, bu[L], bdc);
  L = at(s, c.p, c.j, c.km);
  wt[o] = limit(wt[o], bd[L], buc, bu[L], bdc);
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
IMB_INSTANTIATE(double)
IMB_INSTANTIATE(float)
#undef IMB_INSTANTIATE

}  // namespace imb::dev
