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

#include "mpdata_kernels.cuh"
#include "mpdata_math.cuh"

namespace imb::dev {

namespace {

template <class T, int L, int RW, int NW, bool NONOS>
struct Cfg {
  static constexpr int KPL = L / 32;              // k values per lane
  static constexpr int Q = RW * KPL;              // cells per thread
  static constexpr int RR = NW * RW;              // region rows
  static constexpr int HALO = NONOS ? 2 : 1;      // recomputed rows on each side
  static constexpr int TJ = RR - 2 * HALO;        // output rows per tile
  static constexpr int NT = NW * 32;
  static constexpr int PLANE = RR * L;            // cells of one smem plane
  static constexpr int NSLOT = NONOS ? 9 : 5;
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

// Division flavours: exact IEEE in fp64, fast reciprocal in fp32.
__device__ __forceinline__ double rcp(double a) { return 1.0 / a; }
__device__ __forceinline__ float rcp(float a) { return __frcp_rn(a); }
__device__ __forceinline__ double qdiv(double a, double b) { return a / b; }
__device__ __forceinline__ float qdiv(float a, float b) { return __fdividef(a, b); }

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
  constexpr int Q = C::Q, KPL = C::KPL, RR = C::RR, PL = C::PLANE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  T* s_x1 = sm;                 // 3 slots of psi^(1)
  T* s_v = sm + 3 * PL;         // y-face pseudo-velocity slots
  T* s_w = s_v + (NONOS ? 2 : 1) * PL;
  T* s_bu = s_w + (NONOS ? 2 : 1) * PL;  // beta up   (NONOS)
  T* s_bd = s_bu + PL;                   // beta down (NONOS)

  const int tile = blockIdx.x % a.ntj;
  const int seg = blockIdx.x / a.ntj;
  const int span = a.o1 - a.o0;
  const int ib = a.o0 + static_cast<int>((static_cast<long long>(span) * seg) / a.nseg);
  const int ie = a.o0 + static_cast<int>((static_cast<long long>(span) * (seg + 1)) / a.nseg);
  if (ib >= ie) return;
  const int j0 = tile * C::TJ;
  const int m = a.m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // Per-row global offsets (j wraps periodically); k and smem offsets are
  // recomputed from (warp, lane, q) — q is a compile-time index.
  int gjr[RW], gjmr[RW], gjpr[RW];
#pragma unroll
  for (int rr = 0; rr < RW; ++rr) {
    int j = j0 - C::HALO + warp * RW + rr;
    j = ((j % m) + m) % m;
    gjr[rr] = j * L;
    gjmr[rr] = (j == 0 ? m - 1 : j - 1) * L;
    gjpr[rr] = (j == m - 1 ? 0 : j + 1) * L;
  }
#define IMB_CELL(q)                                                   \
  const int rr_ = (q) / KPL, kk_ = (q) % KPL;                         \
  const int r = warp * RW + rr_;                                      \
  const int k = lane + 32 * kk_;                                      \
  const int km = k == 0 ? L - 1 : k - 1, kp = k == L - 1 ? 0 : k + 1; \
  const int o = r * L + k, om_k = r * L + km, op_k = r * L + kp;      \
  const int gj = gjr[rr_], gjm = gjmr[rr_], gjp = gjpr[rr_];          \
  (void)om_k; (void)op_k; (void)gjm; (void)gjp; (void)km; (void)kp;
#define IMB_CELL_END
  auto slot3 = [](int p) { return ((p % 3) + 3) % 3; };
  auto pl = [&](int p) { return static_cast<long long>(p + a.R) * a.plane; };  // plane offset

  // ---- stage bodies -------------------------------------------------------
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
      const T fxl = flux(__ldg(Xm + c), xc, __ldg(U + c));
      const T fxr = flux(xc, __ldg(Xp + c), __ldg(Up + c));
      const T fyl = flux(__ldg(X + gjm + k), xc, __ldg(V + c));
      const T fyr = flux(xc, __ldg(X + gjp + k), __ldg(V + gjp + k));
      const T fzl = flux(__ldg(X + gj + km), xc, __ldg(W + c));
      const T fzr = flux(xc, __ldg(X + gj + kp), __ldg(W + gj + kp));
      const T div = ((fxr - fxl) + (fyr - fyl)) + (fzr - fzl);
      dst[o] = xc - div / __ldg(H + c);
    }
  };

  // P2: pseudo-velocities around base plane pb: x-face pb+1 (returned in ut),
  // y/z faces of plane pb (smem), and (NONOS) the bounds mx/mn of plane pb.
  auto stage_pseudo = [&](int pb, bool only_u, T* ut, T* vdst, T* wdst, T* mxq, T* mnq) {
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
      const bool row_u = r >= 1 && r < RR - 1;   // x/z faces and bounds
      const bool row_v = r >= 1;                 // y faces
      const T a1c = fabs(s1[o]);
      if (row_u) {  // x-face between planes pb and pb+1 of this column
        const T a2c = fabs(s2[o]);
        const T bp = fabs(s1[o + L]) + fabs(s2[o + L]);
        const T bm = fabs(s1[o - L]) + fabs(s2[o - L]);
        const T cp = fabs(s1[op_k]) + fabs(s2[op_k]);
        const T cm = fabs(s1[om_k]) + fabs(s2[om_k]);
        const int cjp = gjp + k, ckp = gj + kp;
        const T Vs = (__ldg(V1 + c) + __ldg(V2 + c)) + (__ldg(V1 + cjp) + __ldg(V2 + cjp));
        const T Ws = (__ldg(W1 + c) + __ldg(W2 + c)) + (__ldg(W1 + ckp) + __ldg(W2 + ckp));
        ut[q] = pseudo_face<T>(__ldg(U2 + c), __ldg(H1 + c), __ldg(H2 + c), a2c, a1c, bp, bm, Vs,
                               cp, cm, Ws);
      }
      if (only_u) continue;
      if (row_v) {  // y-face between rows r-1 and r of plane pb
        const int om = o - L;
        const int cjm = gjm + k;
        const T aL = fabs(s1[om]);
        const T bp = fabs(s2[om]) + fabs(s2[o]);
        const T bm = fabs(s0[om]) + fabs(s0[o]);
        const T cp = fabs(s1[op_k - L]) + fabs(s1[op_k]);
        const T cm = fabs(s1[om_k - L]) + fabs(s1[om_k]);
        const T Us = (__ldg(U1 + cjm) + __ldg(U1 + c)) + (__ldg(U2 + cjm) + __ldg(U2 + c));
        const int cjmkp = gjm + kp, ckp = gj + kp;
        const T Ws = (__ldg(W1 + cjm) + __ldg(W1 + c)) + (__ldg(W1 + cjmkp) + __ldg(W1 + ckp));
        vdst[o] = pseudo_face<T>(__ldg(V1 + c), __ldg(H1 + cjm), __ldg(H1 + c), a1c, aL, bp, bm,
                                 Us, cp, cm, Ws);
      }
      if (row_u) {  // z-face between k-1 and k
        const int ckm = gj + km;
        const T aL = fabs(s1[om_k]);
        const T bp = fabs(s2[om_k]) + fabs(s2[o]);
        const T bm = fabs(s0[om_k]) + fabs(s0[o]);
        const T cp = fabs(s1[om_k + L]) + fabs(s1[o + L]);
        const T cm = fabs(s1[om_k - L]) + fabs(s1[o - L]);
        const T Us = (__ldg(U1 + ckm) + __ldg(U1 + c)) + (__ldg(U2 + ckm) + __ldg(U2 + c));
        const int cjpkm = gjp + km, cjp = gjp + k;
        const T Vs = (__ldg(V1 + ckm) + __ldg(V1 + c)) + (__ldg(V1 + cjpkm) + __ldg(V1 + cjp));
        wdst[o] = pseudo_face<T>(__ldg(W1 + c), __ldg(H1 + ckm), __ldg(H1 + c), a1c, aL, bp, bm,
                                 Us, cp, cm, Vs);
        if constexpr (NONOS) {
          // 7-point bounds over psi^(1) and psi^n at plane pb.
          const T* X = a.x + pl(pb);
          T hi = s1[o], lo = s1[o];
          const T nb1[6] = {s0[o], s2[o], s1[o - L], s1[o + L], s1[om_k], s1[op_k]};
          const T nbn[7] = {__ldg(X + c),           __ldg(a.x + pl(pb - 1) + c),
                            __ldg(a.x + pl(pb + 1) + c), __ldg(X + gjm + k),
                            __ldg(X + gjp + k),   __ldg(X + ckm),
                            __ldg(X + gj + kp)};
#pragma unroll
          for (int e = 0; e < 6; ++e) {
            hi = fmax(hi, nb1[e]);
            lo = fmin(lo, nb1[e]);
          }
#pragma unroll
          for (int e = 0; e < 7; ++e) {
            hi = fmax(hi, nbn[e]);
            lo = fmin(lo, nbn[e]);
          }
          mxq[q] = hi;
          mnq[q] = lo;
        }
      }
    }
  };

  // ---- register carries (same (j,k) column, previous plane) ----------------
  T ucar[Q], ufresh[Q], fxc[Q], buc[Q], bdc[Q], bun[Q], bdn[Q], mxq[Q], mnq[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    ucar[q] = ufresh[q] = fxc[q] = buc[q] = bdc[q] = bun[q] = bdn[q] = mxq[q] = mnq[q] = T(0);
  }

  const int lag = NONOS ? 2 : 1;  // psi^(1) planes ahead of the output plane
  // warm-up: psi^(1) on the first two planes of the window, then the x-face
  // pseudo-velocity between them.
  stage_donor(ib - lag);
  stage_donor(ib - lag + 1);
  __syncthreads();
  stage_pseudo(ib - lag, true, ucar, nullptr, nullptr, nullptr, nullptr);

  const int tstart = NONOS ? ib - 2 : ib;
  for (int t = tstart; t < ie; ++t) {
    const bool emit = t >= ib;
    stage_donor(t + lag);  // psi^(1) of the newest plane
    __syncthreads();
    if constexpr (NONOS) {
      const int p1 = t + 1;
      T* vA = s_v + (p1 & 1) * PL;          // y-face velocities of plane t+1
      T* wA = s_w + (p1 & 1) * PL;
      const T* vB = s_v + ((p1 + 1) & 1) * PL;  // limited, plane t
      const T* wB = s_w + ((p1 + 1) & 1) * PL;
      stage_pseudo(p1, false, ufresh, vA, wA, mxq, mnq);
      __syncthreads();
      // P3: beta bounds of plane t+1.
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
          const T axl = flux(s0[o], xc, ucar[q]);
          const T axr = flux(xc, s2[o], ufresh[q]);
          const T ayl = flux(s1[o - L], xc, vA[o]);
          const T ayr = flux(xc, s1[o + L], vA[o + L]);
          const T azl = flux(s1[om_k], xc, wA[o]);
          const T azr = flux(xc, s1[op_k], wA[op_k]);
          const T fin = ((pos(axl) - neg(axr)) + (pos(ayl) - neg(ayr))) + (pos(azl) - neg(azr));
          const T fout = ((pos(axr) - neg(axl)) + (pos(ayr) - neg(ayl))) + (pos(azr) - neg(azl));
          const T hc = __ldg(H1 + gj + k);
          const T di = fin + Eps<T>::value, dou = fout + Eps<T>::value;
          T bu, bd;
          if constexpr (sizeof(T) == 8) {
            const T rr2 = rcp(di * dou);
            bu = ((mxq[q] - xc) * hc) * dou * rr2;
            bd = ((xc - mnq[q]) * hc) * di * rr2;
          } else {
            bu = qdiv((mxq[q] - xc) * hc, di);
            bd = qdiv((xc - mnq[q]) * hc, dou);
          }
          bun[q] = bu;
          bdn[q] = bd;
          s_bu[o] = bu;
          s_bd[o] = bd;
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
            vA[o] = limit(vA[o], s_bd[o - L], s_bu[o], s_bu[o - L], s_bd[o]);
          if (r < 2 || r >= RR - 2) continue;
          wA[o] = limit(wA[o], s_bd[om_k], s_bu[o], s_bu[om_k], s_bd[o]);
          const T ul = limit(ucar[q], bdc[q], bun[q], buc[q], bdn[q]);
          const T fxr = flux(s0[o], s1[o], ul);
          if (emit) {
            const T xc = s0[o];
            const T fyl = flux(s0[o - L], xc, vB[o]);
            const T fyr = flux(xc, s0[o + L], vB[o + L]);
            const T fzl = flux(s0[om_k], xc, wB[o]);
            const T fzr = flux(xc, s0[op_k], wB[op_k]);
            const T div = ((fxr - fxc[q]) + (fyr - fyl)) + (fzr - fzl);
            const int j = j0 + r - 2;
            if (j < m) O[gj + k] = xc - div / __ldg(H0 + gj + k);
          }
          fxc[q] = fxr;
        }
      }
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        ucar[q] = ufresh[q];
        buc[q] = bun[q];
        bdc[q] = bdn[q];
      }
      __syncthreads();
    } else {
      // Plain IORD=2: pseudo-velocities of plane t, then the final update.
      stage_pseudo(t, false, ufresh, s_v, s_w, nullptr, nullptr);
      __syncthreads();
      const T* s0 = s_x1 + slot3(t) * PL;
      const T* s1 = s_x1 + slot3(t + 1) * PL;
      const T* H0 = a.h + pl(t);
      T* O = a.out + pl(t);
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        IMB_CELL(q)
        if (r < 1 || r >= RR - 1) continue;
        const T xc = s0[o];
        const T fxl = flux(s_x1[slot3(t - 1) * PL + o], xc, ucar[q]);
        const T fxr = flux(xc, s1[o], ufresh[q]);
        const T fyl = flux(s0[o - L], xc, s_v[o]);
        const T fyr = flux(xc, s0[o + L], s_v[o + L]);
        const T fzl = flux(s0[om_k], xc, s_w[o]);
        const T fzr = flux(xc, s0[op_k], s_w[op_k]);
        const T div = ((fxr - fxl) + (fyr - fyl)) + (fzr - fzl);
        const int j = j0 + r - 1;
        if (j < m) O[gj + k] = xc - div / __ldg(H0 + gj + k);
        ucar[q] = ufresh[q];
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
