// Fused streaming MPDATA step (IORD = 2, optional nonoscillatory limiter):
// one kernel reads psi^n, u, v, w, h and writes psi^{n+1}; every
// intermediate (psi^(1), pseudo-velocities, beta bounds, limited velocities,
// fluxes) lives in shared memory or registers.
//
// Geometry (B200-first):
//  * A warp owns whole rows. A lane holds E = NS*K cells of a row: NS
//    segments of K consecutive k (segment sg covers k in [sg*32K, (sg+1)*32K),
//    lane l its cells sg*32K + l*K + [0, K)). Every global/shared access is a
//    16-byte vector per lane and segment, so a warp moves a whole contiguous
//    row with conflict-free shared-memory wavefronts (fp64 at l = 128 uses
//    2 segments of 2 doubles). The k +- 1 neighbours are in registers or one
//    warp shuffle away: lane 0 of segment sg takes its k - 1 from lane 31 of
//    segment sg - 1 — the value the shuffle of that segment already delivers
//    to lane 0 — so the periodic k wrap and the segment seams close inside
//    the warp with a select, never with a reload.
//  * A block owns a j-tile of TJ output rows plus a recomputed halo of 2 rows
//    (limiter) or 1 row (plain) on each side: RR = NW*RW region rows.
//  * The block streams along i (the slab axis) over a segment of planes. The
//    stages run one plane apart, so along i nothing is recomputed except a
//    two-plane warm-up per segment. Shared memory holds the psi^(1) planes,
//    the y/z pseudo-velocities and both betas of the planes in flight;
//    same-column dependencies along i (x-face velocity, x-flux, the psi^n
//    star extrema) are register carries.
//  * Addressing: every global address is one 32-bit element index (plane
//    offset + row offset + lane offset, the row offsets loop-invariant)
//    scaled into the field pointer by a single IMAD.WIDE, with the segment
//    offsets as load immediates — no 64-bit multiplies in the stream loop.
//    The fused path therefore needs fields of < 2^32 elements (checked by
//    fused_supported's caller through FusedShape).
//  * Inputs come through L1/L2 (warp 0 bulk-prefetches every plane into L2
//    one plane ahead). fp32 at l = 128 also stages psi^n and h, the two most
//    re-read fields, in shared-memory rings filled by bulk async copies (TMA
//    engine, one mbarrier per slot); fp64 has no shared memory left for it.
//  * Divisions: fp64 folds the four divisions of a pseudo-velocity into one
//    reciprocal of hb*dA*dB*dC and the two beta divisions into one (MUFU seed
//    + one cubic Newton step); fp32 divides exactly (div.rn) and is compiled
//    without FMA contraction, so it rounds like the oracle (mpdata_math.cuh).
// The per-cell arithmetic follows SURVEY.md Appendix A (see mpdata_math.cuh).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdlib>
#include <functional>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "mpdata_kernels.cuh"
#include "mpdata_math.cuh"
#include "mpdata_vec.cuh"

namespace imb::dev {

namespace {

#ifdef IMB_PHASE_TIMING
// Debug-only per-phase cycle accounting (lane 0 of every warp), off in the product build.
__device__ unsigned long long g_phase_cycles[10 * 32];  // [slot][warp]
#define IMB_T(i) const long long imb_tp##i = clock64();
#define IMB_ACC(slot, a, b) \
  if (lane == 0)          \
    atomicAdd(&g_phase_cycles[(slot) * 32 + warp], static_cast<unsigned long long>(imb_tp##b - imb_tp##a));
#else
#define IMB_T(i)
#define IMB_ACC(slot, a, b)
#endif

#ifndef IMB_F64_NS  // fp64 at l = 128: two segments of 2 doubles per lane (1: one of 4 spills 364 B)
#define IMB_F64_NS 2
#endif
#ifndef IMB_TWO_F32  // two barriers per plane (see Cfg::TWO): fp32 +7.6 % C4, +4 % C5
#define IMB_TWO_F32 1
#endif
#ifndef IMB_TWO_F64  // fp64: -7 % C4 (224 KB of shared memory leaves 28 KB of L1; spills)
#define IMB_TWO_F64 0
#endif

// exact instruction savings of the limited step (see k_fused): -1 = measured default
#ifndef IMB_FLUXST
#define IMB_FLUXST -1
#endif
#ifndef IMB_BCLAMP
#define IMB_BCLAMP -1
#endif
#ifndef IMB_LFSIGN
#define IMB_LFSIGN -1
#endif
template <class T, int L, int RW, int NW, int NS, bool NONOS, bool STG = false, int WPR = 1,
          bool TMWB = false, bool XR = false, bool X13 = false>
struct Cfg {
  // A row is covered by WPR warps, each holding NS segments of 32*KPT cells.
  static constexpr int KPT = L / (32 * NS * WPR);  // consecutive k per lane and segment
  static_assert(KPT * 32 * NS * WPR == L, "row must split into warp-wide segments");
  static_assert(WPR == 1 || RW == 1, "several warps per row take one row each");
  // XR: two extra region rows beyond one per warp. Warp w owns row w+1; warp 0
  // also runs the donor of row 0 and warp NW-1 the donor and the y-face
  // pseudo-velocity of row RR-1 — the outermost halo rows, which do nothing
  // else. Without it those two rows idle through the pseudo-velocity and
  // bounds phases on two of the four schedulers (14 busy warps on 4
  // schedulers); with it all 16 warps are busy and a tile emits 14 rows
  // instead of 12 for about the same phase times.
  static constexpr int RR = NW * RW / WPR + (XR ? 2 : 0);   // region rows
  static constexpr int HALO = NONOS ? 2 : 1; // recomputed rows on each side
  static constexpr int TJ = RR - 2 * HALO;   // output rows per tile
  static constexpr int NT = NW * 32;
  static constexpr int PLANE = RR * L;       // cells of one smem plane
  // EARLY: the donor of plane t+3 runs in the same barrier phase as the
  // limiter/final update of plane t (3 barriers per plane instead of 4),
  // which takes a 4th psi^(1) slot.
  static constexpr bool EARLY = NONOS && L == 128;  // l=64: measured -3.5%
  // X13 (use_x13): with FLUXST the final update of plane t reads only its own
  // psi^(1)(t) cells (the limiter stored its y/z fluxes), and the same thread's
  // donor of plane t+3 comes later in the same phase, so it may overwrite
  // plane t's slot: three slots again, 18 KB more L1 at l = 128.
  static constexpr int NX1 = (EARLY && !X13) ? 4 : 3;  // psi^(1) slots
  // TWO: the donor of plane t+3 runs with the bounds (phase 2) and the
  // barrier between the final update (phase 3) and the next plane's
  // pseudo-velocities goes away; a third y/z-velocity slot keeps the next
  // plane's pseudo-velocities off the ones a slower warp's final update reads.
  static constexpr bool TWO = EARLY && (sizeof(T) == 4 ? IMB_TWO_F32 : IMB_TWO_F64);
  static constexpr int NVW = NONOS ? (TWO ? 3 : 2) : 1;  // y- and z-velocity slots each
  // TMWB: the z-face velocities and the betas' second plane live in tensor
  // memory (per-thread), so shared memory keeps no z-velocity slot and one
  // beta slot each (see k_fused)
  static constexpr int NWS = TMWB ? 0 : NVW;             // z-velocity slots
  static constexpr int NBS = TMWB ? 1 : 2;               // beta slots (up and down each)
  static constexpr int NSLOT = NONOS ? NX1 + NVW + NWS + 2 * NBS : 5;
  // STG: psi^n and h staged in shared memory by bulk async copies (TMA engine)
  // into rings of 4 (psi^n, rows -1..RR) and 5 (h, rows 0..RR-1) planes, each
  // slot with its own mbarrier.
  static constexpr int XROWS = RR + 2, HROWS = RR, NXS = 4, NHS = 5;
  static constexpr std::size_t STG_BYTES =
      STG ? sizeof(T) * L * (NXS * XROWS + NHS * HROWS) + 8 * (NXS + NHS) : 0;
  static constexpr std::size_t SMEM = sizeof(T) * PLANE * NSLOT + STG_BYTES;
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
  int kseg, lseg;   // per j-tile: kseg segments of lseg planes, then one remainder block
  int o0, o1;       // output plane range (interior coordinates)
  long long plane;  // m * l
  // IORD=3 split (MODE 1 writes, MODE 2 reads): bounds and limited velocities
  T* mxo;
  T* mno;
  T* uo;
  T* vo;
  T* wo;
  // Halo push (epilogue of the final pass): output planes t < R are also
  // stored into the left neighbour's next-step buffer at its right-halo plane
  // lo_ni + t, planes t >= ni - R into the right neighbour's left halo at
  // t - ni. The neighbour may be this slab itself (periodic single slab) or
  // another slab's buffer (same GPU, or a peer GPU over NVLink).
  T* push_lo;
  T* push_hi;
  int lo_ni;
  int ni;
  // L2 prefetch distance in planes (0 = off): each iteration, warp 0 issues
  // one bulk L2 prefetch per input field for the plane `pf` planes beyond
  // the newest one the donor stage reads, so its first touch is an L2 hit.
  int pf;
  int push_sys;  // push targets may be on a peer GPU (system-scope fence)
};

// One double loaded by the lanes with `on` only (the seam lane), into a fresh
// register that the caller selects against the shuffle result.
template <bool GLOBAL>
__device__ __forceinline__ double seam_load(const double* q, bool on) {
  double v;
  if constexpr (GLOBAL)
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q ld.global.nc.f64 %0, [%2];\n\t}"
        : "=d"(v) : "r"(static_cast<unsigned>(on)), "l"(q));
  else
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q ld.shared.f64 %0, [%2];\n\t}"
        : "=d"(v) : "r"(static_cast<unsigned>(on)), "r"(static_cast<unsigned>(__cvta_generic_to_shared(q))));
  return v;
}

// ---- k +- 1 neighbours of a lane's segment vector ---------------------------
// A warp holds NS segments of 32*K consecutive k of a row; inside a segment
// the neighbour is one shuffle away, and with NS == 1 the shuffle also
// closes the periodic wrap. With NS > 1 lane 0 (31) reloads its single
// neighbour across the seam: p is this lane's first cell of the segment
// (the offset folds into the load's immediate once the segment loop is
// unrolled), and the predicated load writes the shuffle's register in place
// (no merge moves).
template <int L, int NS, bool GLOBAL, class T, int K>
__device__ __forceinline__ Vec<T, K> kminus(const Vec<T, K>& a, const T* p, int sg, int lane) {
  Vec<T, K> r;
  r.e[0] = __shfl_sync(kFull, a.e[K - 1], (lane + 31) & 31);
  if constexpr (NS > 1) {
    static_assert(sizeof(T) == 8, "seam reloads are written for fp64");
    const T* q = p + (sg == 0 ? L - 1 : -1);  // lane 0's neighbour (sg is unrolled: an immediate)
    r.e[0] = lane == 0 ? seam_load<GLOBAL>(q, lane == 0) : r.e[0];
  }
#pragma unroll
  for (int e = 1; e < K; ++e) r.e[e] = a.e[e - 1];
  return r;
}
template <int L, int NS, bool GLOBAL, class T, int K>
__device__ __forceinline__ Vec<T, K> kplus(const Vec<T, K>& a, const T* p, int sg, int lane) {
  Vec<T, K> r;
  r.e[K - 1] = __shfl_sync(kFull, a.e[0], (lane + 1) & 31);
  if constexpr (NS > 1) {
    static_assert(sizeof(T) == 8, "seam reloads are written for fp64");
    // p is this lane's first cell of the segment; lane 31 needs the cell
    // after the segment (the next segment's first, or k = 0 after the last)
    const T* q = p + (sg == NS - 1 ? K - L : K);
    r.e[K - 1] = lane == 31 ? seam_load<GLOBAL>(q, lane == 31) : r.e[K - 1];
  }
#pragma unroll
  for (int e = 0; e + 1 < K; ++e) r.e[e] = a.e[e + 1];
  return r;
}
// Shared-memory rows with one segment (fp32): the single out-of-vector
// neighbour is re-read from the row (p = this lane's first cell; the wrap is
// in the offset).
template <int L, class T, int K>
__device__ __forceinline__ Vec<T, K> kminus_s(const Vec<T, K>& a, const T* p, int lane) {
  Vec<T, K> r;
  r.e[0] = p[lane == 0 ? L - 1 : -1];
#pragma unroll
  for (int e = 1; e < K; ++e) r.e[e] = a.e[e - 1];
  return r;
}
template <int L, class T, int K>
__device__ __forceinline__ Vec<T, K> kplus_s(const Vec<T, K>& a, const T* p, int lane) {
  Vec<T, K> r;
  r.e[K - 1] = p[lane == 31 ? K - L : K];
#pragma unroll
  for (int e = 0; e + 1 < K; ++e) r.e[e] = a.e[e + 1];
  return r;
}

#ifndef IMB_FINOUT_SD  // fp64 limiter in/out sums as (sum |f|) +- (left - right) (experiment)
#define IMB_FINOUT_SD 0
#endif
#ifndef IMB_TMEM_STAR  // psi^n star extrema carried in tensor memory (fp64, see k_fused)
#define IMB_TMEM_STAR 1
#endif
#ifndef IMB_TMEM_CACHE  // h (and v, without IMB_TMEM_WB) rows cached in tensor memory (fp64)
#define IMB_TMEM_CACHE 1
#endif
#ifndef IMB_TMEM_WB  // z-face velocities and the older beta plane in tensor memory (fp64)
#define IMB_TMEM_WB 1
#endif
#ifndef IMB_TMEM_CARRY  // x-face velocity and x-flux carries in tensor memory (fp64)
#define IMB_TMEM_CARRY 1
#endif
#ifndef IMB_M2_TMU  // IORD=3 pass 3 (MODE 2): the carries in TMEM instead of the v ring
#define IMB_M2_TMU 1
#endif

#ifndef IMB_XROWS  // extra halo rows handled by warps 0 and NW-1 (see Cfg::XR)
#define IMB_XROWS 1
#endif
#ifndef IMB_XR_YWARP  // see stage_pseudo. Split (2): C4 fp64 +2.5 %, C5 fp64 -0.8 %;
#define IMB_XR_YWARP 3  // all on warp 0 (0): C4 -1.5 %, fp32 -8 % (profiles/r02c_ab_xr_ywarp.txt);
#endif                  // four (segment, element) pieces on one warp per scheduler (3): C4 fp64
                        // +1.3 % over the split (profiles/r02f_ab_xr_y4.txt)
#ifndef IMB_XR_SPLIT_MODES  // bit m: MODE m splits the extra y-face (IORD=3 passes both: -0.8 %)
#define IMB_XR_SPLIT_MODES 1
#endif
#ifndef IMB_XR_Y4_W0  // IMB_XR_YWARP == 3: the four warps taking one (segment, element) piece each
#define IMB_XR_Y4_W0 0
#define IMB_XR_Y4_W1 5
#define IMB_XR_Y4_W2 10
#define IMB_XR_Y4_W3 15
#endif
// (fp32, one element of the lane's four on each of four warps: C4 fp32 -2.9 … -5.9 %,
// profiles/r02f_ab_xr_y4_fp32.txt — every piece repeats the row's loads; not kept)
#ifndef IMB_XR_YSPLIT_W1  // the warp taking the second segment of the split extra y-face
#define IMB_XR_YSPLIT_W1 15
#endif
#ifndef IMB_XR_D17_WARP  // the warp that runs row RR-1's donor when IMB_XR_D17_W0
#define IMB_XR_D17_WARP 0
#endif
#ifndef IMB_XR_D17_W0  // fp32 row RR-1 donor on warp 0: C4 fp32 -6.4 %, C5 -2.4 %; off
#define IMB_XR_D17_W0 0
#endif
#ifndef IMB_XR_Y0C  // fp32: C4 -12.3 % (profiles/r02c_ab_xr_y0c.txt) — extra work on warp 0,
#define IMB_XR_Y0C 0   // which also issues the TMA fills and L2 prefetches, hurts fp32; off
#endif
#ifndef IMB_XR64  // the same for l = 64 rows (two rows per warp, 34 region rows): C2 fp64
#define IMB_XR64 0  // +0.5 %, fp32 -1.9 % (56-64 spill bytes in fp64); off
#endif
// XR_DEFER: warp NW-1 computes row RR-1's y-face of plane t+2 right after its
// donors of plane t+3 (its own rows RR-2 and RR-1 are all it reads), in the
// donor's phase — instead of in the pseudo-velocity phase of plane t+2, where
// its scheduler carries 4 1/3 warps of work. Measured slower (C4 fp64 -2.5 %,
// fp32 -7.4 %): the donor phase is the longer one for that warp. Off.
#ifndef IMB_XR_DEFER
#define IMB_XR_DEFER 0
#endif
// bit m: MODE m uses the extra rows. Measured on C5 (profiles/r02c_ab_xr_modes.txt):
// fp64 without it in MODE 1 (pass 2 of IORD=3, which also stores six fields) +2.1 %;
// fp32 with it in MODE 0 only +0.3 %.
#ifndef IMB_XR_MODES_F64
#define IMB_XR_MODES_F64 5
#endif
#ifndef IMB_XR_MODES_F32
#define IMB_XR_MODES_F32 1
#endif
template <class T, int L, int RW, int NW, int NS, bool NONOS, int WPR, int MODE = 0>
constexpr bool use_xr() {
  constexpr int modes = sizeof(T) == 8 ? IMB_XR_MODES_F64 : IMB_XR_MODES_F32;
  return IMB_XROWS && ((modes >> MODE) & 1) && NONOS &&
         ((L == 128 && RW == 1) || (L == 64 && RW == 2 && IMB_XR64)) && WPR == 1;
}
// Three psi^(1) slots although the donor runs early (Cfg::X13). Needs the
// stored fluxes (FLUXST, fp64) and the donor in the final update's own phase
// (not TWO). IMB_X1_3 is a mask over MODE: C4 fp64 28.16 -> 29.10 Gcell/s
// (+3.3 %); on the IORD=3 passes too, C5 fp64 -1.4 %, so MODE 0 only.
#ifndef IMB_X1_3
#define IMB_X1_3 1
#endif
template <class T, int L, int RW, int NW, int NS, bool NONOS, bool STG, int WPR, int MODE>
constexpr bool use_x13() {
  using C = Cfg<T, L, RW, NW, NS, NONOS, STG, WPR>;
  return C::EARLY && !C::TWO && sizeof(T) == 8 && WPR == 1 && IMB_FLUXST != 0 && ((IMB_X1_3 >> MODE) & 1);
}

// Instantiations that use tensor memory as per-thread storage: the fp64
// limiter shapes with one 4-double lane vector per row (see k_fused: the
// psi^n star ring, the h and v row rings, and TMWB, the z-face velocities and
// betas).
template <class T, int L, int RW, int NW, int NS, bool NONOS, bool STARC, int MODE, bool STG, int WPR>
constexpr bool use_tmem() {
  using C = Cfg<T, L, RW, NW, NS, NONOS, STG, WPR>;
  return sizeof(T) == 8 && NONOS && C::EARLY && !STARC && !STG && RW * NS * C::KPT == 4 && NW == 16;
}
template <class T, int L, int RW, int NW, int NS, bool NONOS, bool STARC, int MODE, bool STG, int WPR>
constexpr bool use_tmwb() {
  return use_tmem<T, L, RW, NW, NS, NONOS, STARC, MODE, STG, WPR>() && IMB_TMEM_WB && IMB_TMEM_CACHE;
}

// ---- tensor memory (TMEM) as per-thread storage ------------------------------
// The stencil has no MMA, so the SM's 256 KB of TMEM is free: a warp reads
// and writes its own 32-lane quarter (lane = thread), 512 32-bit columns per
// lane shared by the NW/4 warps of that quarter. LDTM returns in ~12 cycles
// against several hundred for an L2 hit.
[[maybe_unused]] __device__ __forceinline__ void tmem_ld8(unsigned taddr, unsigned (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                 "=r"(v[7])
               : "r"(taddr)
               );
}
[[maybe_unused]] __device__ __forceinline__ void tmem_st8(unsigned taddr, const unsigned (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               );
}
[[maybe_unused]] __device__ __forceinline__ void tmem_st4(unsigned taddr, const unsigned (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3])
               );
}
[[maybe_unused]] __device__ __forceinline__ void tmem_ld4(unsigned taddr, unsigned (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr)
               );
}
[[maybe_unused]] __device__ __forceinline__ void tmem_ld16(unsigned taddr, unsigned (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15])
      : "r"(taddr));
}
[[maybe_unused]] __device__ __forceinline__ void tmem_st16(unsigned taddr, const unsigned (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}
template <int N>
__device__ __forceinline__ void tmem_ld(unsigned taddr, unsigned (&v)[N]) {
  if constexpr (N == 4) tmem_ld4(taddr, v);
  else if constexpr (N == 8) tmem_ld8(taddr, v);
  else if constexpr (N == 16) tmem_ld16(taddr, v);
  else __trap();  // (instantiated by shapes that never use TMEM)
}
template <int N>
__device__ __forceinline__ void tmem_st(unsigned taddr, const unsigned (&v)[N]) {
  if constexpr (N == 4) tmem_st4(taddr, v);
  else if constexpr (N == 8) tmem_st8(taddr, v);
  else if constexpr (N == 16) tmem_st16(taddr, v);
  else __trap();  // (instantiated by shapes that never use TMEM)
}
// K doubles <-> 2K TMEM columns (lo, hi words); fp32 never stores in TMEM
template <class T, int K>
__device__ __forceinline__ void packv(const Vec<T, K>& a, unsigned* w) {
#pragma unroll
  for (int e = 0; e < K; ++e) {
    if constexpr (sizeof(T) == 8) {
      w[2 * e] = static_cast<unsigned>(__double2loint(a.e[e]));
      w[2 * e + 1] = static_cast<unsigned>(__double2hiint(a.e[e]));
    } else {
      w[2 * e] = w[2 * e + 1] = __float_as_uint(a.e[e]);
    }
  }
}
template <class T, int K>
__device__ __forceinline__ Vec<T, K> unpackv(const unsigned* w) {
  Vec<T, K> r;
#pragma unroll
  for (int e = 0; e < K; ++e) {
    if constexpr (sizeof(T) == 8)
      r.e[e] = __hiloint2double(static_cast<int>(w[2 * e + 1]), static_cast<int>(w[2 * e]));
    else
      r.e[e] = __uint_as_float(w[2 * e]);
  }
  return r;
}
// two doubles <-> four TMEM columns (lo, hi words)
[[maybe_unused]] __device__ __forceinline__ void pack2(const double (&d)[2], unsigned* w) {
  w[0] = static_cast<unsigned>(__double2loint(d[0]));
  w[1] = static_cast<unsigned>(__double2hiint(d[0]));
  w[2] = static_cast<unsigned>(__double2loint(d[1]));
  w[3] = static_cast<unsigned>(__double2hiint(d[1]));
}
[[maybe_unused]] __device__ __forceinline__ void unpack2(const unsigned* w, double (&d)[2]) {
  d[0] = __hiloint2double(static_cast<int>(w[1]), static_cast<int>(w[0]));
  d[1] = __hiloint2double(static_cast<int>(w[3]), static_cast<int>(w[2]));
}
// No "memory" clobbers: TMEM is not memory the compiler tracks, and a clobber
// would pin every global load around the TMEM accesses (measured -2.4 % C4).
// Ordering comes from the registers instead: tmem_wait_ld(v) waits for this
// thread's outstanding LDTM and then "redefines" v, so no use of v can be
// scheduled before the wait (volatile asm statements keep their order).
template <int N>
__device__ __forceinline__ void tmem_wait_ld(unsigned (&v)[N]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("" : "+r"(v[i]));
}
[[maybe_unused]] __device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;"); }

// (MODE 2 returns from the donor before its loop: not a dead-code bug.)
#pragma nv_diag_suppress 128
// MODE 0: one IORD=2 step. MODE 1: donor + first corrective pass of an
// IORD=3 step, additionally writing the pass's limited velocities and 7-point
// bounds. MODE 2: the second corrective pass from psi^(2) (read instead of the
// donor), the limited velocities (as u, v, w) and the accumulated bounds.
template <class T, int L, int RW, int NW, int NS, bool NONOS, bool STARC, int MODE, bool STG, int WPR>
__global__ void __launch_bounds__(NW * 32, 1) k_fused(Args<T> a) {
  constexpr bool TMWB = use_tmwb<T, L, RW, NW, NS, NONOS, STARC, MODE, STG, WPR>();
  constexpr bool XR = use_xr<T, L, RW, NW, NS, NONOS, WPR, MODE>();
  // XR: row RR-1's donor on warp 0 instead of NW-1 (fp32: phase B balance)
  constexpr bool XR_D17_W0 = XR && sizeof(T) == 4 && IMB_XR_D17_W0;
  using C = Cfg<T, L, RW, NW, NS, NONOS, STG, WPR, TMWB, XR, use_x13<T, L, RW, NW, NS, NONOS, STG, WPR, MODE>()>;
  // XR_Y0C (two barriers per plane only): row RR-1's y-face of plane t+2 is
  // computed by warp 0 in the limiter/final phase of iteration t, where warp 0
  // (region row 1) has nothing else to do; the planes it reads are complete
  // after the bounds/donor barrier, and its slot row is not read before the
  // next iteration's bounds phase.
  constexpr bool XR_Y0C = XR && C::TWO && IMB_XR_Y0C;
  static_assert(!STG || (NONOS && MODE != 2 && RW == 1 && NS == 1 && WPR == 1 && C::EARLY),
                "staged inputs: IORD=2 limiter, one row per warp");
  constexpr int K = C::KPT, RR = C::RR, PL = C::PLANE, NC = RW * NS, SEG = 32 * K;
  using V = Vec<T, K>;
  // per-cell arithmetic runs on lane elements: one T, or (fp32) a P2 pair of
  // adjacent k issued as packed FADD2/FMUL2/FFMA2 (bit-identical rounding)
  using LN = Lane<T, K>;
  using S = typename LN::S;
  constexpr int PK = LN::PK;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  T* s_x1 = sm;                          // psi^(1) slots, by plane
  constexpr bool EARLY = C::EARLY;
  T* s_v = sm + C::NX1 * PL;             // y-face pseudo-velocities
  T* s_w = s_v + C::NVW * PL;            // z-face pseudo-velocities (not with TMWB)
  T* s_bu = s_w + C::NWS * PL;           // beta up,   NBS slots (NONOS)
  constexpr bool TWO = C::TWO;
  auto vws = [](int p) { return C::NVW == 3 ? (p + 6) % 3 : (p & 1); };  // p >= -3
  T* s_bd = s_bu + C::NBS * PL;          // beta down, NBS slots (NONOS)
  T* s_xs = s_x1 + C::NSLOT * PL;                 // STG: psi^n ring
  T* s_hs = s_xs + C::NXS * C::XROWS * L;         // STG: h ring
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(s_hs + C::NHS * C::HROWS * L);

  // Blocks [0, ntj*kseg): segment blockIdx/ntj of tile blockIdx%ntj, lseg
  // planes each; then one block per tile for the remaining planes (if any).
  // Issued longest first, the short remainder blocks fill the SMs that the
  // long ones leave idle (see plan_grid).
  const int nbig = a.ntj * a.kseg;
  const bool big = static_cast<int>(blockIdx.x) < nbig;
  const int tile = big ? blockIdx.x % a.ntj : blockIdx.x - nbig;
  const int ib = a.o0 + (big ? static_cast<int>(blockIdx.x / a.ntj) * a.lseg : a.kseg * a.lseg);
  const int ie = big ? ib + a.lseg : a.o1;
  if (ib >= ie) return;
  const int j0 = tile * C::TJ;
  const int m = a.m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef IMB_CHECK_SELFTEST  // proves a failing assert traps (tools/checked_build.sh --selftest)
  IMB_ASSERT(blockIdx.x != 0 || threadIdx.x != 0, "selftest", 0);
#endif
  const int wrow = (warp / WPR) * RW + (XR ? 1 : 0);  // first region row of this warp
  const int lk = (warp % WPR) * (L / WPR) + lane * K;  // this lane's first k of its segment 0
  const int gs0 = (warp % WPR) * NS;               // row segment index of this warp's segment 0
  // SPLIT: fp64 lanes of 4 consecutive k (one segment). Global rows are read
  // and written with 256-bit accesses (lane offset 4*lane); shared rows keep
  // a lane's two halves in the row's two halves (lane offset 2*lane, see
  // sload_split), so every LDS/STS.128 is a conflict-free 512-byte access.
  constexpr bool SPLIT = sizeof(T) == 8 && K == 4;
  static_assert(!SPLIT || (NS == 1 && WPR == 1), "split rows: one segment, one warp per row");
  const int lks = SPLIT ? 2 * lane : lk;  // this lane's offset in a shared row
  const unsigned PLN = static_cast<unsigned>(a.plane);

  // Rows of this warp: region row r = wrow + rr. Element offsets within a
  // plane of this lane's first cell in the row and in its j-1 / j+1
  // neighbours (j wraps periodically) — loop-invariant.
  unsigned gj[RW], gjm[RW], gjp[RW];
#pragma unroll
  for (int rr = 0; rr < RW; ++rr) {
    int j = j0 - C::HALO + wrow + rr;
    j = ((j % m) + m) % m;
    IMB_ASSERT(j >= 0 && j < m, "row outside the plane", j);
    gj[rr] = static_cast<unsigned>(j * L + lk);
    gjm[rr] = static_cast<unsigned>((j == 0 ? m - 1 : j - 1) * L + lk);
    gjp[rr] = static_cast<unsigned>((j == m - 1 ? 0 : j + 1) * L + lk);
  }
  // XR: the extra halo row this warp also handles (-1: none; warp-uniform)
  const int xrow_r = XR ? (warp == 0 ? 0 : (warp == NW - 1 ? RR - 1 : -1)) : -1;
  auto row_offsets = [&](int r, unsigned& g, unsigned& gm, unsigned& gp) {
    int j = j0 - C::HALO + r;
    j = ((j % m) + m) % m;
    g = static_cast<unsigned>(j * L + lk);
    gm = static_cast<unsigned>((j == 0 ? m - 1 : j - 1) * L + lk);
    gp = static_cast<unsigned>((j == m - 1 ? 0 : j + 1) * L + lk);
  };
  auto SLD = [](const T* p) {
    if constexpr (SPLIT) return sload_split<T, K, L>(p);
    else return sload<T, K>(p);
  };
#ifndef IMB_OUT_CS  // the step's output (the next launch's input) with streaming stores too
#define IMB_OUT_CS 0  // C4 +-0, C5 fp64 +0.2 %: off
#endif
#ifndef IMB_M2_NA  // MODE 2: the bounds fields, read once per cell, bypass L1 allocation
#define IMB_M2_NA 1  // C5 fp64 +0.7 %, fp32 +-0 (profiles/r02f_ab_cache_policy.txt)
#endif
#ifndef IMB_M1_CS  // pass 2 of IORD=3 writes its six intermediate fields with streaming stores
#define IMB_M1_CS 1  // C5 fp64 +0.7 %, fp32 +-0
#endif
  auto ISTORE = [](T* p, const V& v) {  // MODE 1's intermediates (next read by the MODE 2 launch)
    if constexpr (IMB_M1_CS) vstore_cs(p, v);
    else vstore(p, v);
  };
  auto SST = [](T* p, const V& v) {
    if constexpr (SPLIT) sstore_split<T, K, L>(p, v);
    else vstore(p, v);
  };
  auto slot3 = [](int p) { return C::NX1 == 4 ? ((p + 8) & 3) : (p + 6) % 3; };  // p >= -3
  // element offset of plane p of the padded slab
  auto pl = [&](int p) -> unsigned {
    IMB_ASSERT(p + a.R >= 0 && p < a.ni + a.R, "plane outside the padded slab", p);
    return static_cast<unsigned>(p + a.R) * PLN;
  };
  // cell group c = (row rr, segment sg): this lane's first cell of the
  // segment relative to its first cell of the row
  auto sgo = [](int c) { return (c % NS) * SEG; };
  // k +- 1 of a global row (p = this lane's cell pointer of the segment) or
  // of a shared row (fp64 shuffles, fp32 re-reads the out-of-vector value:
  // +1.4 % C4, +1 % C2 over shuffles)
  constexpr bool SRL = sizeof(T) == 4 && NS * WPR == 1;
  constexpr int NSEG = NS * WPR;  // segments per row
#define KMG(c, vec, p) kminus<L, NSEG, true>(vec, p, gs0 + (c) % NS, lane)
#define KPG(c, vec, p) kplus<L, NSEG, true>(vec, p, gs0 + (c) % NS, lane)
#define KMS(c, vec, p) (SRL ? kminus_s<L>(vec, p, lane) : kminus<L, NSEG, false>(vec, p, gs0 + (c) % NS, lane))
#define KPS(c, vec, p) (SRL ? kplus_s<L>(vec, p, lane) : kplus<L, NSEG, false>(vec, p, gs0 + (c) % NS, lane))

  // STG rings: psi^n planes from xb = ib - 3, h planes from hb = ib - 2 (the
  // first each warm-up donor reads); slot and fill (mbarrier phase) by plane.
  const int xb = ib - 3, hb = ib - 2;
  auto xslot = [&](int q) { return (q - xb) & (C::NXS - 1); };
  auto hslot = [&](int q) { return (q - hb) % C::NHS; };
  // this lane's first cell of region row r in the staged rings
  auto xrow = [&](int q, int r) { return s_xs + (xslot(q) * C::XROWS + r + 1) * L + lk; };
  auto hrow = [&](int q, int r) { return s_hs + (hslot(q) * C::HROWS + r) * L + lk; };
  const int jstage = j0 - C::HALO;  // global row of region row 0
  // one thread: rows jfirst.. of plane q of field f (periodic in j) -> dst
  auto stage_rows = [&](T* dst, const T* f, int q, int jfirst, int nrows, unsigned long long* bar) {
    const unsigned bytes = static_cast<unsigned>(nrows * L * sizeof(T));
    mbar_expect_tx(bar, bytes);
    const unsigned base = pl(q);
    const int j = ((jfirst % m) + m) % m;
    const int first = j + nrows <= m ? nrows : m - j;
    bulk_g2s(dst, f + (base + static_cast<unsigned>(j * L)),
             static_cast<unsigned>(first * L * sizeof(T)), bar);
    if (first < nrows)
      bulk_g2s(dst + first * L, f + base, static_cast<unsigned>((nrows - first) * L * sizeof(T)), bar);
  };
  auto fill_x = [&](int q) {
    stage_rows(s_xs + xslot(q) * C::XROWS * L, a.x, q, jstage - 1, C::XROWS, &mbar[xslot(q)]);
  };
  auto fill_h = [&](int q) {
    stage_rows(s_hs + hslot(q) * C::HROWS * L, a.h, q, jstage, C::HROWS, &mbar[C::NXS + hslot(q)]);
  };
  const unsigned mbar_s = smem_u32(mbar);
  auto wait_x = [&](int q) {
    mbar_wait_s(mbar_s + 8u * xslot(q), static_cast<unsigned>((q - xb) >> 2) & 1u);
  };
  auto wait_h = [&](int q) {
    mbar_wait_s(mbar_s + 8u * (C::NXS + hslot(q)), static_cast<unsigned>((q - hb) / C::NHS) & 1u);
  };
  if constexpr (STG) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < C::NXS + C::NHS; ++i) mbar_init(&mbar[i], 1);
      mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int q = ib - 3; q <= ib; ++q) fill_x(q);
      for (int q = ib - 2; q <= ib + 1; ++q) fill_h(q);
    }
  }
  // MODE 1: plane t+1 values of an own tile row are stored once (segments
  // abut: this block owns planes [ib, ie), the last segment also plane o1).
  auto keep = [&](int t, int r) {
    const int p = t + 1;
    return p >= ib && (p < ie || ie == a.o1) && r >= C::HALO && r < RR - C::HALO &&
           j0 + r - C::HALO < m;
  };
  // Phase barrier. (A point-to-point variant — each warp waiting only for its
  // j-neighbour warps through shared-memory progress counters — was measured
  // 3-4x slower than the hardware barrier and removed.)
  auto nb_sync = [&]() { __syncthreads(); };

  // TMS: the psi^n star extrema of plane p (max and min of psi^n over the
  // cell and its 6 face neighbours, which the donor of p has in registers
  // anyway) go to a 3-plane TMEM ring and come back in the bounds phase of
  // p two iterations later — instead of reloading 5 psi^n rows from L2 and
  // redoing 12 fp64 compare-selects there. fp64 only: fp32 carries them in
  // registers (STARC).
  // With the star ring, each warp's 128 TMEM columns also hold a 4-plane
  // ring of its h row (donor -> pseudo, bounds, final) and a 3-plane ring of
  // its v rows j and j+1 (donor -> pseudo): 8 of the 14 L2 loads of the
  // pseudo-velocity phase and the bounds/final h loads become LDTM.
  //   columns [0, 48) star (3 x 16), [48, 80) h (4 x 8), [80, 128) v (3 x 16)
  //
  // TMWB (instead of the v rows): the z-face pseudo-velocities and the betas
  // are only ever read by the thread that computed them (the k +- 1 partner
  // is a shuffle away), apart from beta's j-1 read of the newest plane. So
  // the z-velocities of planes t and t+1 and this thread's betas of the older
  // plane go to TMEM, and shared memory keeps one beta plane (up, down) and no
  // z-velocity plane: 64 KB less shared memory, i.e. 64 KB more L1.
  //   columns [80, 112) betas (2 planes x 16: segment c -> up [8c, 8c+4), down [8c+4, 8c+8)),
  //           [112, 128) z-velocities (2 planes x 8: segment c -> [4c, 4c+4))
  //
  // MODE 2 (pass 3 of IORD=3) reads its bounds instead of a psi^n star, so
  // its v ring takes the star's columns [0, 48) and it keeps TMWB.
  constexpr bool TMM = use_tmem<T, L, RW, NW, NS, NONOS, STARC, MODE, STG, WPR>();
  constexpr bool TMS = TMM && IMB_TMEM_STAR && MODE != 2;     // psi^n star ring
  constexpr bool TMH = TMM && IMB_TMEM_CACHE;                  // h ring
  constexpr bool TMC = TMH && (!TMWB || (MODE == 2 && !IMB_M2_TMU));  // v rows ring
  // TMU (MODE 0/1 with TMWB): the x-face velocity carries (planes t, t+1)
  // and the x-flux carry live in TMEM too, in the columns a 2-slot star ring
  // and a 3-slot h ring leave free (star(p) is last read by bounds(p), before
  // donor(p+2) reuses its slot in the same iteration; h(p) by final(p), before
  // donor(p+3)). Layout: star [0,32) h [32,56) u [56,72) fx [72,80).
  constexpr bool TMU = TMWB && (MODE != 2 || IMB_M2_TMU) && IMB_TMEM_CARRY;
  // Exact instruction savings of the limited step (round 2, last session; A/B in
  // profiles/r02f_ab_*.txt). Each knob: -1 = the measured default, 0 = off, 1 = on.
  //  FLUXST  the limiter stores the limited y/z-face FLUXES of plane t+1 in the velocity
  //          slots, so the final update reads them instead of forming each flux twice
  //          (fp64 all modes; fp32 passes 2/3 of IORD=3 only: fp32 MODE 0 measured -1.1 %)
  //  BCLAMP  beta stored as min(1, beta): the face limits drop their own clamp
  //          (min(1, a, b) = min(min(1, a), min(1, b)) exactly); fp64
  //  LFSIGN  a face's limit and its limited flux share the sign test of the velocity; fp64
  //  KSHARE  (mpdata_math.cuh) the in-lane k pair's max/min feeds both cells' bounds; fp64
  //          (bit 1; bit 0, the donor's psi^n star, spills: -1.8 %). Alone it is -0.4 % on
  //          the IORD=3 passes, together with LFSIGN +1.7 % (C5 fp64 13.25 against 13.04)
  constexpr bool F64 = sizeof(T) == 8;
  constexpr bool FLUXST = NONOS && (IMB_FLUXST < 0 ? (F64 || MODE != 0) : IMB_FLUXST != 0);
  constexpr bool BCLAMP = NONOS && (IMB_BCLAMP < 0 ? F64 : IMB_BCLAMP != 0);
  constexpr bool LFSIGN = NONOS && PK == 1 && (IMB_LFSIGN < 0 ? F64 : IMB_LFSIGN != 0);
  constexpr int KSHARE = IMB_KSHARE < 0 ? 2 : IMB_KSHARE;
  static_assert(!(C::EARLY && C::NX1 == 3) || (FLUXST && !C::TWO), "three psi^(1) slots with the early donor need the stored fluxes");
  __shared__ unsigned s_tmem_base;
  unsigned tm_lane = 0;
  if constexpr (TMM) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                   ::"r"(smem_u32(&s_tmem_base)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // this warp's lane quarter and its 128-column share of it
    tm_lane = s_tmem_base + (static_cast<unsigned>((warp & 3) * 32) << 16) +
              static_cast<unsigned>(warp >> 2) * (512u / (NW / 4));
  }
  auto tm_star = [&](int p) {
    return tm_lane + (TMU ? static_cast<unsigned>(p & 1) : static_cast<unsigned>((p + 6) % 3)) * 16u;
  };
  auto tm_h = [&](int p) {
    return TMU ? tm_lane + 32u + static_cast<unsigned>((p + 6) % 3) * 8u
               : tm_lane + 48u + static_cast<unsigned>((p + 8) & 3) * 8u;
  };
  auto tm_u = [&](int p) { return tm_lane + 56u + static_cast<unsigned>(p & 1) * 8u; };
  auto tm_fx = [&]() { return tm_lane + 72u; };
  auto tm_v = [&](int p) { return tm_lane + (MODE == 2 ? 0u : 80u) + static_cast<unsigned>((p + 6) % 3) * 16u; };
  auto tm_b = [&](int p) { return tm_lane + 80u + static_cast<unsigned>(p & 1) * 16u; };
  auto tm_w = [&](int p) { return tm_lane + 112u + static_cast<unsigned>(p & 1) * 8u; };
  // A V is CW = 2K TMEM columns; every ring slot holds NC*K = 4 doubles of
  // a row (8 columns) or two such rows / a max-min pair (16 columns).
  constexpr int CW = 2 * K;
  static_assert(!TMM || NC * K == 4, "TMEM rings hold 4 doubles per row and lane");
  auto vfrom = [](const unsigned* w) { return unpackv<T, K>(w); };
  auto tst = [&](unsigned addr, const V& x) {  // one V -> CW columns
    unsigned w[CW];
    packv(x, w);
    tmem_st<CW>(addr, w);
  };
  auto tst2 = [&](unsigned addr, const V& x, const V& y) {  // two Vs -> 2 CW columns
    unsigned w[2 * CW];
    packv(x, w);
    packv(y, w + CW);
    tmem_st<2 * CW>(addr, w);
  };
  auto tld = [&](unsigned addr) {
    unsigned w[CW];
    tmem_ld<CW>(addr, w);
    tmem_wait_ld(w);
    return vfrom(w);
  };
  auto tld2 = [&](unsigned addr, V& x, V& y) {
    unsigned w[2 * CW];
    tmem_ld<2 * CW>(addr, w);
    tmem_wait_ld(w);
    x = vfrom(w);
    y = vfrom(w + CW);
  };
  // TMWB: z-velocities of plane p, segment c, and their k+1 neighbours. With
  // two segments of a row (K = 2) the row is one TMEM load; lane 31's
  // neighbour is lane 0's first cell of the next segment (of segment 0 after
  // the last: periodic), which lane 0 offers in place of its own to the single
  // shuffle. With one segment (K = 4) the shuffle closes the periodic row.
  auto tm_wk = [&](int p, int c, V& wc, V& wcp) {
    if constexpr (NC == 1) {
      wc = tld(tm_w(p));
#pragma unroll
      for (int e = 0; e + 1 < K; ++e) wcp.e[e] = wc.e[e + 1];
      wcp.e[K - 1] = __shfl_sync(kFull, wc.e[0], (lane + 1) & 31);
    } else {
      static_assert(!TMWB || NC == 1 || (NC == 2 && K == 2), "TMWB: 1 segment, or 2 of 2 doubles");
      V s0, s1;
      tld2(tm_w(p), s0, s1);
      wc = c == 0 ? s0 : s1;
      const T offer = lane == 0 ? (c == 0 ? s1.e[0] : s0.e[0]) : wc.e[0];
#pragma unroll
      for (int e = 0; e + 1 < K; ++e) wcp.e[e] = wc.e[e + 1];
      wcp.e[K - 1] = __shfl_sync(kFull, offer, (lane + 1) & 31);
    }
  };

  // psi^n star extrema (STARC): of plane t+1 (nmx), t+2 (nmx_mid, EARLY) and
  // the donor's newest plane (nmx_new)
  V nmx_new[NC], nmn_new[NC], nmx[NC], nmn[NC], nmx_mid[NC], nmn_mid[NC];

  // P1: psi^(1) at plane p (donor cell) for all region rows: rows rbase..
  // with element offsets gj_/gjm_/gjp_. OWN: the warp's own rows, which also
  // keep the psi^n star and fill the TMEM rings; the XR extra row only needs
  // its psi^(1) in shared memory.
  auto stage_donor_rows = [&](int p, int rbase, const unsigned* gj_, const unsigned* gjm_,
                              const unsigned* gjp_, auto own_tag) {
    constexpr bool OWN = decltype(own_tag)::value;
    const unsigned px = pl(p);
    T* dst = s_x1 + slot3(p) * PL;
    if constexpr (MODE == 2) {  // psi^(2) is an input: stage it, carry the bounds
#pragma unroll
      for (int c = 0; c < (OWN ? NC : NS); ++c) {
        const int rr = c / NS, so = sgo(c);
        const unsigned ij = px + gj_[rr];
        SST(dst + (rbase + rr) * L + lks + so, vload<T, K>(a.x + ij + so));
        if constexpr (!OWN) continue;
        if constexpr (STARC) {
          nmx_new[c] = vload<T, K>(a.mxo + ij + so);
          nmn_new[c] = vload<T, K>(a.mno + ij + so);
        }
        if constexpr (TMH)  // the h and v rings, as the donor of MODE 0/1 fills them
          tst(tm_h(p) + CW * static_cast<unsigned>(c), vload<T, K>(a.h + ij + so));
        if constexpr (TMC)
          tst2(tm_v(p) + 2 * CW * static_cast<unsigned>(c), vload<T, K>(a.v + ij + so),
               vload<T, K>(a.v + (px + gjp_[rr]) + so));
      }
      if constexpr (TMH && OWN) tmem_wait_st();
      return;
    }
    if constexpr (STG && OWN) {
      // donors run in plane order: the older two psi^n planes were waited
      // for by the previous donor (all three by the segment's first)
      if (p == ib - 2) {  // (STG implies the limiter: lag 2)
        wait_x(p - 1);
        wait_x(p);
      }
      wait_x(p + 1);
      wait_h(p);
    }
#pragma unroll
    for (int c = 0; c < (OWN ? NC : NS); ++c) {
      const int rr = c / NS, so = sgo(c);
      const int r = rbase + rr;
      const unsigned ij = px + gj_[rr];
      const T* X = a.x + ij + so;
      V xc, xm, xp, ym, yp, zm, zp, hc;
      if constexpr (STG) {
        const T* xr = xrow(p, r) + so;
        xc = sload<T, K>(xr);
        xm = sload<T, K>(xrow(p - 1, r) + so);
        xp = sload<T, K>(xrow(p + 1, r) + so);
        ym = sload<T, K>(xr - L);
        yp = sload<T, K>(xr + L);
        zm = KMS(c, xc, xr);
        zp = KPS(c, xc, xr);
        hc = sload<T, K>(hrow(p, r) + so);
      } else {
        xc = vload<T, K>(X);
        xm = vload<T, K>(a.x + (ij - PLN) + so);
        xp = vload<T, K>(a.x + (ij + PLN) + so);
        ym = vload<T, K>(a.x + (px + gjm_[rr]) + so);
        yp = vload<T, K>(a.x + (px + gjp_[rr]) + so);
        zm = KMG(c, xc, X);
        zp = KPG(c, xc, X);
        hc = vload<T, K>(a.h + ij + so);
      }
      const V uc = vload<T, K>(a.u + ij + so), up = vload<T, K>(a.u + (ij + PLN) + so);
      const V vc = vload<T, K>(a.v + ij + so), vp = vload<T, K>(a.v + (px + gjp_[rr]) + so);
      if constexpr (TMH && OWN) tst(tm_h(p) + CW * static_cast<unsigned>(c), hc);  // h -> [CW c, CW c + CW)
      if constexpr (TMC && OWN) tst2(tm_v(p) + 2 * CW * static_cast<unsigned>(c), vc, vp);  // v rows j, j+1
      const T* W = a.w + ij + so;
      const V wc = vload<T, K>(W);
      const V wp = KPG(c, wc, W);
      V res;
#pragma unroll
      for (int e = 0; e < K; e += PK) {
        auto g = [e](const V& v) { return LN::get(v, e); };
        const S x0 = g(xc);
        const S fxl = upflux(g(xm), x0, g(uc));
        const S fxr = upflux(x0, g(xp), g(up));
        const S fyl = upflux(g(ym), x0, g(vc));
        const S fyr = upflux(x0, g(yp), g(vp));
        const S fzl = upflux(g(zm), x0, g(wc));
        const S fzr = upflux(x0, g(zp), g(wp));
        const S div = ((fxr - fxl) + (fyr - fyl)) + (fzr - fzl);
        LN::put(res, e, x0 - qdiv(div, g(hc)));
        if constexpr (NONOS && (STARC || TMS) && OWN) {
          S smx, smn;
          if constexpr ((KSHARE & 1) && sizeof(T) == 8 && K == 2) {
            // (zp[0] = xc[1] and zm[1] = xc[0]: one pair max/min serves both cells)
            star_minmax_pair(tmax(xc.e[0], xc.e[1]), tmin(xc.e[0], xc.e[1]), e == 0 ? zm.e[0] : zp.e[1],
                             g(xm), g(xp), g(ym), g(yp), smx, smn);
          } else {
            star_minmax(x0, g(xm), g(xp), g(ym), g(yp), g(zm), g(zp), smx, smn);
          }
          LN::put(nmx_new[c], e, smx);
          LN::put(nmn_new[c], e, smn);
        }
      }
      SST(dst + r * L + lks + so, res);
      if constexpr (TMS && OWN)  // segment c -> columns [2CW c, 2CW c + 2CW): max, then min
        tst2(tm_star(p) + 2 * CW * static_cast<unsigned>(c), nmx_new[c], nmn_new[c]);
    }
    if constexpr (TMS && OWN) tmem_wait_st();
  };
  auto stage_donor = [&](int p) {
    stage_donor_rows(p, wrow, gj, gjm, gjp, std::true_type{});
    if constexpr (XR) {
      if constexpr (XR_D17_W0) {
        // row RR-1's donor on warp IMB_XR_D17_WARP (fp32: scheduler 0 has the
        // slack in the bounds/donor phase; warp NW-1 carries row RR-1's y-face)
        if (warp == 0) {
          unsigned xg[1], xgm[1], xgp[1];
          row_offsets(0, xg[0], xgm[0], xgp[0]);
          stage_donor_rows(p, 0, xg, xgm, xgp, std::false_type{});
        }
        if (warp == IMB_XR_D17_WARP) {
          unsigned xg[1], xgm[1], xgp[1];
          row_offsets(RR - 1, xg[0], xgm[0], xgp[0]);
          stage_donor_rows(p, RR - 1, xg, xgm, xgp, std::false_type{});
        }
      } else if (xrow_r >= 0) {  // warps 0 and NW-1: the outermost halo row
        unsigned xg[1], xgm[1], xgp[1];
        row_offsets(xrow_r, xg[0], xgm[0], xgp[0]);
        stage_donor_rows(p, xrow_r, xg, xgm, xgp, std::false_type{});
      }
    }
  };

  // XR: the y-face pseudo-velocity between rows RR-2 and RR-1 of plane pb,
  // run by warp NW-1 after its own row (row RR-1 has no x/z faces). Same
  // arithmetic as the y-face of stage_pseudo; every operand comes from shared
  // memory or global memory (the TMEM rings hold the warp's own row).
  // W15: called by warp NW-1 only, whose xrow_r is RR-1 when it owns the
  // extra donor (the same offsets, computed from the register it has anyway)
  auto pseudo_y_extra = [&](int pb, T* vdst, int cbeg, int cend, auto w15_tag, int ebeg = 0, int eend = C::KPT) {
    constexpr bool W15 = decltype(w15_tag)::value;
    const int r = RR - 1;
    unsigned xg, xgm, xgp;
    row_offsets(W15 && NS == 1 && !XR_D17_W0 ? xrow_r : r, xg, xgm, xgp);
    (void)xgp;
    const T* s0 = s_x1 + slot3(pb - 1) * PL;
    const T* s1 = s_x1 + slot3(pb) * PL;
    const T* s2 = s_x1 + slot3(pb + 1) * PL;
    const unsigned p1 = pl(pb), p2 = p1 + PLN;
#pragma unroll
    for (int c = 0; c < NS; ++c) {
      if (NS > 1 && (c < cbeg || c >= cend)) continue;  // warp-uniform
      const int sg = sgo(c);
      const int so = r * L + lks + sg;
      const unsigned i1 = p1 + xg, i2 = p2 + xg;
      const V x1 = SLD(s1 + so);
      const V a1 = vabs(x1);
      const V x1m = SLD(s1 + so - L);
      const V a1m = vabs(x1m);
      const V a1km = vabs(KMS(c, x1, s1 + so));
      const V x0 = SLD(s0 + so), x2 = SLD(s2 + so);
      const V u1c = vload<T, K>(a.u + i1 + sg), u2c = vload<T, K>(a.u + i2 + sg);
      const T* W1 = a.w + i1 + sg;
      const V w1 = vload<T, K>(W1);
      const V v1 = vload<T, K>(a.v + i1 + sg);
      const V h1c = STG ? sload<T, K>(hrow(pb, r) + sg) : vload<T, K>(a.h + i1 + sg);
      V bp, bm, cp, cm, Us, Ws;
      {
        const V a0m = vabs(SLD(s0 + so - L)), a2m = vabs(SLD(s2 + so - L));
        const V a1mkp = vabs(KPS(c, x1m, s1 + so - L));
        const V a1mkm = vabs(KMS(c, x1m, s1 + so - L));
        const V a1kp = vabs(KPS(c, x1, s1 + so));
#pragma unroll
        for (int e = 0; e < K; e += PK) {
          auto g = [e](const V& v) { return LN::get(v, e); };
          LN::put(bp, e, g(a2m) + fabs(g(x2)));
          LN::put(bm, e, g(a0m) + fabs(g(x0)));
          LN::put(cp, e, g(a1mkp) + g(a1kp));
          LN::put(cm, e, g(a1mkm) + g(a1km));
        }
      }
      {
        const V u1m = vload<T, K>(a.u + (p1 + xgm) + sg), u2m = vload<T, K>(a.u + (p2 + xgm) + sg);
#pragma unroll
        for (int e = 0; e < K; e += PK) {
          auto g = [e](const V& v) { return LN::get(v, e); };
          LN::put(Us, e, (g(u1m) + g(u1c)) + (g(u2m) + g(u2c)));
        }
      }
      {
        const T* W1m = a.w + (p1 + xgm) + sg;
        const V w1m = vload<T, K>(W1m);
        const V w1mkp = KPG(c, w1m, W1m), w1kp = KPG(c, w1, W1);
#pragma unroll
        for (int e = 0; e < K; e += PK) {
          auto g = [e](const V& v) { return LN::get(v, e); };
          LN::put(Ws, e, (g(w1m) + g(w1)) + (g(w1mkp) + g(w1kp)));
        }
      }
      const V h1m = STG ? sload<T, K>(hrow(pb, r - 1) + sg) : vload<T, K>(a.h + (p1 + xgm) + sg);
      V res;
#pragma unroll
      for (int e = 0; e < K; e += PK) {
        if (e < ebeg || e >= eend) continue;  // (constants at the call sites: the unused lanes' sums fold away)
        auto g = [e](const V& v) { return LN::get(v, e); };
        LN::put(res, e, pseudo_face(g(v1), g(h1m), g(h1c), g(a1), g(a1m), g(bp), g(bm), g(Us), g(cp),
                                    g(cm), g(Ws)));
      }
      if (ebeg == 0 && eend == K) {
        SST(vdst + so, res);
      } else {  // a piece of the vector (IMB_XR_YWARP == 3): element stores
        if constexpr (!SPLIT && PK == 1) {
#pragma unroll
          for (int e = 0; e < K; ++e)
            if (e >= ebeg && e < eend) vdst[so + e] = res.e[e];
        }
      }
    }
  };

  // P2: pseudo-velocities around base plane pb: x-face pb+1 (into ut), y and
  // z faces of plane pb (into smem).
  auto stage_pseudo = [&](int pb, bool only_u, V* ut, T* vdst, T* wdst) {
    const T* s0 = s_x1 + slot3(pb - 1) * PL;
    const T* s1 = s_x1 + slot3(pb) * PL;
    const T* s2 = s_x1 + slot3(pb + 1) * PL;
    const unsigned p1 = pl(pb), p2 = p1 + PLN;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int rr = c / NS, sg = sgo(c);
      const int r = wrow + rr;
      if (r < 1) continue;  // warp-uniform
      const bool row_u = r < RR - 1;  // x/z faces (y faces: every r >= 1)
      const unsigned i1 = p1 + gj[rr], i2 = p2 + gj[rr];
      const int so = r * L + lks + sg;  // smem offset of this vector
      const V x1 = SLD(s1 + so);
      const V a1 = vabs(x1);
      const V a1m = vabs(SLD(s1 + so - L));
      const T* U2 = a.u + i2 + sg;
      const V u2c = vload<T, K>(U2);
      // v rows j, j+1 and h row j of planes pb, pb+1 (TMEM ring or L2)
      V h1c, h2, v1, v2, v1p, v2p;
      const unsigned cw = CW * static_cast<unsigned>(c);
      if constexpr (TMH && !TMC) {
        unsigned ha[CW], hb[CW];
        tmem_ld<CW>(tm_h(pb) + cw, ha);
        tmem_ld<CW>(tm_h(pb + 1) + cw, hb);
        v1 = vload<T, K>(a.v + i1 + sg);
        v2 = vload<T, K>(a.v + i2 + sg);
        v1p = vload<T, K>(a.v + (p1 + gjp[rr]) + sg);
        v2p = vload<T, K>(a.v + (p2 + gjp[rr]) + sg);
        tmem_wait_ld(ha);
        tmem_wait_ld(hb);
        h1c = vfrom(ha);
        h2 = vfrom(hb);
      } else if constexpr (TMC) {
        unsigned wa[2 * CW], wb[2 * CW], ha[CW], hb[CW];
        tmem_ld<2 * CW>(tm_v(pb) + 2 * cw, wa);
        tmem_ld<2 * CW>(tm_v(pb + 1) + 2 * cw, wb);
        tmem_ld<CW>(tm_h(pb) + cw, ha);
        tmem_ld<CW>(tm_h(pb + 1) + cw, hb);
        tmem_wait_ld(wa);
        tmem_wait_ld(wb);  // (already complete: these only order the register uses)
        tmem_wait_ld(ha);
        tmem_wait_ld(hb);
        v1 = vfrom(wa);
        v1p = vfrom(wa + CW);
        v2 = vfrom(wb);
        v2p = vfrom(wb + CW);
        h1c = vfrom(ha);
        h2 = vfrom(hb);
      } else {
        h1c = STG ? sload<T, K>(hrow(pb, r) + sg) : vload<T, K>(a.h + i1 + sg);
        h2 = STG ? sload<T, K>(hrow(pb + 1, r) + sg) : vload<T, K>(a.h + i2 + sg);
        v1 = vload<T, K>(a.v + i1 + sg);
        v2 = vload<T, K>(a.v + i2 + sg);
        v1p = vload<T, K>(a.v + (p1 + gjp[rr]) + sg);
        v2p = vload<T, K>(a.v + (p2 + gjp[rr]) + sg);
      }
      const V a1km = vabs(KMS(c, x1, s1 + so));
      if (row_u) {  // x-face between planes pb and pb+1 of this column
        const V x2 = SLD(s2 + so);
        const V a2 = vabs(x2);
        const V a1kp = vabs(KPS(c, x1, s1 + so));
        const V a2kp = vabs(KPS(c, x2, s2 + so)), a2km = vabs(KMS(c, x2, s2 + so));
        V bp, bm, cp, cm, Vs, Ws;
        {
          const V a1p = vabs(SLD(s1 + so + L)), a2p = vabs(SLD(s2 + so + L));
          const V a2m = vabs(SLD(s2 + so - L));
#pragma unroll
          for (int e = 0; e < K; e += PK) {
            auto g = [e](const V& v) { return LN::get(v, e); };
            LN::put(bp, e, g(a1p) + g(a2p));
            LN::put(bm, e, g(a1m) + g(a2m));
            LN::put(cp, e, g(a1kp) + g(a2kp));
            LN::put(cm, e, g(a1km) + g(a2km));
          }
        }
        {
#pragma unroll
          for (int e = 0; e < K; e += PK) {
            auto g = [e](const V& v) { return LN::get(v, e); };
            LN::put(Vs, e, (g(v1) + g(v2)) + (g(v1p) + g(v2p)));
          }
        }
        {
          const T* W1 = a.w + i1 + sg;
          const T* W2 = a.w + i2 + sg;
          const V w1 = vload<T, K>(W1), w2 = vload<T, K>(W2);
          const V w1p = KPG(c, w1, W1), w2p = KPG(c, w2, W2);
#pragma unroll
          for (int e = 0; e < K; e += PK) {
            auto g = [e](const V& v) { return LN::get(v, e); };
            LN::put(Ws, e, (g(w1) + g(w2)) + (g(w1p) + g(w2p)));
          }
        }
        V ures;
#pragma unroll
        for (int e = 0; e < K; e += PK) {
          auto g = [e](const V& v) { return LN::get(v, e); };
          LN::put(ures, e, pseudo_face(g(u2c), g(h1c), g(h2), g(a2), g(a1), g(bp), g(bm), g(Vs), g(cp),
                                       g(cm), g(Ws)));
        }
        if constexpr (TMU) tst(tm_u(pb) + CW * static_cast<unsigned>(c), ures);
        else ut[c] = ures;
      }
      if (only_u) continue;
      const V x0 = SLD(s0 + so);
      const V x2 = SLD(s2 + so);
      const T* U1 = a.u + i1 + sg;
      const V u1c = vload<T, K>(U1);
      const T* W1 = a.w + i1 + sg;
      const V w1 = vload<T, K>(W1);
      {  // y-face between rows r-1 and r of plane pb
        const V x1m = SLD(s1 + so - L);
        V bp, bm, cp, cm, Us, Ws;
        {
          const V a0m = vabs(SLD(s0 + so - L)), a2m = vabs(SLD(s2 + so - L));
          const V a1mkp = vabs(KPS(c, x1m, s1 + so - L));
          const V a1mkm = vabs(KMS(c, x1m, s1 + so - L));
          const V a1kp = vabs(KPS(c, x1, s1 + so));
#pragma unroll
          for (int e = 0; e < K; e += PK) {
            auto g = [e](const V& v) { return LN::get(v, e); };
            LN::put(bp, e, g(a2m) + fabs(g(x2)));
            LN::put(bm, e, g(a0m) + fabs(g(x0)));
            LN::put(cp, e, g(a1mkp) + g(a1kp));
            LN::put(cm, e, g(a1mkm) + g(a1km));
          }
        }
        {
          const V u1m = vload<T, K>(a.u + (p1 + gjm[rr]) + sg), u2m = vload<T, K>(a.u + (p2 + gjm[rr]) + sg);
#pragma unroll
          for (int e = 0; e < K; e += PK) {
            auto g = [e](const V& v) { return LN::get(v, e); };
            LN::put(Us, e, (g(u1m) + g(u1c)) + (g(u2m) + g(u2c)));
          }
        }
        {
          const T* W1m = a.w + (p1 + gjm[rr]) + sg;
          const V w1m = vload<T, K>(W1m);
          const V w1mkp = KPG(c, w1m, W1m), w1kp = KPG(c, w1, W1);
#pragma unroll
          for (int e = 0; e < K; e += PK) {
            auto g = [e](const V& v) { return LN::get(v, e); };
            LN::put(Ws, e, (g(w1m) + g(w1)) + (g(w1mkp) + g(w1kp)));
          }
        }
        const V h1m = STG ? sload<T, K>(hrow(pb, r - 1) + sg) : vload<T, K>(a.h + (p1 + gjm[rr]) + sg);
        V res;
#pragma unroll
        for (int e = 0; e < K; e += PK) {
          auto g = [e](const V& v) { return LN::get(v, e); };
          LN::put(res, e, pseudo_face(g(v1), g(h1m), g(h1c), g(a1), g(a1m), g(bp), g(bm), g(Us), g(cp),
                                      g(cm), g(Ws)));
        }
        SST(vdst + so, res);
      }
      if (row_u) {  // z-face between k-1 and k
        V bp, bm, cp, cm, Us, Vs;
        {
          const V x1p = SLD(s1 + so + L);
          const V x1m = SLD(s1 + so - L);
          const V a1pkm = vabs(KMS(c, x1p, s1 + so + L));
          const V a1mkm = vabs(KMS(c, x1m, s1 + so - L));
          const V a2km = vabs(KMS(c, x2, s2 + so)), a0km = vabs(KMS(c, x0, s0 + so));
#pragma unroll
          for (int e = 0; e < K; e += PK) {
            auto g = [e](const V& v) { return LN::get(v, e); };
            LN::put(bp, e, g(a2km) + fabs(g(x2)));
            LN::put(bm, e, g(a0km) + fabs(g(x0)));
            LN::put(cp, e, g(a1pkm) + fabs(g(x1p)));
            LN::put(cm, e, g(a1mkm) + g(a1m));
          }
        }
        {
          const V u2km = KMG(c, u2c, U2), u1km = KMG(c, u1c, U1);
#pragma unroll
          for (int e = 0; e < K; e += PK) {
            auto g = [e](const V& v) { return LN::get(v, e); };
            LN::put(Us, e, (g(u1km) + g(u1c)) + (g(u2km) + g(u2c)));
          }
        }
        {
          const T* V1 = a.v + i1 + sg;
          const T* V1p = a.v + (p1 + gjp[rr]) + sg;

          const V v1km = KMG(c, v1, V1), v1pkm = KMG(c, v1p, V1p);
#pragma unroll
          for (int e = 0; e < K; e += PK) {
            auto g = [e](const V& v) { return LN::get(v, e); };
            LN::put(Vs, e, (g(v1km) + g(v1)) + (g(v1pkm) + g(v1p)));
          }
        }
        const V h1km = STG ? KMS(c, h1c, hrow(pb, r) + sg) : KMG(c, h1c, a.h + i1 + sg);
        V res;
#pragma unroll
        for (int e = 0; e < K; e += PK) {
          auto g = [e](const V& v) { return LN::get(v, e); };
          LN::put(res, e, pseudo_face(g(w1), g(h1km), g(h1c), g(a1), g(a1km), g(bp), g(bm), g(Us), g(cp),
                                      g(cm), g(Vs)));
        }
        if constexpr (TMWB) {
          tst(tm_w(pb) + CW * static_cast<unsigned>(c), res);
        } else {
          SST(wdst + so, res);
        }
      }
    }
    if constexpr (TMWB) {
      if (!only_u || TMU) tmem_wait_st();
    }
    if constexpr (XR) {
      if (!IMB_XR_DEFER && !only_u) {
        // who computes row RR-1's y-face: 0 warp 0 (row 1, whose pseudo phase
        // has slack), 1 warp NW-1, 2 one segment each (two-segment rows)
        if constexpr (IMB_XR_YWARP == 3 && NS == 2 && K == 2 && ((IMB_XR_SPLIT_MODES >> MODE) & 1)) {
          // four pieces (segment, element) on one warp of each scheduler
          if (warp == IMB_XR_Y4_W0) pseudo_y_extra(pb, vdst, 0, 1, std::false_type{}, 0, 1);
          if (warp == IMB_XR_Y4_W1) pseudo_y_extra(pb, vdst, 0, 1, std::false_type{}, 1, 2);
          if (warp == IMB_XR_Y4_W2) pseudo_y_extra(pb, vdst, 1, 2, std::false_type{}, 0, 1);
          if (warp == IMB_XR_Y4_W3) pseudo_y_extra(pb, vdst, 1, 2, std::false_type{}, 1, 2);
        } else if constexpr (IMB_XR_YWARP >= 2 && NS == 2 && ((IMB_XR_SPLIT_MODES >> MODE) & 1)) {
          if (warp == 0) pseudo_y_extra(pb, vdst, 0, 1, std::false_type{});
          if (warp == IMB_XR_YSPLIT_W1) pseudo_y_extra(pb, vdst, 1, 2, std::false_type{});  // (NS == 2: no W15 path)
        } else {
          if constexpr (IMB_XR_YWARP == 0) {
            if (warp == 0) pseudo_y_extra(pb, vdst, 0, NS, std::false_type{});
          } else if constexpr (!XR_Y0C) {
            if (warp == NW - 1) pseudo_y_extra(pb, vdst, 0, NS, std::true_type{});
          }
        }
      }
    }
  };

  // ---- register carries along i (same (j,k) column) -------------------------
  V ucar[NC], ufresh[NC], fxc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int e = 0; e < K; ++e) {
      ucar[c].e[e] = ufresh[c].e[e] = fxc[c].e[e] = T(0);
      nmx[c].e[e] = nmn[c].e[e] = nmx_new[c].e[e] = nmn_new[c].e[e] = T(0);
      nmx_mid[c].e[e] = nmn_mid[c].e[e] = T(0);
    }

  const int lag = NONOS ? 2 : 1;  // psi^(1) planes ahead of the output plane
  // warm-up: psi^(1) on the first two planes of the window, then the x-face
  // pseudo-velocity between them.
  stage_donor(ib - lag);
  stage_donor(ib - lag + 1);
  if constexpr (STG) {  // x(ib-3), x(ib-2) are dead: their slots take x(ib+1), x(ib+2)
    __syncthreads();
    if (threadIdx.x == 0) {
      fill_x(ib + 1);
      fill_x(ib + 2);
    }
  }
  if constexpr (NONOS && STARC) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      nmx[c] = nmx_new[c];
      nmn[c] = nmn_new[c];
    }
  }
  if constexpr (EARLY) {
    stage_donor(ib - lag + 2);
    if constexpr (STARC) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        nmx_mid[c] = nmx_new[c];
        nmn_mid[c] = nmn_new[c];
      }
    }
  }
  __syncthreads();
  stage_pseudo(ib - lag, true, ucar, nullptr, nullptr);
  if constexpr (XR_Y0C) {  // the first plane the loop's pseudo phase reads
    if (warp == 0) pseudo_y_extra(ib - 1, s_v + vws(ib - 1) * PL, 0, NS, std::false_type{});
  }
  if constexpr (XR && IMB_XR_DEFER) {  // the first plane the loop's pseudo phase reads
    if (warp == NW - 1) pseudo_y_extra(ib - 1, s_v + vws(ib - 1) * PL, 0, NS, std::true_type{});
  }
  if constexpr (sizeof(T) == 4 || L != 128) {
    // Scheduling fence between the warm-up and the streaming loop: measured
    // +12% (fp32) / +10% (l=64 fp64) from the different instruction schedule
    // ptxas then picks; -2.5% for fp64 at l=128, where it is left out.
    __syncwarp();
    if (lane == 0) __threadfence_block();
  }

  const int tstart = NONOS ? ib - 2 : ib;
  // Rows a plane's donor touches: region rows plus one on each side (y +- 1).
  const int pf_j = j0 - C::HALO - 1;
  const int pf_rows = (RR + 2 < m ? RR + 2 : m);
  for (int t = tstart; t < ie; ++t) {
    const bool emit = t >= ib;
    if constexpr (STG) {  // one iteration ahead of the donor that first reads them
      // The refilled slots' last readers finished before the previous barrier
      // (their loads have returned), so no proxy fence is needed before the
      // async-proxy writes — the ordering a TMA pipeline gets from its "empty"
      // mbarrier (a fence.proxy.async here measured -1.5 %).
      if (threadIdx.x == 0) {
        if (t + 5 <= ie + 2) fill_x(t + 5);
        if (!TWO && t + 4 <= ie + 1) fill_h(t + 4);
      }
    }
    if (a.pf > 0 && warp == 0 && lane < 5 && !(STG && (lane == 0 || lane == 4))) {
      const int p = t + lag + 1 + a.pf;
      if (p <= ie + lag && p < a.ni + a.R) {
        const T* f = lane == 0 ? a.x : lane == 1 ? a.u : lane == 2 ? a.v : lane == 3 ? a.w : a.h;
        const unsigned base = pl(p);
        int j = pf_j < 0 ? pf_j + m : pf_j;
        const int first = (j + pf_rows <= m) ? pf_rows : m - j;
        l2_prefetch(f + (base + static_cast<unsigned>(j * L)), static_cast<unsigned>(first * L * sizeof(T)));
        if (first < pf_rows)
          l2_prefetch(f + base, static_cast<unsigned>((pf_rows - first) * L * sizeof(T)));
      }
    }
#ifndef IMB_M2_PFB  // MODE 2: L2-prefetch the bounds planes the next iteration's bounds phase reads
#define IMB_M2_PFB 1
#endif
    if constexpr (MODE == 2 && !STARC && IMB_M2_PFB) {
      if (a.pf > 0 && warp == 0 && (lane == 5 || lane == 6)) {
        const int p = t + 2;  // bounds(t + 1) of the next iteration reads plane t + 2
        if (p < ie + 1 && p < a.ni + a.R) {
          const T* f = lane == 5 ? a.mxo : a.mno;
          const unsigned base = pl(p);
          const int jb = j0 - C::HALO, nrows = (RR < m ? RR : m);
          const int j = jb < 0 ? jb + m : jb;
          const int first = (j + nrows <= m) ? nrows : m - j;
          l2_prefetch(f + (base + static_cast<unsigned>(j * L)), static_cast<unsigned>(first * L * sizeof(T)));
          if (first < nrows)
            l2_prefetch(f + base, static_cast<unsigned>((nrows - first) * L * sizeof(T)));
        }
      }
    }
    IMB_T(0)
    if constexpr (!EARLY) {
      stage_donor(t + lag);  // psi^(1) of the newest plane
      nb_sync();
    }
    IMB_T(1)
    IMB_T(2)
    IMB_ACC(0, 0, 1)
    IMB_ACC(1, 1, 2)
    if constexpr (NONOS) {
      const int p1 = t + 1;
      T* vA = s_v + vws(p1) * PL;              // y-face velocities, plane t+1
      T* wA = s_w + vws(p1) * PL;
      const T* vB = s_v + vws(t) * PL;         // limited, plane t
      const T* wB = s_w + vws(t) * PL;
      T* buA = s_bu + (C::NBS == 2 ? (p1 & 1) : 0) * PL;  // beta, plane t+1
      T* bdA = s_bd + (C::NBS == 2 ? (p1 & 1) : 0) * PL;
      const T* buB = s_bu + ((p1 + 1) & 1) * PL;  // beta, plane t
      const T* bdB = s_bd + ((p1 + 1) & 1) * PL;
      stage_pseudo(p1, false, ufresh, vA, wA);
      IMB_T(3)
      nb_sync();
      if constexpr (STG && TWO) {  // h(t-1)'s last reader, final(t-1), is behind this barrier
        if (threadIdx.x == 0 && t + 4 <= ie + 1) fill_h(t + 4);
      }
      IMB_T(4)
      IMB_ACC(2, 2, 3)
      IMB_ACC(3, 3, 4)
      // P3: 7-point bounds and beta of plane t+1.
      {
        const T* s0 = s_x1 + slot3(t) * PL;
        const T* s1 = s_x1 + slot3(t + 1) * PL;
        const T* s2 = s_x1 + slot3(t + 2) * PL;
        const unsigned q1 = pl(p1);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const int rr = c / NS, sg = sgo(c);
          const int r = wrow + rr;
          if (r < 1 || r >= RR - 1) continue;
          const int so = r * L + lks + sg;
          const unsigned i1 = q1 + gj[rr];
          const V xc = SLD(s1 + so);
          const V xm = SLD(s0 + so), xp = SLD(s2 + so);
          const V ym = SLD(s1 + so - L), yp = SLD(s1 + so + L);
          const V zm = KMS(c, xc, s1 + so), zp = KPS(c, xc, s1 + so);
          V mx, mn;
          if constexpr (STARC) {
            mx = nmx[c];
            mn = nmn[c];
          } else if constexpr (TMS) {  // (warp-uniform here: the whole warp owns row r)
            tld2(tm_star(p1) + 2 * CW * static_cast<unsigned>(c), mx, mn);
          } else if constexpr (MODE == 2) {  // bounds of the previous pass
            if constexpr (IMB_M2_NA) {
              mx = vload_na<T, K>(a.mxo + i1 + sg);
              mn = vload_na<T, K>(a.mno + i1 + sg);
            } else {
              mx = vload<T, K>(a.mxo + i1 + sg);
              mn = vload<T, K>(a.mno + i1 + sg);
            }
          } else {  // psi^n star of plane t+1, reloaded
            const T* N = a.x + i1 + sg;
            const V nc = vload<T, K>(N);
            const V n0 = vload<T, K>(a.x + (i1 - PLN) + sg), n2 = vload<T, K>(a.x + (i1 + PLN) + sg);
            const V nym = vload<T, K>(a.x + (q1 + gjm[rr]) + sg), nyp = vload<T, K>(a.x + (q1 + gjp[rr]) + sg);
            const V nzm = KMG(c, nc, N), nzp = KPG(c, nc, N);
#pragma unroll
            for (int e = 0; e < K; ++e) {
              mx.e[e] = tmax(tmax(tmax(nc.e[e], n0.e[e]), tmax(n2.e[e], nym.e[e])),
                             tmax(tmax(nyp.e[e], nzm.e[e]), nzp.e[e]));
              mn.e[e] = tmin(tmin(tmin(nc.e[e], n0.e[e]), tmin(n2.e[e], nym.e[e])),
                             tmin(tmin(nyp.e[e], nzm.e[e]), nzp.e[e]));
            }
          }
          const V va = SLD(vA + so), vap = SLD(vA + so + L);
          V wa, wap;
          if constexpr (TMWB) {
            tm_wk(p1, c, wa, wap);
          } else {
            wa = SLD(wA + so);
            wap = KPS(c, wa, wA + so);
          }
          V hc;
          if constexpr (TMH) {
            hc = tld(tm_h(p1) + CW * static_cast<unsigned>(c));
          } else {
            hc = STG ? sload<T, K>(hrow(p1, r) + sg) : vload<T, K>(a.h + i1 + sg);
          }
          V uL = ucar[c], uR = ufresh[c];  // x-face velocities (t|t+1), (t+1|t+2)
          if constexpr (TMU) {
            unsigned wl[CW], wr[CW];
            tmem_ld<CW>(tm_u(t) + CW * static_cast<unsigned>(c), wl);
            tmem_ld<CW>(tm_u(p1) + CW * static_cast<unsigned>(c), wr);
            tmem_wait_ld(wl);
            tmem_wait_ld(wr);
            uL = vfrom(wl);
            uR = vfrom(wr);
          }
          V bu, bd, his, los;
#pragma unroll
          for (int e = 0; e < K; e += PK) {
            auto g = [e](const V& v) { return LN::get(v, e); };
            const S x0 = g(xc);
            S hi, lo;
            if constexpr ((KSHARE & 2) && sizeof(T) == 8 && K == 2) {
              bound_minmax_pair(g(mx), g(mn), tmax(xc.e[0], xc.e[1]), tmin(xc.e[0], xc.e[1]),
                                e == 0 ? zm.e[0] : zp.e[1], g(xm), g(xp), g(ym), g(yp), hi, lo);
            } else {
              bound_minmax(g(mx), g(mn), x0, g(xm), g(xp), g(ym), g(yp), g(zm), g(zp), hi, lo);
            }
            LN::put(his, e, hi);
            LN::put(los, e, lo);
            const S axl = upflux(g(xm), x0, g(uL));
            const S axr = upflux(x0, g(xp), g(uR));
            const S ayl = upflux(g(ym), x0, g(va));
            const S ayr = upflux(x0, g(yp), g(vap));
            const S azl = upflux(g(zm), x0, g(wa));
            const S azr = upflux(x0, g(zp), g(wap));
            // 2*pos(f) = f + |f| and -2*neg(f) = |f| - f are exact, so these
            // are the oracle's inflow/outflow sums scaled by exactly 2.
            S fin2, fout2;
            if constexpr (std::is_same<S, double>::value && IMB_FINOUT_SD) {
              // fp64: in + out = sum |f| and in - out = sum_left f - sum_right f
              // (12 adds instead of 34; rounds differently from the oracle's sums)
              const S sa = ((fabs(axl) + fabs(axr)) + (fabs(ayl) + fabs(ayr))) + (fabs(azl) + fabs(azr));
              const S sd = ((axl - axr) + (ayl - ayr)) + (azl - azr);
              fin2 = sa + sd;
              fout2 = sa - sd;
            } else {
              fin2 = (((axl + fabs(axl)) + (fabs(axr) - axr)) +
                      ((ayl + fabs(ayl)) + (fabs(ayr) - ayr))) +
                     ((azl + fabs(azl)) + (fabs(azr) - azr));
              fout2 = (((axr + fabs(axr)) + (fabs(axl) - axl)) +
                       ((ayr + fabs(ayr)) + (fabs(ayl) - ayl))) +
                      ((azr + fabs(azr)) + (fabs(azl) - azl));
            }
            const S half = LN::cst(T(0.5)), eps = LN::cst(Eps<T>::value);
            const S di = half * fin2 + eps, dou = half * fout2 + eps;
            if constexpr (sizeof(T) == 8) {
              const T rr2 = rcp(di * dou);
              bu.e[e] = ((hi - x0) * hc.e[e]) * dou * rr2;
              bd.e[e] = ((x0 - lo) * hc.e[e]) * di * rr2;
              if constexpr (BCLAMP) {  // min(1, beta) once per cell instead of once per face limit
                bu.e[e] = tmin(T(1), bu.e[e]);
                bd.e[e] = tmin(T(1), bd.e[e]);
              }
            } else {
              if constexpr (BCLAMP) {
                LN::put(bu, e, tmin(LN::cst(T(1)), qdiv((hi - x0) * g(hc), di)));
                LN::put(bd, e, tmin(LN::cst(T(1)), qdiv((x0 - lo) * g(hc), dou)));
              } else {
                LN::put(bu, e, qdiv((hi - x0) * g(hc), di));
                LN::put(bd, e, qdiv((x0 - lo) * g(hc), dou));
              }
            }
          }
          SST(buA + so, bu);
          SST(bdA + so, bd);
          if constexpr (TMWB) {  // this thread's betas of plane t+1, for its own x-face limit next iteration
            tst2(tm_b(p1) + 2 * CW * static_cast<unsigned>(c), bu, bd);
          }
          if constexpr (MODE == 1) {  // bounds for the next pass
            if (keep(t, r)) {
              ISTORE(a.mxo + i1 + sg, his);
              ISTORE(a.mno + i1 + sg, los);
            }
          }
        }
      }
      if constexpr (TWO) {
        if (t + 3 <= ie + 1) {
          stage_donor(t + 3);  // the last plane pseudo(ie) reads is ie+1
          if constexpr (XR && IMB_XR_DEFER) {
            if (warp == NW - 1) {
              __syncwarp();  // this warp's psi^(1) rows of plane t+3, lane to lane
              pseudo_y_extra(t + 2, s_v + vws(t + 2) * PL, 0, NS, std::true_type{});
            }
          }
        }
      }
      if constexpr (TMWB) tmem_wait_st();
      IMB_T(5)
      nb_sync();
      IMB_T(6)
      IMB_ACC(4, 4, 5)
      IMB_ACC(5, 5, 6)
      // P4: limit plane t+1 velocities; P5: final update of plane t.
      {
        const T* s0 = s_x1 + slot3(t) * PL;
        const T* s1 = s_x1 + slot3(t + 1) * PL;
        const unsigned q0 = pl(t), q1 = q0 + PLN;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const int rr = c / NS, sg = sgo(c);
          const int r = wrow + rr;
          if (r < 2 || r >= RR - 1) continue;
          const int so = r * L + lks + sg;
          const V bu = SLD(buA + so), bd = SLD(bdA + so);
          V x1;
          if constexpr (FLUXST) x1 = SLD(s1 + so);
          {
            const V va = SLD(vA + so);
            const V bum = SLD(buA + so - L), bdm = SLD(bdA + so - L);
            V res;
            if constexpr (FLUXST) {
              // the slot keeps the limited y-face FLUX of plane t+1 (both
              // rows that share the face read it in the next iteration's
              // final update instead of forming it twice)
              const V y1m = SLD(s1 + so - L);
              V fy;
#pragma unroll
              for (int e = 0; e < K; e += PK) {
                auto g = [e](const V& v) { return LN::get(v, e); };
                if constexpr (LFSIGN) {
                  S vl;
                  LN::put(fy, e, limit_flux<BCLAMP>(g(va), g(bdm), g(bu), g(bum), g(bd), g(y1m), g(x1), vl));
                  LN::put(res, e, vl);
                } else {
                  const S vl = limit_sel<BCLAMP>(g(va), g(bdm), g(bu), g(bum), g(bd));
                  LN::put(res, e, vl);
                  LN::put(fy, e, upflux(g(y1m), g(x1), vl));
                }
              }
              SST(vA + so, fy);
            } else {
#pragma unroll
              for (int e = 0; e < K; e += PK) {
                auto g = [e](const V& v) { return LN::get(v, e); };
                LN::put(res, e, limit_sel<BCLAMP>(g(va), g(bdm), g(bu), g(bum), g(bd)));
              }
              SST(vA + so, res);
            }
            if constexpr (MODE == 1) {
              if (keep(t, r)) ISTORE(a.vo + (q1 + gj[rr]) + sg, res);
            }
          }
          if (r >= RR - 2) continue;
          V fxr;
          {
            V wa, buo, bdo;
            if constexpr (TMWB) {
              unsigned t8[2 * CW], w4[CW];
              tmem_ld<2 * CW>(tm_b(t) + 2 * CW * static_cast<unsigned>(c), t8);
              tmem_ld<CW>(tm_w(p1) + CW * static_cast<unsigned>(c), w4);
              tmem_wait_ld(t8);
              tmem_wait_ld(w4);
              buo = vfrom(t8);
              bdo = vfrom(t8 + CW);
              wa = vfrom(w4);
            } else {
              wa = SLD(wA + so);
              buo = SLD(buB + so);
              bdo = SLD(bdB + so);
            }
            const V bukm = KMS(c, bu, buA + so), bdkm = KMS(c, bd, bdA + so);
            const V xc = SLD(s0 + so);
            if constexpr (!FLUXST) x1 = SLD(s1 + so);
            const V uc = TMU ? tld(tm_u(t) + CW * static_cast<unsigned>(c)) : ucar[c];
            V wres, uls, fz;
            V x1km;
            if constexpr (FLUXST) x1km = KMS(c, x1, s1 + so);
#pragma unroll
            for (int e = 0; e < K; e += PK) {
              auto g = [e](const V& v) { return LN::get(v, e); };
              if constexpr (LFSIGN) {
                S wl, ul;
                if constexpr (FLUXST) {
                  LN::put(fz, e, limit_flux<BCLAMP>(g(wa), g(bdkm), g(bu), g(bukm), g(bd), g(x1km), g(x1), wl));
                } else {
                  wl = limit_sel<BCLAMP>(g(wa), g(bdkm), g(bu), g(bukm), g(bd));
                }
                LN::put(wres, e, wl);
                LN::put(fxr, e, limit_flux<BCLAMP>(g(uc), g(bdo), g(bu), g(buo), g(bd), g(xc), g(x1), ul));
                LN::put(uls, e, ul);
              } else {
                const S wl = limit_sel<BCLAMP>(g(wa), g(bdkm), g(bu), g(bukm), g(bd));
                LN::put(wres, e, wl);
                if constexpr (FLUXST) LN::put(fz, e, upflux(g(x1km), g(x1), wl));
                const S ul = limit_sel<BCLAMP>(g(uc), g(bdo), g(bu), g(buo), g(bd));
                LN::put(uls, e, ul);
                LN::put(fxr, e, upflux(g(xc), g(x1), ul));
              }
            }
            if constexpr (TMWB) {  // (FLUXST: the limited z-face flux of plane t+1)
              tst(tm_w(p1) + CW * static_cast<unsigned>(c), FLUXST ? fz : wres);
            } else {
              SST(wA + so, FLUXST ? fz : wres);
            }
            if constexpr (MODE == 1) {
              if (keep(t, r)) {
                ISTORE(a.wo + (q1 + gj[rr]) + sg, wres);
                ISTORE(a.uo + (q1 + gj[rr]) + sg, uls);
              }
            }
          }
          if (emit) {
            const V xc = SLD(s0 + so);
            V ym, yp, zm, zp;
            if constexpr (!FLUXST) {
              ym = SLD(s0 + so - L);
              yp = SLD(s0 + so + L);
              zm = KMS(c, xc, s0 + so);
              zp = KPS(c, xc, s0 + so);
            }
            const V vb = SLD(vB + so), vbp = SLD(vB + so + L);
            V wb, wbp;
            if constexpr (TMWB) {
              tm_wk(t, c, wb, wbp);
            } else {
              wb = SLD(wB + so);
              wbp = KPS(c, wb, wB + so);
            }
            V hc;
            if constexpr (TMH) {
              hc = tld(tm_h(t) + CW * static_cast<unsigned>(c));
            } else {
              hc = STG ? sload<T, K>(hrow(t, r) + sg) : vload<T, K>(a.h + (q0 + gj[rr]) + sg);
            }
            const V fxl = TMU ? tld(tm_fx() + CW * static_cast<unsigned>(c)) : fxc[c];
            V res;
#pragma unroll
            for (int e = 0; e < K; e += PK) {
              auto g = [e](const V& v) { return LN::get(v, e); };
              const S x0 = g(xc);
              S fyl, fyr, fzl, fzr;
              if constexpr (FLUXST) {  // the slots hold the limited fluxes themselves
                fyl = g(vb);
                fyr = g(vbp);
                fzl = g(wb);
                fzr = g(wbp);
              } else {
                fyl = upflux(g(ym), x0, g(vb));
                fyr = upflux(x0, g(yp), g(vbp));
                fzl = upflux(g(zm), x0, g(wb));
                fzr = upflux(x0, g(zp), g(wbp));
              }
              const S div = ((g(fxr) - g(fxl)) + (fyr - fyl)) + (fzr - fzl);
              LN::put(res, e, x0 - qdiv(div, g(hc)));
            }
            const int j = j0 + r - 2;
            if (j < m) {
              if constexpr (MODE == 1 || IMB_OUT_CS) ISTORE(a.out + (q0 + gj[rr]) + sg, res);
              else vstore(a.out + (q0 + gj[rr]) + sg, res);
            }
          }
          if constexpr (TMU) tst(tm_fx() + CW * static_cast<unsigned>(c), fxr);
          else fxc[c] = fxr;
        }
      }
      if constexpr (TMWB) tmem_wait_st();
      if constexpr (XR_Y0C) {
        if (warp == 0 && t + 2 <= ie) pseudo_y_extra(t + 2, s_v + vws(t + 2) * PL, 0, NS, std::false_type{});
      }
      IMB_T(9)
      if constexpr (EARLY && !TWO) {
        if (t + 3 <= ie + 1) {
          stage_donor(t + 3);  // the last plane pseudo(ie) reads is ie+1
          if constexpr (XR && IMB_XR_DEFER) {
            if (warp == NW - 1) {
              __syncwarp();  // this warp's psi^(1) rows of plane t+3, lane to lane
              pseudo_y_extra(t + 2, s_v + vws(t + 2) * PL, 0, NS, std::true_type{});
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        ucar[c] = ufresh[c];
        if constexpr (STARC && EARLY) {
          nmx[c] = nmx_mid[c];
          nmn[c] = nmn_mid[c];
          nmx_mid[c] = nmx_new[c];
          nmn_mid[c] = nmn_new[c];
        } else if constexpr (STARC) {
          nmx[c] = nmx_new[c];
          nmn[c] = nmn_new[c];
        }
      }
      IMB_T(7)
      if constexpr (!TWO) nb_sync();
      IMB_T(8)
      IMB_ACC(6, 6, 9)
      IMB_ACC(8, 9, 7)
      IMB_ACC(7, 7, 8)
    } else {
      // Plain IORD=2: pseudo-velocities of plane t, then the final update.
      stage_pseudo(t, false, ufresh, s_v, s_w);
      nb_sync();
      const T* sm1 = s_x1 + slot3(t - 1) * PL;
      const T* s0 = s_x1 + slot3(t) * PL;
      const T* s1 = s_x1 + slot3(t + 1) * PL;
      const unsigned q0 = pl(t);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int rr = c / NS, sg = sgo(c);
        const int r = wrow + rr;
        if (r < 1 || r >= RR - 1) continue;
        const int so = r * L + lks + sg;
        const V xc = SLD(s0 + so);
        const V xm = SLD(sm1 + so), xp = SLD(s1 + so);
        const V ym = SLD(s0 + so - L), yp = SLD(s0 + so + L);
        const V zm = KMS(c, xc, s0 + so), zp = KPS(c, xc, s0 + so);
        const V vv = SLD(s_v + so), vvp = SLD(s_v + so + L);
        const V ww = SLD(s_w + so);
        const V wwp = KPS(c, ww, s_w + so);
        const V hc = vload<T, K>(a.h + (q0 + gj[rr]) + sg);
        V res;
#pragma unroll
        for (int e = 0; e < K; e += PK) {
          auto g = [e](const V& v) { return LN::get(v, e); };
          const S x0 = g(xc);
          const S fxl = upflux(g(xm), x0, g(ucar[c]));
          const S fxr = upflux(x0, g(xp), g(ufresh[c]));
          const S fyl = upflux(g(ym), x0, g(vv));
          const S fyr = upflux(x0, g(yp), g(vvp));
          const S fzl = upflux(g(zm), x0, g(ww));
          const S fzr = upflux(x0, g(zp), g(wwp));
          const S div = ((fxr - fxl) + (fyr - fyl)) + (fzr - fzl);
          LN::put(res, e, x0 - qdiv(div, g(hc)));
        }
        const int j = j0 + r - 1;
        if (j < m) vstore(a.out + (q0 + gj[rr]) + sg, res);
        ucar[c] = ufresh[c];
      }
      nb_sync();
    }
  }
  // Halo push epilogue (outside the streaming loop so the hot loop's
  // schedule is untouched): re-read this block's output planes t < R and
  // t >= ni - R of its own tile rows (written above by this block; visible
  // after the barrier) and store them into the neighbours' halo planes.
  if constexpr (MODE != 1) {
    if (a.push_lo != nullptr || a.push_hi != nullptr) {
      __syncthreads();
      const int tl = (ib > 0 ? ib : 0), th = (ie < a.R ? ie : a.R);          // [tl, th): t < R
      const int ul = (ib > a.ni - a.R ? ib : a.ni - a.R), uh = ie;           // t >= ni - R
      for (int pass = 0; pass < 2; ++pass) {
        const int p0 = pass == 0 ? tl : ul, p1 = pass == 0 ? th : uh;
        T* dstb = pass == 0 ? a.push_lo : a.push_hi;
        if (dstb == nullptr) continue;
        for (int t = p0; t < p1; ++t) {
          const int dplane = pass == 0 ? a.R + a.lo_ni + t : a.R + t - a.ni;
          IMB_ASSERT(pass == 0 ? (dplane >= a.lo_ni + a.R && dplane < a.lo_ni + 2 * a.R)
                               : (dplane >= 0 && dplane < a.R),
                     "halo push plane", dplane);
          const unsigned dbase = static_cast<unsigned>(dplane) * PLN;
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const int rr = c / NS, sg = sgo(c);
            const int r = wrow + rr;
            if (r < C::HALO || r >= RR - C::HALO || j0 + r - C::HALO >= m) continue;
            // L2-coherent load: a.out was written by this kernel
            vstore(dstb + (dbase + gj[rr]) + sg, vload_cg<T, K>(a.out + (pl(t) + gj[rr]) + sg));
          }
        }
      }
      // Pushes into a peer GPU (NVLink) are made visible system-wide before
      // this kernel completes and the neighbour's flag word is raised.
      if (a.push_sys && (tl < th || ul < uh)) __threadfence_system();
    }
  }
  if constexpr (TMM) {
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem_base));
  }
#undef KMG
#undef KPG
#undef KMS
#undef KPS
}
#pragma nv_diag_default 128

}  // namespace

// Choose the i-segmentation of every j-tile: kseg segments of lseg planes
// plus one remainder segment, blocks issued longest first. Each candidate
// lseg is scored by simulating the block scheduler (a block goes to the
// resident slot that frees first; a block costs its planes + the warm-up);
// the smallest makespan wins, then the fewest blocks. Uniform splits are the
// candidates with no remainder. Plans are cached per shape.
#ifndef IMB_ONLY_F32  // precision-independent host code lives in the fp64 object
Plan plan_grid(std::int64_t m, int tj, std::int64_t planes, int resident, int warm) {
  static std::mutex mu;
  static std::map<std::tuple<std::int64_t, int, std::int64_t, int, int>, Plan> cache;
  const auto key = std::make_tuple(m, tj, planes, resident, warm);
  std::lock_guard<std::mutex> lock(mu);
  if (auto it = cache.find(key); it != cache.end()) return it->second;
  const int ntj = static_cast<int>((m + tj - 1) / tj);
  Plan best{ntj, 1, static_cast<int>(planes), ntj};
  long long best_span = LLONG_MAX;
  const long long min_len = std::max<long long>(1, planes / 256);
  std::vector<long long> slot;
  static const long long max_len = [] {
    const char* e = std::getenv("IMB_SEG_MAX");  // A/B knob: longest segment in planes
    return e ? std::max(1LL, std::atoll(e)) : LLONG_MAX;
  }();
  for (long long len = std::min<long long>(planes, max_len); len >= min_len; --len) {
    const long long k = planes / len, rem = planes - k * len;
    const long long blocks = ntj * k + (rem > 0 ? ntj : 0);
    if (blocks > 16LL * resident || blocks > INT_MAX / 2) continue;
    // longest-first list scheduling on `resident` slots
    slot.assign(static_cast<std::size_t>(std::min<long long>(resident, blocks)), 0);
    std::make_heap(slot.begin(), slot.end(), std::greater<long long>());
    long long makespan = 0;
    auto issue = [&](long long count, long long cost) {
      for (long long b = 0; b < count; ++b) {
        std::pop_heap(slot.begin(), slot.end(), std::greater<long long>());
        slot.back() += cost;
        makespan = std::max(makespan, slot.back());
        std::push_heap(slot.begin(), slot.end(), std::greater<long long>());
      }
    };
    issue(ntj * k, len + warm);
    if (rem > 0) issue(ntj, rem + warm);
    if (makespan < best_span || (makespan == best_span && blocks < best.blocks)) {
      best_span = makespan;
      best = Plan{ntj, static_cast<int>(k), static_cast<int>(len), static_cast<int>(blocks)};
    }
  }
  cache.emplace(key, best);
  return best;
}
#endif

namespace {

template <class T, int L, int RW, int NW, int NS, bool NONOS, bool STARC, int MODE, bool STG = false,
          int WPR = 1>
int launch_cfg(const FusedShape& fs, const Args<T>& proto, int num_sms, cudaStream_t st) {
  using C = Cfg<T, L, RW, NW, NS, NONOS, STG, WPR,
                use_tmwb<T, L, RW, NW, NS, NONOS, STARC, MODE, STG, WPR>(),
                use_xr<T, L, RW, NW, NS, NONOS, WPR, MODE>(),
                use_x13<T, L, RW, NW, NS, NONOS, STG, WPR, MODE>()>;
  auto kern = k_fused<T, L, RW, NW, NS, NONOS, STARC, MODE, STG, WPR>;
  // Function attributes and occupancy are per device: configure each device
  // once (a group or a measurement may drive several GPUs from one process).
  static std::mutex mu;
  static std::map<int, int> per_sm_of;  // device -> resident blocks per SM
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = per_sm_of.find(dev);
    if (it == per_sm_of.end()) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(C::SMEM)) != cudaSuccess)
        return -1;
      int n = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, C::NT, C::SMEM) != cudaSuccess ||
          n < 1)
        return -1;  // the launch could not be resident: report, do not launch
      it = per_sm_of.emplace(dev, n).first;
    }
    per_sm = it->second;
  }
  static const int warm_env = [] {
    const char* e = std::getenv("IMB_WARM");  // experiment: warm-up cost in plane-times
    return e ? std::atoi(e) : -1;
  }();
  const int warm = warm_env >= 0 ? warm_env : (NONOS ? 3 : 2);  // measured: 3 beats 4 by 2 % at 128-plane slabs
  const Plan p = plan_grid(fs.m, C::TJ, fs.o1 - fs.o0, per_sm * num_sms, warm);
  Args<T> a = proto;
  a.m = static_cast<int>(fs.m);
  a.R = static_cast<int>(fs.R);
  a.ntj = p.ntj;
  a.kseg = p.kseg;
  a.lseg = p.lseg;
  a.o0 = static_cast<int>(fs.o0);
  a.o1 = static_cast<int>(fs.o1);
  a.plane = fs.m * fs.l;
  static const int pf = [] {
    const char* e = std::getenv("IMB_PF");  // measured: 1 plane ahead +5% (C4 fp64)
    return e ? std::atoi(e) : 1;
  }();
  a.pf = pf;
  kern<<<p.blocks, C::NT, C::SMEM, st>>>(a);
  return 1;
}

template <class T, bool NONOS, int MODE>
int dispatch_l(const FusedShape& fs, const Args<T>& a, int num_sms, cudaStream_t st) {
  // fp64 keeps lane vectors at 2 doubles (register budget) and reloads the
  // psi^n star; fp32 holds 4 floats per lane and carries the star.
  constexpr bool D = sizeof(T) == 8;
  switch (fs.l) {
    case 128:
#ifdef IMB_F32_RW2  // experiment: fp32 with two rows per warp (8 cells per thread, 32-row tiles)
      if constexpr (!D && NONOS)
        return launch_cfg<T, 128, 2, 16, 1, NONOS, true, MODE>(fs, a, num_sms, st);
#endif
      if constexpr (!D && NONOS && MODE != 2) {
        // psi^n and h staged by bulk async copies: C4 fp32 +3.3 %, C5 fp32 +1 %
        // (IMB_STG=0 turns it off for A/B runs)
        static const bool stg = [] {
          const char* e = std::getenv("IMB_STG");
          return !(e && e[0] == '0');
        }();
        // (the staged rings copy XROWS rows of a plane in at most two pieces)
        if (stg && fs.m >= Cfg<T, 128, 1, 16, 1, NONOS, true, 1, false,
                               use_xr<T, 128, 1, 16, 1, NONOS, 1, MODE>()>::XROWS)
          return launch_cfg<T, 128, 1, 16, 1, NONOS, true, MODE, true>(fs, a, num_sms, st);
      }
#ifdef IMB_F64_WPR2_NW  // experiment: two warps per row (one 2-double segment per lane)
      if constexpr (D)
        return launch_cfg<T, 128, 1, IMB_F64_WPR2_NW, 1, NONOS, false, MODE, false, 2>(fs, a, num_sms, st);
#endif
      return launch_cfg<T, 128, 1, 16, D ? IMB_F64_NS : 1, NONOS, !D, MODE>(fs, a, num_sms, st);
    case 64: return launch_cfg<T, 64, 2, 16, 1, NONOS, !D, MODE>(fs, a, num_sms, st);
    case 32: return launch_cfg<T, 32, 4, 16, 1, NONOS, !D, MODE>(fs, a, num_sms, st);
    default: return 0;
  }
}

}  // namespace

#ifndef IMB_ONLY_F32
bool fused_supported(int iord, int nonos, std::int64_t m, std::int64_t l, std::int64_t planes) {
  // the kernel addresses every field with 32-bit element indices
  const bool fits = planes > 0 && planes * m * l < (std::int64_t{1} << 32);
  const bool shape = (l == 32 || l == 64 || l == 128) && m >= 3 && m < (1 << 20) && fits;
  return shape && (iord == 2 || (iord == 3 && nonos));
}
#endif

#if defined(IMB_PHASE_TIMING)
#ifdef IMB_ONLY_F32
extern "C" int imb_debug_phase_cycles_f32(unsigned long long* out, int reset) {
#else
extern "C" int imb_debug_phase_cycles(unsigned long long* out, int reset) {
#endif
  cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(g_phase_cycles));
  if (reset) {
    unsigned long long z[10 * 32] = {};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  }
  return 0;
}
#endif

template <class T>
int launch_fused(const FusedShape& fs, int iord, int nonos, const T* x, const T* u, const T* v,
                 const T* w, const T* h, T* out, int num_sms, cudaStream_t st,
                 const HaloPush<T>& push) {
  if (iord != 2) return 0;
  Args<T> a{x, u, v, w, h, out, 0, 0, 0, 0, 0, 0, 0, 0, nullptr, nullptr, nullptr, nullptr, nullptr,
            push.lo, push.hi, static_cast<int>(push.lo_ni), static_cast<int>(fs.ni)};
  a.push_sys = push.sys ? 1 : 0;
  return nonos ? dispatch_l<T, true, 0>(fs, a, num_sms, st)
               : dispatch_l<T, false, 0>(fs, a, num_sms, st);
}

template <class T>
int launch_fused3(const FusedShape& fs, const T* x, const T* u, const T* v, const T* w,
                  const T* h, T* x2, T* mx, T* mn, T* u2, T* v2, T* w2, T* out, int num_sms,
                  cudaStream_t st, const HaloPush<T>& push) {
  // pass 2 (with the donor) over the output planes widened by the radius of
  // the limited pass 3 (2), then pass 3 on the requested planes.
  FusedShape f1 = fs;
  f1.o0 = fs.o0 - 2;
  f1.o1 = fs.o1 + 2;
  Args<T> a1{x, u, v, w, h, x2, 0, 0, 0, 0, 0, 0, 0, 0, mx, mn, u2, v2, w2,
             nullptr, nullptr, 0, static_cast<int>(fs.ni)};
  const int n = dispatch_l<T, true, 1>(f1, a1, num_sms, st);
  if (n <= 0) return n;
  Args<T> a2{x2, u2, v2, w2, h, out, 0, 0, 0, 0, 0, 0, 0, 0, mx, mn, nullptr, nullptr, nullptr,
             push.lo, push.hi, static_cast<int>(push.lo_ni), static_cast<int>(fs.ni)};
  a2.push_sys = push.sys ? 1 : 0;
  const int n2 = dispatch_l<T, true, 2>(fs, a2, num_sms, st);
  return n2 < 0 ? n2 : n + n2;
}

// Each precision is its own object (Makefile): fp32 is built with
// --fmad=false so it rounds exactly like the oracle (mpdata_math.cuh).
#ifndef IMB_ONLY_F32
template int launch_fused<double>(const FusedShape&, int, int, const double*, const double*,
                                  const double*, const double*, const double*, double*, int,
                                  cudaStream_t, const HaloPush<double>&);
#endif
#ifndef IMB_ONLY_F64
template int launch_fused<float>(const FusedShape&, int, int, const float*, const float*,
                                 const float*, const float*, const float*, float*, int,
                                 cudaStream_t, const HaloPush<float>&);
#endif
#ifndef IMB_ONLY_F32
template int launch_fused3<double>(const FusedShape&, const double*, const double*, const double*,
                                   const double*, const double*, double*, double*, double*,
                                   double*, double*, double*, double*, int, cudaStream_t,
                                   const HaloPush<double>&);
#endif
#ifndef IMB_ONLY_F64
template int launch_fused3<float>(const FusedShape&, const float*, const float*, const float*,
                                  const float*, const float*, float*, float*, float*, float*,
                                  float*, float*, float*, int, cudaStream_t,
                                  const HaloPush<float>&);

#endif

}  // namespace imb::dev
