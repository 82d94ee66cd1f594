// Launch interface of the sm_100a MPDATA kernels (host side of csrc/*.cu).
// Every launcher returns the number of kernels it launched (for the
// launch-count evidence) and never synchronises.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "recipe.cuh"

namespace imb::dev {

// A plane range [p0, p1) of a padded slab with m x l planes.
struct Span {
  std::int64_t m, l, p0, p1;
};

template <class T>
int launch_update(const Span& s, const T* x, const T* U, const T* V, const T* W, const T* h,
                  T* out, cudaStream_t st);
template <class T>
int launch_pseudo(const Span& s, const T* x, const T* U, const T* V, const T* W, const T* h,
                  T* ut, T* vt, T* wt, cudaStream_t st);
template <class T>
int launch_bounds(const Span& s, const T* x, const T* xn, int first, T* mx, T* mn,
                  cudaStream_t st);
template <class T>
int launch_beta(const Span& s, const T* x, const T* ut, const T* vt, const T* wt, const T* h,
                const T* mx, const T* mn, T* bu, T* bd, cudaStream_t st);
template <class T>
int launch_limit(const Span& s, T* ut, T* vt, T* wt, const T* bu, const T* bd, cudaStream_t st);

// Seeded recipe into the five padded-slab fields. Plane p holds global
// i = (i0 + p - R) mod n, so halo planes are generated, not exchanged.
template <class T>
int launch_init(const recipe::Params& prm, std::int64_t i0, std::int64_t R, std::int64_t planes,
                T* x, T* u, T* v, T* w, T* h, cudaStream_t st);

// Reference surrogate stage ops on the padded GridField layout
// (workload.hpp:66-74): 7-point max/min over the interior.
int launch_stage7(const double* in, double* out, std::int64_t n, std::int64_t m, std::int64_t l,
                  std::int64_t halo, bool is_max, cudaStream_t st);

// ---- fused streaming step (csrc/mpdata_fused.cu) ----------------------
struct FusedShape {
  std::int64_t m, l;      // plane extents
  std::int64_t ni, R;     // interior planes, halo planes of the padded slab
  std::int64_t o0, o1;    // output plane range, local interior coordinates
};
// Halo push targets of a fused step (see mpdata_fused.cu Args): the
// neighbours' next-step buffers (padded-slab base pointers); null = none.
template <class T>
struct HaloPush {
  T* lo = nullptr;          // left neighbour's output buffer
  std::int64_t lo_ni = 0;   // left neighbour's interior planes
  T* hi = nullptr;          // right neighbour's output buffer
  bool sys = false;         // a target is on another GPU: fence system-wide after the stores
};
// Segmentation of a streaming launch: per j-tile of `tj` rows, kseg
// segments of lseg planes plus one remainder segment (blocks issued longest
// first); chosen by simulating the block scheduler (mpdata_fused.cu).
struct Plan {
  int ntj, kseg, lseg, blocks;
};
Plan plan_grid(std::int64_t m, int tj, std::int64_t planes, int resident, int warm);
// True when the fused kernel supports this (iord, nonos, m, l) combination on
// a padded slab of `planes` planes (its fields are indexed with 32 bits).
bool fused_supported(int iord, int nonos, std::int64_t m, std::int64_t l, std::int64_t planes);
template <class T>
int launch_fused(const FusedShape& fs, int iord, int nonos, const T* x, const T* u, const T* v,
                 const T* w, const T* h, T* out, int num_sms, cudaStream_t st,
                 const HaloPush<T>& push = {});
// IORD=3 + limiter as two fused launches: donor + pass 2 (writing psi^(2),
// its limited velocities and bounds on planes widened by 2), then pass 3.
template <class T>
int launch_fused3(const FusedShape& fs, const T* x, const T* u, const T* v, const T* w,
                  const T* h, T* x2, T* mx, T* mn, T* u2, T* v2, T* w2, T* out, int num_sms,
                  cudaStream_t st, const HaloPush<T>& push = {});

}  // namespace imb::dev
