// Per-lane vectors of K consecutive k values and their load/store helpers,
// plus the mbarrier / bulk-copy wrappers of the fused streaming kernel
// (mpdata_fused.cu holds the k +- 1 neighbour helpers).
#pragma once

#include <cuda_runtime.h>

#include <cstdio>

namespace imb::dev {
namespace {

constexpr unsigned kFull = 0xffffffffu;

// Checked build (-DIMB_CHECKED, tools/checked_build.sh): device-side bounds
// asserts on plane indices, rows and shared-memory offsets — the stand-in for
// compute-sanitizer, which this GPU pool does not allow.
#ifdef IMB_CHECKED
#define IMB_ASSERT(cond, what, v)                                                          \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("IMB_CHECKED %s: %lld (block %d thread %d)\n", what, static_cast<long long>(v), \
             static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));                  \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
__device__ __forceinline__ void check_shared(const void* p, unsigned bytes) {
  unsigned dyn;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
  extern __shared__ unsigned char imb_smem_base[];
  const long long off = static_cast<long long>(__cvta_generic_to_shared(p)) -
                        static_cast<long long>(__cvta_generic_to_shared(imb_smem_base));
  IMB_ASSERT(__isShared(p) && off >= 0 && off + bytes <= dyn, "shared offset", off);
}
#else
#define IMB_ASSERT(cond, what, v) ((void)0)
__device__ __forceinline__ void check_shared(const void*, unsigned) {}
#endif

__device__ __forceinline__ void l2_prefetch(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes));
}

// ---- mbarrier + bulk async copy (TMA engine) -------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
// global -> shared bulk copy (16-B aligned, a multiple of 16 B), completing on b
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void mbar_wait_s(unsigned b, unsigned parity) {  // shared address
  asm volatile(
      "{\n\t.reg .pred P;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n\t}" ::"r"(b),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

// ---- per-lane vectors of K consecutive k values ---------------------------
template <class T, int K>
struct Vec {
  T e[K];
};

template <class T, int K>
__device__ __forceinline__ Vec<T, K> vload(const T* p) {  // global, read-only path
  Vec<T, K> r;
  if constexpr (sizeof(T) == 8 && K == 4) {  // one 256-bit load (sm_100: global only)
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
        : "=d"(r.e[0]), "=d"(r.e[1]), "=d"(r.e[2]), "=d"(r.e[3]) : "l"(p));
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

// Read-only global load that does not allocate in L1 (data read once per cell).
template <class T, int K>
__device__ __forceinline__ Vec<T, K> vload_na(const T* p) {
  Vec<T, K> r;
  if constexpr (sizeof(T) == 8 && K == 2) {
    asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.e[0]), "=d"(r.e[1]) : "l"(p));
  } else if constexpr (sizeof(T) == 4 && K == 4) {
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
        : "=f"(r.e[0]), "=f"(r.e[1]), "=f"(r.e[2]), "=f"(r.e[3]) : "l"(p));
  } else {
    r = vload<T, K>(p);
  }
  return r;
}

// Global load through L2 only (coherent with this kernel's own earlier stores).
template <class T, int K>
__device__ __forceinline__ Vec<T, K> vload_cg(const T* p) {
  Vec<T, K> r;
  if constexpr (sizeof(T) == 8 && K == 4) {
    asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(r.e[0]), "=d"(r.e[1]), "=d"(r.e[2]), "=d"(r.e[3]) : "l"(p) : "memory");
  } else if constexpr (sizeof(T) == 8 && K == 2) {
    const double2 a = __ldcg(reinterpret_cast<const double2*>(p));
    r.e[0] = a.x; r.e[1] = a.y;
  } else if constexpr (sizeof(T) == 4 && K == 4) {
    const float4 a = __ldcg(reinterpret_cast<const float4*>(p));
    r.e[0] = a.x; r.e[1] = a.y; r.e[2] = a.z; r.e[3] = a.w;
  } else if constexpr (sizeof(T) == 4 && K == 2) {
    const float2 a = __ldcg(reinterpret_cast<const float2*>(p));
    r.e[0] = a.x; r.e[1] = a.y;
  } else {
    r.e[0] = __ldcg(p);
  }
  return r;
}

template <class T, int K>
__device__ __forceinline__ Vec<T, K> sload(const T* p) {  // shared
  check_shared(p, sizeof(T) * K);
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

// Global store with the evict-first (streaming) policy: for fields that are
// written once and next read by another launch, long after L2 has turned over.
template <class T, int K>
__device__ __forceinline__ void vstore_cs(T* p, const Vec<T, K>& v) {
  if constexpr (sizeof(T) == 8 && K == 2) {
    __stcs(reinterpret_cast<double2*>(p), make_double2(v.e[0], v.e[1]));
  } else if constexpr (sizeof(T) == 4 && K == 4) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(v.e[0], v.e[1], v.e[2], v.e[3]));
  } else if constexpr (sizeof(T) == 4 && K == 2) {
    __stcs(reinterpret_cast<float2*>(p), make_float2(v.e[0], v.e[1]));
  } else {
#pragma unroll
    for (int e = 0; e < K; ++e) __stcs(p + e, v.e[e]);
  }
}

template <class T, int K>
__device__ __forceinline__ void vstore(T* p, const Vec<T, K>& v) {  // shared or global
#ifdef IMB_CHECKED
  if (__isShared(p)) check_shared(p, sizeof(T) * K);
#endif
  if constexpr (sizeof(T) == 8 && K == 4) {  // global only: one 256-bit store (shared: sstore)
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v.e[0]), "d"(v.e[1]),
                 "d"(v.e[2]), "d"(v.e[3])
                 : "memory");
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

// Shared-memory rows of fp64 lanes holding 4 consecutive k (SPLIT layout):
// a lane's first two doubles sit in the row's first half at 16 B * lane, its
// last two in the second half (L/2 doubles on), so each half is one
// conflict-free 512-byte LDS.128/STS.128 wavefront set. p = the row + 2 * lane.
template <class T, int K, int L>
__device__ __forceinline__ Vec<T, K> sload_split(const T* p) {
  static_assert(sizeof(T) == 8 && K == 4, "split rows hold 4 doubles per lane");
  check_shared(p, 16);
  check_shared(p + L / 2, 16);
  Vec<T, K> r;
  const double2 a = reinterpret_cast<const double2*>(p)[0];
  const double2 b = reinterpret_cast<const double2*>(p + L / 2)[0];
  r.e[0] = a.x; r.e[1] = a.y; r.e[2] = b.x; r.e[3] = b.y;
  return r;
}
template <class T, int K, int L>
__device__ __forceinline__ void sstore_split(T* p, const Vec<T, K>& v) {
  static_assert(sizeof(T) == 8 && K == 4, "split rows hold 4 doubles per lane");
  check_shared(p, 16);
  check_shared(p + L / 2, 16);
  reinterpret_cast<double2*>(p)[0] = make_double2(v.e[0], v.e[1]);
  reinterpret_cast<double2*>(p + L / 2)[0] = make_double2(v.e[2], v.e[3]);
}

template <class T, int K>
__device__ __forceinline__ Vec<T, K> vabs(const Vec<T, K>& a) {
  Vec<T, K> r;
#pragma unroll
  for (int e = 0; e < K; ++e) r.e[e] = fabs(a.e[e]);
  return r;
}

}  // namespace
}  // namespace imb::dev
