// Device-side seeded initialisation and the reference's surrogate 7-point
// stages. Compiled with --fmad=false so the recipe arithmetic rounds exactly
// like the host (-ffp-contract=off) and the two are bit-identical.
#include <cuda_runtime.h>

#include "mpdata_kernels.cuh"

namespace imb::dev {

namespace {

template <class T>
__global__ void k_init(recipe::Params prm, std::int64_t i0, std::int64_t R, std::int64_t planes,
                       T* __restrict__ x, T* __restrict__ u, T* __restrict__ v,
                       T* __restrict__ w, T* __restrict__ h) {
  const std::int64_t plane = prm.m * prm.l;
  const std::int64_t total = planes * plane;
  for (std::int64_t t = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
       t < total; t += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t p = t / plane, r = t % plane;
    std::int64_t gi = (i0 + p - R) % prm.n;
    if (gi < 0) gi += prm.n;
    double vals[5];
    recipe::cell(prm, gi, r / prm.l, r % prm.l, vals);
    x[t] = static_cast<T>(vals[0]);
    u[t] = static_cast<T>(vals[1]);
    v[t] = static_cast<T>(vals[2]);
    w[t] = static_cast<T>(vals[3]);
    h[t] = static_cast<T>(vals[4]);
  }
}

__global__ void k_stage7(const double* __restrict__ in, double* __restrict__ out, std::int64_t n,
                         std::int64_t m, std::int64_t l, std::int64_t halo, bool is_max) {
  const std::int64_t t = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n * m * l) return;
  const std::int64_t i = t / (m * l), j = (t / l) % m, k = t % l;
  const std::int64_t sm = m + 2 * halo, sl = l + 2 * halo;
  auto g = [&](std::int64_t a, std::int64_t b, std::int64_t c) {
    return in[((a + halo) * sm + (b + halo)) * sl + (c + halo)];
  };
  double r = g(i, j, k);
  const double nb[6] = {g(i - 1, j, k), g(i + 1, j, k), g(i, j - 1, k),
                        g(i, j + 1, k), g(i, j, k - 1), g(i, j, k + 1)};
#pragma unroll
  for (int q = 0; q < 6; ++q) r = is_max ? fmax(r, nb[q]) : fmin(r, nb[q]);
  out[((i + halo) * sm + (j + halo)) * sl + (k + halo)] = r;
}

}  // namespace

template <class T>
int launch_init(const recipe::Params& prm, std::int64_t i0, std::int64_t R, std::int64_t planes,
                T* x, T* u, T* v, T* w, T* h, cudaStream_t st) {
  k_init<T><<<148 * 8, 256, 0, st>>>(prm, i0, R, planes, x, u, v, w, h);
  return 1;
}
template int launch_init<double>(const recipe::Params&, std::int64_t, std::int64_t, std::int64_t,
                                 double*, double*, double*, double*, double*, cudaStream_t);
template int launch_init<float>(const recipe::Params&, std::int64_t, std::int64_t, std::int64_t,
                                float*, float*, float*, float*, float*, cudaStream_t);

int launch_stage7(const double* in, double* out, std::int64_t n, std::int64_t m, std::int64_t l,
                  std::int64_t halo, bool is_max, cudaStream_t st) {
  const std::int64_t cells = n * m * l;
  k_stage7<<<static_cast<unsigned>((cells + 255) / 256), 256, 0, st>>>(in, out, n, m, l, halo,
                                                                       is_max);
  return 1;
}

}  // namespace imb::dev
