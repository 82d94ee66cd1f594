// Bitwise check of the packed fp32 pair helpers (mpdata_math.cuh P2) against
// the scalar fp32 forms, on random operands. Build: nvcc --fmad=false.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "mpdata_math.cuh"
using namespace imb::dev;
constexpr int NF = 10;
__global__ void k(const float* in, unsigned* bad, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (2 * i + 1 >= n / 11) return;
  const float* a = in + 22 * i;
  float s[NF][2];
  P2 p[NF];
  for (int h = 0; h < 2; ++h) {
    const float* o = a + 11 * h;
    s[0][h] = o[0] + o[1];
    s[1][h] = o[0] - o[1];
    s[2][h] = o[0] * o[1];
    s[3][h] = upflux(o[0], o[1], o[2]);
    s[4][h] = limit_sel(o[2], o[3], o[4], o[5], o[6]);
    s[5][h] = qdiv(o[0], o[1]);
    s[6][h] = rcp_rn(o[1]);
    s[7][h] = pseudo_face<float>(o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7], o[8], o[9], o[10]);
    s[8][h] = tmax(o[0], o[1]);
    s[9][h] = 0.5f * o[0] + Eps<float>::value;
  }
  auto G = [&](int q) { return P2{a[q], a[11 + q]}; };
  p[0] = G(0) + G(1);
  p[1] = G(0) - G(1);
  p[2] = G(0) * G(1);
  p[3] = upflux(G(0), G(1), G(2));
  p[4] = limit_sel(G(2), G(3), G(4), G(5), G(6));
  p[5] = qdiv(G(0), G(1));
  p[6] = rcp_rn(G(1));
  p[7] = pseudo_face(G(0), G(1), G(2), G(3), G(4), G(5), G(6), G(7), G(8), G(9), G(10));
  p[8] = tmax(G(0), G(1));
  p[9] = splat2(0.5f) * G(0) + splat2(Eps<float>::value);
  for (int f = 0; f < NF; ++f) {
    if (__float_as_uint(p[f].x) != __float_as_uint(s[f][0])) atomicAdd(&bad[2 * f], 1u);
    if (__float_as_uint(p[f].y) != __float_as_uint(s[f][1])) atomicAdd(&bad[2 * f + 1], 1u);
  }
}
int main() {
  const int n = 22 * 1 << 20;
  float* h = (float*)malloc(n * 4);
  srand(1);
  for (int i = 0; i < n; ++i) h[i] = (rand() / (float)RAND_MAX) * 4.0f - 1.0f + ((i % 11) == 1 ? 2.5f : 0.f);
  float* d; unsigned* b;
  cudaMalloc(&d, n * 4); cudaMalloc(&b, 2 * NF * 4); cudaMemset(b, 0, 2 * NF * 4);
  cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
  k<<<(n / 22 + 255) / 256, 256>>>(d, b, n);
  unsigned hb[2 * NF];
  cudaMemcpy(hb, b, sizeof hb, cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  const char* nm[NF] = {"add", "sub", "mul", "upflux", "limit_sel", "qdiv", "rcp_rn", "pseudo_face", "tmax", "mul_add"};
  for (int f = 0; f < NF; ++f) printf("%-12s mismatches lo %u hi %u\n", nm[f], hb[2 * f], hb[2 * f + 1]);
  return 0;
}
