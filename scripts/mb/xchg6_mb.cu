// Backward-pattern exchange: P producers each publish F column partials
// (st_flag4 by F/4 threads, as bwd_partials does), every consumer sums its nr
// rows over the P producers with the kernel's gather_sum; vs the forward
// pattern (R words per producer, own-column quads).
#include <cstdio>
#include "mb_common.cuh"
using namespace dmlp;

template <bool BWD>
__global__ void __launch_bounds__(512, 1) k_x(int P, int F, int nr, unsigned long long* buf,
                                               int iters, long long* out, int* err) {
  __shared__ float red[512];
  __shared__ float res[64];
  const int c = blockIdx.x, tid = threadIdx.x;
  const int stride = (F + 15) / 16 * 16;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    const uint32_t seq = it + 1;
    unsigned long long* b = buf + (size_t)(seq & 1) * P * stride;
    if (c < P && 4 * tid < F) {
      float4 p = make_float4(1.f, 2.f, 3.f, 4.f);
      st_flag4(b + (size_t)c * stride + 4 * tid, p, F - 4 * tid, seq);
    }
    const int r0 = (c * nr) % F;
    gather_sum(b, stride, P, r0, nr, red, seq, err, [&](int k, float a) { res[k] = a; });
  }
  long long t1 = clock64();
  if (tid == 0) out[c] = (t1 - t0) / iters;
  if (res[0] == 12345.f) out[0] = 0;
}

void run(int P, int F, int nr) {
  int* err; long long* d; unsigned long long* buf;
  cudaMalloc(&err, 4); cudaMalloc(&d, 148 * 8); cudaMalloc(&buf, 1 << 26); cudaMemset(buf, 0, 1 << 26);
  k_x<true><<<148, 512>>>(P, F, nr, buf, 2000, d, err);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < 148; i++) mx = h[i] > mx ? h[i] : mx;
  printf("bwd pattern P=%3d F=%4d nr=%2d cycles/exchange=%lld %s\n", P, F, nr, mx, cudaGetErrorString(e));
  cudaFree(err); cudaFree(d); cudaFree(buf);
}
int main() {
  run(148, 1000, 8); run(148, 2000, 8); run(148, 2500, 17); run(148, 64, 8); run(148, 8, 8);
  run(125, 1000, 8); run(74, 1000, 8);
  return 0;
}
