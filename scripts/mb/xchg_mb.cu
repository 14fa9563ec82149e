// Exchange microbenchmark: 148 CTAs x 512 threads; per iteration every CTA
// "computes" for `work` cycles, publishes R flag words (threads < R), then
// gathers every producer's words with the kernel's own gather_y (protocol E)
// or a variant.  Reports cycles per iteration (slowest CTA).
#include <cstdio>
#include "mb_common.cuh"
using namespace dmlp;

__device__ __forceinline__ void spin(long long cyc) {
  const long long t0 = clock64();
  while (clock64() - t0 < cyc) {}
}

// V: 0 gather_y; 1 gather_y with __nanosleep backoff between rounds
template <int V>
__global__ void __launch_bounds__(512, 1) k_x(LayerDev ly, unsigned long long* buf, int iters,
                                               long long work, long long* out, int* err) {
  __shared__ float dst[4096];
  const int c = blockIdx.x, tid = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    const uint32_t seq = it + 1;
    unsigned long long* b = buf + ((size_t)(seq & 1) * ly.P << ly.ylog);
    if (work) spin(work);
    __syncthreads();
    if (c < ly.P && tid < ly.R) st_flag(b + ((size_t)c << ly.ylog) + tid, 1.0f * tid, seq);
    gather_y(b, ly, dst, seq, err);
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[c] = (t1 - t0) / iters;
}

int main() {
  int* err; long long* d; unsigned long long* buf;
  cudaMalloc(&err, 4); cudaMalloc(&d, 148 * 8); cudaMalloc(&buf, 1 << 24);
  for (int R : {7}) {
    for (long long work : {0LL}) {
      cudaMemset(buf, 0, 1 << 24);
      LayerDev ly{};
      ly.R = R; ly.fo = R * 148; ly.P = 148;
      int lg = 0; while ((1 << lg) < (R < 16 ? 16 : R)) lg++;
      ly.ylog = lg;
      for (int dyn : {0, 200 * 1024}) {
      cudaFuncSetAttribute(k_x<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
      k_x<0><<<148, 512, dyn>>>(ly, buf, 2000, work, d, err);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      long long mx = 0; for (int i = 0; i < 148; i++) mx = h[i] > mx ? h[i] : mx;
      printf("R=%2d work=%5lld dyn=%6d cycles/iter=%6lld (exchange ~%6lld) %s\n", R, work, dyn, mx, mx - work, cudaGetErrorString(e));
      }
    }
  }
  return 0;
}
