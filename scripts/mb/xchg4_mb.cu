// Does the all-to-all exchange get cheaper with fewer (bigger) producers?
// NP producer CTAs publish R words each (same total words), all 148 CTAs gather.
#include <cstdio>
#include "mb_common.cuh"
using namespace dmlp;
__global__ void __launch_bounds__(512, 1) k_x(LayerDev ly, unsigned long long* buf, int iters,
                                               long long* out, int* err) {
  extern __shared__ float dst[];
  const int c = blockIdx.x, tid = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    const uint32_t seq = it + 1;
    unsigned long long* b = buf + ((size_t)(seq & 1) * ly.P << ly.ylog);
    if (c < ly.P && tid < ly.R) st_flag(b + ((size_t)c << ly.ylog) + tid, 1.0f * tid, seq);
    gather_y(b, ly, dst, seq, err);
    __syncthreads();
  }
  long long t1 = clock64();
  float a = 0; for (int i = 0; i < 32; i++) a += dst[(tid + i) & 1023];
  if (tid == 0) out[c] = (t1 - t0) / iters;
  if (a == 12345.f) out[0] = 0;
}
void run(int NP, int R) {
  int* err; long long* d; unsigned long long* buf;
  cudaMalloc(&err, 4); cudaMalloc(&d, 148 * 8); cudaMalloc(&buf, 1 << 24); cudaMemset(buf, 0, 1 << 24);
  LayerDev ly{}; ly.R = R; ly.fo = R * NP; ly.P = NP;
  int lg = 0; while ((1 << lg) < (R < 16 ? 16 : R)) lg++; ly.ylog = lg;
  cudaFuncSetAttribute(k_x, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  k_x<<<148, 512, 16384>>>(ly, buf, 2000, d, err);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < 148; i++) mx = h[i] > mx ? h[i] : mx;
  printf("producers=%3d R=%2d words=%d cycles/exchange=%lld %s\n", NP, R, NP * R, mx, cudaGetErrorString(e));
}
int main() { run(148, 7); run(74, 14); run(37, 28); run(148, 14); run(74, 28); run(19, 28); run(10, 28); run(1, 28); return 0; }
