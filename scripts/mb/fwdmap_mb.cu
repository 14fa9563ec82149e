// fwd_rows cost by thread mapping (G row groups, CH chunk) at one row-block shape, smem.
#include <cstdio>
#include "train_phases.cuh"
using namespace dmlp;
__global__ void __launch_bounds__(512, 1) k(int R, int pitch, int gs, int CH, int iters,
                                             unsigned long long* xb, long long* out, long long* sub) {
  extern __shared__ __align__(16) float sm[];
  float* v = sm; float* red = v + pitch; float* tc = red + 512; float* W = tc + 64;
  const int tid = threadIdx.x;
  for (int i = tid; i < pitch; i += 512) v[i] = 0.001f * (i % 13);
  for (int i = tid; i < R * pitch; i += 512) W[i] = 0.01f * (i % 7) - 0.03f;
  __shared__ long long ph[4];
  if (tid < 4) ph[tid] = 0;
  __syncthreads();
  LayerDev ly{}; ly.pitch = pitch; ly.gs = gs; ly.CH = CH;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    fwd_dispatch<true>(reinterpret_cast<const float4*>(W), ly, R, reinterpret_cast<const float4*>(v),
                       red, tc, nullptr, xb + blockIdx.x * 64, it + 1, (tid == 0) ? ph : nullptr);
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) { out[blockIdx.x] = (t1 - t0) / iters; if (blockIdx.x == 0) { sub[0] = ph[0] / iters; sub[1] = ph[1] / iters; } }
}
void run(int R, int fi, int gs, int CH) {
  const int pitch = (fi + 4) / 4 * 4;
  unsigned long long* xb; long long* d; long long* sub;
  cudaMalloc(&xb, 148 * 64 * 8); cudaMalloc(&d, 148 * 8); cudaMalloc(&sub, 16);
  const int smem = (pitch + 512 + 64 + R * pitch) * 4;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<148, 512, smem>>>(R, pitch, gs, CH, 500, xb, d, sub);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148], hs[2]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost); cudaMemcpy(hs, sub, 16, cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < 148; i++) mx = h[i] > mx ? h[i] : mx;
  printf("R=%2d fi=%4d G=%2d CH=%2d cycles=%5lld (loads..sync %lld, tree..store %lld) %s\n", R, fi, 1 << gs, CH, mx, hs[0], hs[1], cudaGetErrorString(e));
}
int main() {
  run(17, 841, 0, 16); run(17, 841, 1, 16); run(17, 841, 2, 8); run(17, 841, 3, 4);
  run(11, 2000, 0, 16); run(11, 2000, 1, 8); run(7, 1500, 0, 8); run(7, 841, 0, 8); run(4, 1000, 0, 4);
  return 0;
}
