// bwd_partials / reg_partials / update costs in isolation (smem), with and without publishing.
#include <cstdio>
#include "train_phases.cuh"
using namespace dmlp;
template <int MODE>  // 0 bwd_partials smem, 1 update_rows smem, 2 reg_partials(14,4,1), 3 reg_update
__global__ void __launch_bounds__(512, 1) k(int R, int pitch, int fi, int iters, unsigned long long* xb, long long* out) {
  extern __shared__ __align__(16) float sm[];
  float* v = sm; float* dl = v + pitch; float* ds = dl + 32; float* pbuf = ds + 32; float* W = pbuf + 64;
  const int tid = threadIdx.x;
  for (int i = tid; i < pitch; i += 512) v[i] = 0.001f * (i % 13);
  for (int i = tid; i < 32; i += 512) { dl[i] = 1e-3f * i; ds[i] = 1e-6f * i; }
  for (int i = tid; i < R * pitch; i += 512) W[i] = 0.01f * (i % 7) - 0.03f;
  float w[14][4];
  reg_load<14, 4, 1>(w, W, W, pitch, R);
  __syncthreads();
  unsigned long long* slot = xb + (size_t)blockIdx.x * 4096;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    if (MODE == 0) bwd_partials<true, false>(reinterpret_cast<float4*>(W), pitch >> 2, fi, 0, R, dl, ds, reinterpret_cast<const float4*>(v), pbuf, slot, it + 1);
    if (MODE == 1) update_rows<true>(reinterpret_cast<float4*>(W), pitch >> 2, 0, R, reinterpret_cast<const float4*>(v), ds);
    if (MODE == 2) reg_partials<14, 4, 1>(w, W, fi, R, dl, slot, it + 1);
    if (MODE == 3) reg_update<14, 4, 1>(w, W, pitch, R, v, ds);
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = (t1 - t0) / iters;
  float a = 0; for (int k = 0; k < 14; k++) for (int m = 0; m < 4; m++) a += w[k][m];
  if (a == 1234.5f) out[1] = 1;
}
template <int MODE> void run(const char* nm, int R, int fi) {
  const int pitch = (fi + 4) / 4 * 4;
  unsigned long long* xb; long long* d; cudaMalloc(&xb, 148 * 4096 * 8); cudaMalloc(&d, 148 * 8);
  const int smem = (pitch + 128 + 14 * 512 + R * pitch) * 4 + 4096;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<MODE><<<148, 512, smem>>>(R, pitch, fi, 500, xb, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < 148; i++) mx = h[i] > mx ? h[i] : mx;
  printf("%-14s R=%2d fi=%4d cycles=%5lld %s\n", nm, R, fi, mx, cudaGetErrorString(e));
}
int main() {
  run<0>("bwd_partials", 11, 2000); run<0>("bwd_partials", 4, 1000); run<0>("bwd_partials", 7, 1000);
  run<1>("update_rows", 11, 2000); run<1>("update_rows", 17, 841); run<1>("update_rows", 7, 1000);
  run<2>("reg_partials", 14, 2500); run<3>("reg_update", 14, 2500);
  return 0;
}
