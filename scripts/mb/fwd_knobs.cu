// Which part of fwd_rows costs what: knob bits remove pieces.
#include <cstdio>
#include "train_phases.cuh"
using namespace dmlp;
template <bool RES, int CH, int K>
__device__ __forceinline__ void fwdk(const float* __restrict__ W, int pitch, int G, int C, int nr,
                                      const float* __restrict__ v, float* red, float* tc,
                                      float* yown, unsigned long long* yslot, uint32_t seq) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int TG = kThreads / G, g = tid / TG, u = tid - g * TG, WG = kWarps / G;
  const int nj = nr > g ? (nr - g + G - 1) / G : 0;
  const int njmax = (nr + G - 1) / G;
  for (int j0 = 0; j0 < njmax; j0 += CH) {
    float acc[CH];
#pragma unroll
    for (int jj = 0; jj < CH; jj++) acc[jj] = 0.0f;
    const int jn = nj - j0;
    const float* Wg = W + (size_t)(g + G * j0) * pitch;
    if (!(K & 1))
    for (int m = 0; m < C; m += 2) {
      const int c0 = u + m * TG, c1 = c0 + TG;
      const bool ok0 = c0 < pitch, ok1 = m + 1 < C && c1 < pitch;
      float w0[CH], w1[CH];
#pragma unroll
      for (int jj = 0; jj < CH; jj++) {
        w0[jj] = (ok0 && jj < jn) ? ldw<RES>(Wg + (size_t)jj * G * pitch + c0) : 0.0f;
        w1[jj] = (ok1 && jj < jn) ? ldw<RES>(Wg + (size_t)jj * G * pitch + c1) : 0.0f;
      }
      const float x0 = ok0 ? v[c0] : 0.0f, x1 = ok1 ? v[c1] : 0.0f;
#pragma unroll
      for (int jj = 0; jj < CH; jj++) acc[jj] = fmaf(w1[jj], x1, fmaf(w0[jj], x0, acc[jj]));
    }
    float s = acc[0];
    if (!(K & 2)) s = xpose_reduce<CH>(acc, lane);
    if ((lane & (32 / CH - 1)) == 0) red[warp * CH + lane / (32 / CH)] = s;
    __syncthreads();
    if (!(K & 4) && tid < G * CH) {
      const int gg = tid / CH, jj = tid - gg * CH;
      const int k = gg + G * (j0 + jj);
      if (k < nr) {
        float a = red[(gg * WG) * CH + jj];
        for (int w = gg * WG + 1; w < (gg + 1) * WG; w++) a += red[w * CH + jj];
        float t = a, y = a;
        if (!(K & 8)) y = tanh_scaled_noinline(a, &t);
        tc[k] = t;
        if (yown) yown[k] = y;
        if (!(K & 16) && yslot) st_flag(yslot + k, y, seq);
      }
    }
    if (j0 + CH < njmax) __syncthreads();
  }
}
template <int K, int CH>
__global__ void __launch_bounds__(kThreads, 1) kk(int R, int pitch, int G, int C, unsigned long long* xbuf, int iters, long long* out) {
  extern __shared__ __align__(16) float sm[];
  float* v = sm; float* red = v + pitch; float* tc = red + 512; float* W = tc + 32;
  const int tid = threadIdx.x;
  for (int i = tid; i < pitch; i += kThreads) v[i] = 0.001f * (i % 13);
  for (int i = tid; i < R * pitch; i += kThreads) W[i] = 0.01f * (i % 7);
  __syncthreads();
  unsigned long long* slot = xbuf + (size_t)blockIdx.x * 4096;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) { fwdk<true, CH, K>(W, pitch, G, C, R, v, red, tc, nullptr, slot, it + 1); __syncthreads(); }
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = (t1 - t0) / iters;
}
template <int K, int CH>
void run(int R, int fi, int G) {
  const int pitch = (fi + 4) / 4 * 4; const int C = (pitch + kThreads / G - 1) / (kThreads / G);
  unsigned long long* xb; long long* d; cudaMalloc(&xb, 148 * 4096 * 8); cudaMalloc(&d, 148 * 8);
  int smem = (pitch + 512 + 32 + R * pitch) * 4;
  cudaFuncSetAttribute(kk<K, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kk<K, CH><<<148, kThreads, smem>>>(R, pitch, G, C, xb, 500, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < 148; i++) mx = h[i] > mx ? h[i] : mx;
  printf("knobs=%2d (noload %d noreduce %d nofinal %d notanh %d nostore %d) R=%d fi=%d G=%d CH=%d cycles=%lld %s\n", K, K&1, (K>>1)&1, (K>>2)&1, (K>>3)&1, (K>>4)&1, R, fi, G, CH, mx, cudaGetErrorString(e));
  cudaFree(xb); cudaFree(d);
}
int main() {
  run<0, 8>(7, 841, 1); run<16, 8>(7, 841, 1); run<8, 8>(7, 841, 1); run<24, 8>(7, 841, 1);
  run<28, 8>(7, 841, 1); run<30, 8>(7, 841, 1); run<31, 8>(7, 841, 1); run<1, 8>(7, 841, 1);
  run<0, 16>(14, 2500, 1); run<8, 16>(14, 2500, 1); run<28, 16>(14, 2500, 1); run<30, 16>(14, 2500, 1);
  return 0;
}
