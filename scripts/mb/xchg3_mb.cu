#include <cstdio>
#include "mb_common.cuh"
using namespace dmlp;
// V0: sync, publish, gather (static dst); V1: no pre-publish sync; V2: dynamic dst;
// V3: publish by threads 0..R-1 then gather into dynamic smem, no pre-sync (xchg2 mode 1)
template <int V>
__global__ void __launch_bounds__(512, 1) k_x(LayerDev ly, unsigned long long* buf, int iters,
                                               long long* out, int* err) {
  __shared__ float sdst[4096];
  extern __shared__ float ddst[];
  float* dst = (V >= 2 && V != 4) ? ddst : sdst;
  const int c = blockIdx.x, tid = threadIdx.x;
  __shared__ long long tp[2];
  if (tid == 0) tp[0] = tp[1] = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    const uint32_t seq = it + 1;
    unsigned long long* b = buf + ((size_t)(seq & 1) * ly.P << ly.ylog);
    if (V == 0 || V == 2) __syncthreads();
    if (c < ly.P && tid < ly.R) st_flag(b + ((size_t)c << ly.ylog) + tid, 1.0f * tid, seq);
    if (V == 5) {
      // inline gather_y with a stamp after the poll
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      int off[kGatherU];
      unsigned long long v[kGatherU];
      const long long ta = clock64();
#pragma unroll
      for (int u = 0; u < kGatherU; u++) {
        const int p = warp + kWarps * u;
        off[u] = (p < ly.P && lane < ly.R) ? (p << ly.ylog) + lane : -1;
      }
      poll_batch<kGatherU>(b, off, v, seq, err);
      const long long tb = clock64();
#pragma unroll
      for (int u = 0; u < kGatherU; u++)
        if (off[u] >= 0) sdst[(off[u] >> ly.ylog) * ly.R + (off[u] & 15)] = __uint_as_float((uint32_t)v[u]);
      const long long tc = clock64();
      if (tid == 0) { tp[0] += tb - ta; tp[1] += tc - tb; }
    } else
    gather_y(b, ly, dst, seq, err);
    __syncthreads();
  }
  long long t1 = clock64();
  if (V == 4 || V == 5) { float a = 0; for (int i = 0; i < 64; i++) a += sdst[(tid + i) & 4095]; if (a == 1234.5f) out[0] = 0; }
  if (tid == 0) out[c] = (t1 - t0) / iters;
  if (V == 5 && tid == 0 && c == 0) printf("  V5 cta0: poll %lld stores %lld per iter\n", tp[0] / iters, tp[1] / iters);
}
template <int V> void run(int R) {
  int* err; long long* d; unsigned long long* buf;
  cudaMalloc(&err, 4); cudaMalloc(&d, 148 * 8); cudaMalloc(&buf, 1 << 24); cudaMemset(buf, 0, 1 << 24);
  LayerDev ly{}; ly.R = R; ly.fo = R * 148; ly.P = 148;
  int lg = 0; while ((1 << lg) < (R < 16 ? 16 : R)) lg++; ly.ylog = lg;
  const int dyn = V >= 2 ? 16384 : 0;
  cudaFuncSetAttribute(k_x<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
  k_x<V><<<148, 512, dyn>>>(ly, buf, 2000, d, err);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < 148; i++) mx = h[i] > mx ? h[i] : mx;
  printf("V=%d R=%d cycles/iter=%lld %s\n", V, R, mx, cudaGetErrorString(e));
}
int main() { run<0>(7); run<4>(7); run<5>(7); return 0; }
