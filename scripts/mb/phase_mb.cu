// Phase microbenchmark: times the persistent kernel's own phase routines
// (paper_1003_0358_b200/csrc/train_phases.cuh) in isolation, one CTA per SM,
// at the row-block shapes of the BASELINE configs.  cycles per call, slowest CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1003_0358_b200/csrc phase_mb.cu -o phase_mb
#include <cstdio>
#include "train_phases.cuh"
using namespace dmlp;

// which: 0 fwd, 1 bwd partial (smem: partial only / global: fused), 2 update
template <bool RES>
__global__ void __launch_bounds__(kThreads, 1)
    k_phase(int which, int R, int pitch, int fi, int G, int C, int CH, float* gw,
            unsigned long long* xbuf, int iters, long long* out) {
  extern __shared__ __align__(16) float sm[];
  float* v = sm;                       // pitch
  float* red = v + pitch;              // 512
  float* tc = red + 512;               // 32
  float* dl = tc + 32;                 // 32
  float* ds = dl + 32;                 // 32
  float* pbuf = ds + 32;               // G*pitch
  float* W = RES ? pbuf + G * pitch : gw + (size_t)blockIdx.x * R * pitch;
  const int tid = threadIdx.x;
  for (int i = tid; i < pitch; i += kThreads) v[i] = 0.001f * (i % 13);
  for (int i = tid; i < 32; i += kThreads) { dl[i] = 1e-3f * i; ds[i] = 1e-6f * i; }
  if (RES) for (int i = tid; i < R * pitch; i += kThreads) W[i] = 0.01f * (i % 7);
  __syncthreads();
  LayerDev ly{};
  ly.pitch = pitch; ly.fi = fi; ly.G = G; ly.C = C; ly.CH = CH;
  unsigned long long* slot = xbuf + (size_t)blockIdx.x * 4096;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    if (which == 0) fwd_dispatch<RES>(W, ly, R, v, red, tc, nullptr, slot, it + 1);
    else if (which == 1) {
      if (RES) bwd_partials<true, false>(W, pitch, fi, G, C, R, dl, ds, v, pbuf, slot, it + 1);
      else bwd_partials<false, true>(W, pitch, fi, G, C, R, dl, ds, v, pbuf, slot, it + 1);
    } else update_rows<RES>(W, pitch, G, C, R, v, ds);
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = (t1 - t0) / iters;
}

static void run(const char* name, bool res, int which, int R, int fi) {
  const int pitch = (fi + 1 + 3) / 4 * 4;
  int best = 1 << 30, G = 1, C = 1;
  for (int g = 1; g <= kWarps; g *= 2) {
    const int TG = kThreads / g, c = (pitch + TG - 1) / TG, nj = (R + g - 1) / g;
    const int cost = c * nj + (g > 1 ? 2 : 0) + 8 * ((nj + 15) / 16 - 1);
    if (cost < best) { best = cost; G = g; C = c; }
  }
  const int nj = (R + G - 1) / G;
  const int CH = nj <= 4 ? 4 : nj <= 8 ? 8 : 16;
  float* gw; unsigned long long* xb; long long* d;
  cudaMalloc(&gw, (size_t)148 * R * pitch * 4); cudaMemset(gw, 0, (size_t)148 * R * pitch * 4);
  cudaMalloc(&xb, 148 * 4096 * 8); cudaMalloc(&d, 148 * 8);
  const int smem = (pitch + 512 + 96 + G * pitch + (res ? R * pitch : 0)) * 4;
  auto k = res ? k_phase<true> : k_phase<false>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<148, kThreads, smem>>>(which, R, pitch, fi, G, C, CH, gw, xb, 500, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < 148; i++) mx = h[i] > mx ? h[i] : mx;
  const double bytes = 4.0 * R * pitch * (which == 2 || (which == 1 && !res) ? 2 : 1);
  printf("%-8s %-5s R=%2d fi=%4d G=%d C=%d CH=%2d  cycles=%6lld  B/clk/SM=%6.1f  %s\n", name,
         res ? "smem" : "L2", R, fi, G, C, CH, mx, bytes / mx, cudaGetErrorString(e));
  cudaFree(gw); cudaFree(xb); cudaFree(d);
}

int main() {
  const int shapes[][2] = {{17, 841}, {14, 2500}, {11, 2000}, {7, 1500}, {4, 1000}, {7, 841}, {7, 1000}};
  const char* nm[] = {"fwd", "bwdpart", "update"};
  for (int w = 0; w < 3; w++)
    for (auto& s : shapes) {
      run(nm[w], true, w, s[0], s[1]);
      run(nm[w], false, w, s[0], s[1]);
    }
  return 0;
}
