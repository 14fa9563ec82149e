// Exchange microbenchmark, kernel-shaped: NL layers per "sample", each with
// its own double-buffered slot array; between exchanges every CTA runs the
// real forward routine (fwd_rows, smem-resident R x pitch block, exact tanh,
// st_flag publish) -- so the measured per-exchange time includes exactly the
// kernel's compute+publish+gather sequence.  mode 0: compute + exchange,
// mode 1: exchange only (publish zeros), mode 2: compute only.
#include <cstdio>
#include "mb_common.cuh"
using namespace dmlp;

__global__ void __launch_bounds__(512, 1) k_x(int R, int pitch, int NL, unsigned long long* buf,
                                               int iters, int mode, long long* out, int* err,
                                               int NB) {
  extern __shared__ __align__(16) float sm[];
  float* v = sm;                 // pitch
  float* red = v + pitch;        // 512
  float* tc = red + 512;         // 64
  float* W = tc + 64;            // R*pitch
  const int c = blockIdx.x, tid = threadIdx.x;
  for (int i = tid; i < pitch; i += 512) v[i] = (i % 7) * 0.01f;
  for (int i = tid; i < R * pitch; i += 512) W[i] = (i % 5) * 0.001f;
  LayerDev ly{};
  ly.R = R; ly.fo = R * 148; ly.P = 148; ly.pitch = pitch; ly.gs = 0;
  ly.CH = R <= 4 ? 4 : R <= 8 ? 8 : 16;
  int lg = 0; while ((1 << lg) < (R < 16 ? 16 : R)) lg++;
  ly.ylog = lg;
  const size_t per = (size_t)2 * 148 << lg;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    const uint32_t seq = it + 1;
    for (int l = 0; l < NL; l++) {
      unsigned long long* b = buf + per * l + ((size_t)(NB == 2 ? (seq & 1) : 0) * 148 << lg);
      unsigned long long* mine = b + ((size_t)c << lg);
      if (mode != 1) {
        fwd_dispatch<true>(reinterpret_cast<const float4*>(W), ly, R,
                           reinterpret_cast<const float4*>(v), red, tc, nullptr,
                           mode == 0 ? mine : nullptr, seq);
      } else if (tid < R) {
        st_flag(mine + tid, 0.5f, seq);
      }
      if (mode != 2) gather_y(b, ly, v, seq, err);
      __syncthreads();
    }
  }
  long long t1 = clock64();
  if (tid == 0) out[c] = (t1 - t0) / ((long long)iters * NL);
}

int main() {
  int* err; long long* d; unsigned long long* buf;
  cudaMalloc(&err, 4); cudaMalloc(&d, 148 * 8); cudaMalloc(&buf, 1 << 26);
  for (int R : {7}) {
    const int pitch = 1004;
    for (int NL : {1, 5})
    for (int NB : {1, 2})
    for (int mode : {0, 1}) {
      cudaMemset(buf, 0, 1 << 26);
      const int smem = (pitch + 512 + 64 + R * pitch) * 4;
      cudaFuncSetAttribute(k_x, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k_x<<<148, 512, smem>>>(R, pitch, NL, buf, 400, mode, d, err, NB);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      long long mx = 0; for (int i = 0; i < 148; i++) mx = h[i] > mx ? h[i] : mx;
      printf("R=%2d NL=%d NB=%d mode=%d (%s) cycles per layer=%6lld %s\n", R, NL, NB, mode,
             mode == 0 ? "compute+exchange" : mode == 1 ? "exchange only" : "compute only", mx,
             cudaGetErrorString(e));
    }
  }
  return 0;
}
