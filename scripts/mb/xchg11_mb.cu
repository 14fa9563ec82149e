// Backward (reduce-scatter) exchange: flat vs 2-CTA-cluster pre-combine.
// 148 CTAs x 512 threads.  Every CTA holds F column partials.  Flat: each
// CTA publishes all F (st_flag4, as bwd_partials), every consumer sums its
// nr rows over 148 producers (the kernel's gather_sum).  Pair: the CTAs of a
// 2-CTA cluster split the columns in halves; each writes the partner's half
// of its partials into the partner's shared memory (DSMEM), cluster barrier,
// each adds and publishes its half -- half the stores, 74 producers to poll.
#include <cooperative_groups.h>
#include <cstdio>
#include "mb_common.cuh"
using namespace dmlp;
namespace cg = cooperative_groups;

__device__ __forceinline__ void st_flag4_256(unsigned long long* p, float4 x, int valid,
                                             uint32_t seq) {
  const unsigned long long h = (unsigned long long)seq << 32;
  if (valid >= 4)
    asm volatile("st.relaxed.gpu.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p),
                 "l"(h | __float_as_uint(x.x)), "l"(h | __float_as_uint(x.y)),
                 "l"(h | __float_as_uint(x.z)), "l"(h | __float_as_uint(x.w))
                 : "memory");
  else
    st_flag4(p, x, valid, seq);
}

template <bool PAIR, bool V256 = false>
__global__ void __launch_bounds__(512, 1) k_x(int F, int nr, unsigned long long* buf, int iters,
                                               long long* out, int* err) {
  __shared__ float red[512];
  __shared__ float res[64];
  __shared__ __align__(16) float recv[1280];  // partner's half of the partials (F <= 2560)
  cg::cluster_group cl = cg::this_cluster();
  const int c = blockIdx.x, tid = threadIdx.x;
  const int stride = (F + 15) / 16 * 16;
  const int P = PAIR ? gridDim.x / 2 : gridDim.x;
  const int half = (F / 2 + 3) / 4 * 4;  // column split, quad aligned
  const int rank = PAIR ? (int)cl.block_rank() : 0;
  float* peer = PAIR ? cl.map_shared_rank(recv, rank ^ 1) : recv;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    const uint32_t seq = it + 1;
    unsigned long long* b = buf + (size_t)(seq & 1) * P * stride;
    if (!PAIR) {
      for (int q = tid; 4 * q < F; q += blockDim.x) {
        const float4 p = make_float4(c + 1.f, c + 2.f, c + 3.f, c + 4.f);
        if (V256) st_flag4_256(b + (size_t)c * stride + 4 * q, p, F - 4 * q, seq);
        else st_flag4(b + (size_t)c * stride + 4 * q, p, F - 4 * q, seq);
      }
    } else {
      const int lo = rank ? half : 0, hi = rank ? F : half;         // my columns
      const int plo = rank ? 0 : half, phi = rank ? half : F;       // partner's columns
      for (int q = tid; plo + 4 * q < phi; q += blockDim.x)          // DSMEM: partner's half
        reinterpret_cast<float4*>(peer)[q] = make_float4(c + 1.f, c + 2.f, c + 3.f, c + 4.f);
      cl.sync();
      for (int q = tid; lo + 4 * q < hi; q += blockDim.x) {
        const float4 r = reinterpret_cast<const float4*>(recv)[q];
        const float4 p = make_float4(c + 1.f + r.x, c + 2.f + r.y, c + 3.f + r.z, c + 4.f + r.w);
        st_flag4(b + (size_t)(c >> 1) * stride + lo + 4 * q, p, hi - lo - 4 * q, seq);
      }
    }
    const int r0 = (c * nr) % (F - nr);
    gather_sum(b, stride, P, r0, nr, red, seq, err, [&](int k, float a) { res[k] = a; });
    if (PAIR) cl.sync();  // recv is rewritten by the partner next iteration
  }
  long long t1 = clock64();
  if (tid == 0) out[c] = (t1 - t0) / iters;
  if (res[0] == 12345.f) out[0] = 0;
}

template <bool PAIR, bool V256 = false>
void run(int F, int nr) {
  int* err; long long* d; unsigned long long* buf;
  cudaMalloc(&err, 4); cudaMalloc(&d, 148 * 8); cudaMalloc(&buf, 1 << 26);
  cudaMemset(buf, 0, 1 << 26); cudaMemset(err, 0, 4);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = 0;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = PAIR ? 2 : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_x<PAIR, V256>, F, nr, buf, 2000, d, err);
  cudaError_t e2 = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < 148; i++) mx = h[i] > mx ? h[i] : mx;
  printf("%s%s F=%4d nr=%2d cycles/exchange=%lld %s %s\n", PAIR ? "pair" : "flat", V256 ? "-256b" : "", F, nr, mx,
         cudaGetErrorString(e), cudaGetErrorString(e2));
  cudaFree(err); cudaFree(d); cudaFree(buf);
}
int main() {
  const int Fs[] = {1000, 1500, 2000, 2500}, nrs[] = {7, 11, 14, 17};
  for (int rep = 0; rep < 2; rep++)
    for (int i = 0; i < 4; i++) { run<false>(Fs[i], nrs[i]); run<false, true>(Fs[i], nrs[i]); }
  return 0;
}
