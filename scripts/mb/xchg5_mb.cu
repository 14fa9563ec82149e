// Cluster pre-combine vs flat publish for the all-to-all exchange.
// 148 CTAs x 512 threads in clusters of CS.  Flat: every CTA publishes R words
// in its own slot, every CTA polls all 148 slots.  Cluster: the CS CTAs of a
// cluster write their R words into the leader's smem (DSMEM), cluster barrier,
// the leader publishes CS*R words, every CTA polls 148/CS slots.
#include <cooperative_groups.h>
#include <cstdio>
#include "mb_common.cuh"
using namespace dmlp;
namespace cg = cooperative_groups;

template <int CS, bool COMBINE>
__global__ void __launch_bounds__(512, 1) k_x(int R, unsigned long long* buf, int iters,
                                               long long* out, int* err) {
  __shared__ float dst[4096];
  __shared__ float comb[64];
  cg::cluster_group cl = cg::this_cluster();
  const int c = blockIdx.x, tid = threadIdx.x;
  const int rank = (int)cl.block_rank();
  LayerDev ly{};
  const int P = COMBINE ? gridDim.x / CS : gridDim.x;
  const int RP = COMBINE ? R * CS : R;
  ly.R = RP; ly.fo = RP * P; ly.P = P;
  int lg = 0; while ((1 << lg) < (RP < 16 ? 16 : RP)) lg++;
  ly.ylog = lg;
  float* leader_comb = cl.map_shared_rank(comb, 0);
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    const uint32_t seq = it + 1;
    unsigned long long* b = buf + ((size_t)(seq & 1) * P << lg);
    if (!COMBINE) {
      if (tid < R) st_flag(b + ((size_t)c << lg) + tid, 1.0f * tid, seq);
    } else {
      if (tid < R) leader_comb[rank * R + tid] = 1.0f * tid + c;
      cl.sync();
      if (rank == 0 && tid < RP) st_flag(b + ((size_t)(c / CS) << lg) + tid, comb[tid], seq);
    }
    gather_y(b, ly, dst, seq, err);
    __syncthreads();
  }
  long long t1 = clock64();
  float a = 0; for (int i = 0; i < 32; i++) a += dst[(tid + i) & 1023];
  if (tid == 0) out[c] = (t1 - t0) / iters;
  if (a == 12345.f) out[0] = 0;
}

template <int CS, bool COMBINE>
void run(int R) {
  int* err; long long* d; unsigned long long* buf;
  cudaMalloc(&err, 4); cudaMalloc(&d, 148 * 8); cudaMalloc(&buf, 1 << 24); cudaMemset(buf, 0, 1 << 24);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = 0;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  int ncl = 0;
  cudaOccupancyMaxActiveClusters(&ncl, (void*)k_x<CS, COMBINE>, &cfg);
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_x<CS, COMBINE>, R, buf, 2000, d, err);
  cudaError_t e2 = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < 148; i++) mx = h[i] > mx ? h[i] : mx;
  printf("CS=%d combine=%d R=%d max co-resident clusters=%d (need %d): cycles/exchange=%lld %s %s\n",
         CS, (int)COMBINE, R, ncl, 148 / CS, mx, cudaGetErrorString(e), cudaGetErrorString(e2));
}
int main() {
  run<1, false>(7); run<2, false>(7); run<2, true>(7); run<4, false>(7); run<4, true>(7);
  run<1, false>(14); run<2, true>(14); run<4, true>(14);
  return 0;
}
