// Backward (reduce-scatter) exchange with consumer-homed words.  Every column
// partial has exactly one consumer (the owner of that row in the layer below),
// so the words of consumer c can live in 2-KB granules homed on c's die
// (granules and SMs classified by load latency, as die_mb.cu).  148 CTAs x 512
// threads; consumer c owns nr rows; its region is [148 producers][16 words]
// (one 128-B line per producer entry, nr <= 16 padded to whole sectors),
// split over 2-KB granules (16 entries each).  Producer p writes its 148 x nr
// partials as 256-bit flag-word quads; consumer c polls its nr words of every
// producer (warp w: producers w, w+16, ...; lane k: row k; batches of 10
// polls per lane, the kernel's gather_sum) and sums them in fixed order.
// Modes: 0 contiguous (default hashing), 1 consumer's die, 2 the other die.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_1003_0358_b200/csrc \
//        scripts/mb/xchg12_mb.cu -o /tmp/xchg12_mb && /tmp/xchg12_mb
#include <algorithm>
#include <cstdio>
#include <vector>
#include "train_phases.cuh"
using namespace dmlp;

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__global__ void k_lat(const float* pool, int ngran, int* lat) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  float acc = 0;
  for (int g = 0; g < ngran; g++) {
    const float* p = pool + (size_t)g * 512;
    const long long t0 = clock64();
    float v;
    asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    acc += v;
    lat[g] = (int)(clock64() - t0);
  }
  if (acc == 1234.5f) lat[0] = 0;
}

// per CTA: 1 if it is on CTA 0's die (a near granule loads faster than a far one)
__global__ void k_die(const float* nearg, const float* farg, int* die) {
  if (threadIdx.x != 0) return;
  float acc = 0;
  long long bn = 1 << 30, bf = 1 << 30;
  for (int r = 0; r < 8; r++) {
    float v;
    long long t0 = clock64();
    asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(nearg + r) : "memory");
    acc += v;
    long long t1 = clock64();
    asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(farg + r) : "memory");
    acc += v;
    long long t2 = clock64();
    bn = min(bn, t1 - t0);
    bf = min(bf, t2 - t1);
  }
  die[blockIdx.x] = (bn < bf ? 0 : 1) + (acc == 1234.5f);
}

constexpr int kP = 148, kEnt = 16, kGpr = kP / 16 + 1;  // granules per consumer region

// gt[(buf * kP + c) * kGpr + g]: granule g of consumer c's region for buffer buf
__global__ void __launch_bounds__(512, 1)
    k_x(int nr, unsigned long long** gt, const unsigned long long* base, int iters, long long* out,
        int* err) {
  __shared__ float red[512];
  __shared__ float res[32];
  const int c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nq = (nr + 3) / 4;  // quads per consumer entry
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    const uint32_t seq = it + 1;
    unsigned long long** g = gt + (size_t)(seq & 1) * kP * kGpr;
    // publish: quad (d, q) = rows 4q.. of consumer d, as 256-bit stores
    for (int i = tid; i < kP * nq; i += 512) {
      const int d = i / nq, q = i - d * nq;
      unsigned long long* e = g[d * kGpr + (c >> 4)] + (c & 15) * kEnt + 4 * q;
      const float v = c + 1.0f;
      st_flag4(e, make_float4(v, v, v, v), 4, seq);
    }
    // gather: warp w sums producers w, w + 16, ... (lane k: row k)
    const bool kv = lane < nr;
    float acc = 0.0f;
    int off[kGatherU];
    unsigned long long v[kGatherU];
    unsigned long long* const* mine = g + c * kGpr;  // word offsets from the pool base
#pragma unroll
    for (int u = 0; u < kGatherU; u++) {
      const int p = warp + 16 * u;
      off[u] = (kv && p < kP) ? (int)((mine[p >> 4] + (p & 15) * kEnt + lane) - base) : -1;
    }
    poll_batch<kGatherU>(base, off, v, seq, err);
#pragma unroll
    for (int u = 0; u < kGatherU; u++)
      if (off[u] >= 0) acc += __uint_as_float((uint32_t)v[u]);
    red[warp * 32 + lane] = acc;
    __syncthreads();
    if (tid < nr) {
      float s = 0.0f;
      for (int w = 0; w < 16; w++) s += red[w * 32 + tid];
      res[tid] = s;
    }
    __syncthreads();
  }
  if (tid == 0) out[c] = (clock64() - t0) / iters;
  if (res[0] == 12345.f) out[0] = 0;
}

int main() {
  const int NG = 32768;  // 64 MB pool of 2-KB granules
  float* pool;
  cudaMalloc(&pool, (size_t)NG * 2048);
  cudaMemset(pool, 0, (size_t)NG * 2048);
  int* dlat;
  cudaMalloc(&dlat, NG * 4);
  k_lat<<<1, 32>>>(pool, NG, dlat);
  cudaDeviceSynchronize();
  std::vector<int> lat(NG);
  cudaMemcpy(lat.data(), dlat, NG * 4, cudaMemcpyDeviceToHost);
  std::vector<int> s = lat;
  std::sort(s.begin(), s.end());
  const int thr = (s[NG / 4] + s[3 * NG / 4]) / 2;
  std::vector<int> g0, g1;  // near / far of CTA 0
  for (int g = 1; g < NG; g++) (lat[g] < thr ? g0 : g1).push_back(g);
  int* ddie;
  cudaMalloc(&ddie, kP * 4);
  k_die<<<kP, 32>>>(pool + (size_t)g0[0] * 512, pool + (size_t)g1[0] * 512, ddie);
  cudaDeviceSynchronize();
  std::vector<int> die(kP);
  cudaMemcpy(die.data(), ddie, kP * 4, cudaMemcpyDeviceToHost);
  int n0 = 0;
  for (int c = 0; c < kP; c++) n0 += die[c] == 0;
  printf("granule latency p25 %d p75 %d; CTAs on CTA0's die %d of %d\n", s[NG / 4],
         s[3 * NG / 4], n0, kP);
  // the gather uses 32-bit word offsets from the pool base (64 MB: 8M words)
  const unsigned long long* pbase = reinterpret_cast<const unsigned long long*>(pool);
  std::vector<unsigned long long*> h(2 * kP * kGpr);
  unsigned long long** dg;
  cudaMalloc(&dg, h.size() * sizeof(void*));
  int* err;
  cudaMalloc(&err, 4);
  cudaMemset(err, 0, 4);
  long long* dout;
  cudaMalloc(&dout, kP * 8);
  for (int nr : {7, 11, 14, 16}) {
    for (int mode = 0; mode < 3; mode++) {
      size_t i0 = 0, i1 = 0, nx = 0;
      for (int b = 0; b < 2; b++)
        for (int c = 0; c < kP; c++)
          for (int k = 0; k < kGpr; k++) {
            int g;
            const bool own0 = die[c] == 0;
            if (mode == 0) g = 1 + (int)(nx++);
            else if ((mode == 1) == own0) g = g0[i0++];
            else g = g1[i1++];
            h[(b * kP + c) * kGpr + k] = reinterpret_cast<unsigned long long*>(pool + (size_t)g * 512);
          }
      cudaMemset(pool, 0, (size_t)NG * 2048);
      cudaMemcpy(dg, h.data(), h.size() * sizeof(void*), cudaMemcpyHostToDevice);
      long long best = 1LL << 60;
      for (int rep = 0; rep < 2; rep++) {
        int iters = 1000 + 1000 * rep;
        void* args[] = {&nr, &dg, &pbase, &iters, &dout, &err};
        cudaMemset(pool, 0, (size_t)NG * 2048);
        cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_x, dim3(kP), dim3(512), args, 0, 0);
        cudaError_t e2 = cudaDeviceSynchronize();
        long long ho[kP];
        cudaMemcpy(ho, dout, sizeof ho, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int c = 0; c < kP; c++) mx = std::max(mx, ho[c]);
        best = std::min(best, mx);
        if (e != cudaSuccess || e2 != cudaSuccess)
          printf("error %s %s\n", cudaGetErrorString(e), cudaGetErrorString(e2));
      }
      printf("nr=%2d %s: %lld cycles per exchange (max over CTAs)\n", nr,
             mode == 0 ? "contiguous      " : mode == 1 ? "consumer's die  " : "other die       ",
             best);
    }
  }
  return 0;
}
