// Poll pressure in a full-volume forward exchange (C4-like: 148 producers x
// R words, every CTA gathers all P*R words, thread t owns words t, t+512, ...).
// The hardware floor of one hop is the flag word's one-way latency (~1K
// cycles, xchg7_mb ping); what the consumers' polls add on top is measured
// here for several polling disciplines:
//   0: every thread keeps all its words in flight, re-polls the unready ones
//      each round (poll_batch, the kernel's discipline);
//   1: poll only the thread's first word until it is ready, then the rest
//      (one load in flight per thread while waiting);
//   2: as 0 with __nanosleep(S) between rounds;
//   3: as 1 with __nanosleep(S) between rounds of the first word.
#include <cstdio>
#include "train_phases.cuh"
using namespace dmlp;

constexpr int kMaxW = 8;

__global__ void __launch_bounds__(512, 1) k_vol(unsigned long long* buf, int R, int ylog, int iters,
                                                int mode, int sleep_ns, long long* out, int* err) {
  const int c = blockIdx.x, tid = threadIdx.x;
  const int P = gridDim.x, F = P * R;
  __shared__ float sink[512];
  int off[kMaxW];
#pragma unroll
  for (int u = 0; u < kMaxW; u++) {
    const int i = tid + 512 * u;
    off[u] = i < F ? ((i / R) << ylog) + (i % R) : -1;
  }
  const long long t0 = clock64();
  for (int it = 1; it <= iters; it++) {
    const uint32_t seq = it;
    unsigned long long* b = buf + ((size_t)(seq & 1) * P << ylog);
    if (tid < R) st_flag(b + ((size_t)c << ylog) + tid, 1.0f + tid, seq);
    unsigned long long v[kMaxW];
    if (mode == 1 || mode == 3) {
      if (off[0] >= 0) {
        unsigned long long w = ld_flag(b + off[0]);
        while ((uint32_t)(w >> 32) != seq) {
          if (mode == 3) __nanosleep(sleep_ns);
          w = ld_flag(b + off[0]);
        }
        v[0] = w;
      }
      int o2[kMaxW];
#pragma unroll
      for (int u = 0; u < kMaxW; u++) o2[u] = u == 0 ? -1 : off[u];
      unsigned long long v2[kMaxW];
      poll_batch<kMaxW>(b, o2, v2, seq, err);
#pragma unroll
      for (int u = 1; u < kMaxW; u++) v[u] = v2[u];
    } else {
#pragma unroll
      for (int u = 0; u < kMaxW; u++) v[u] = off[u] >= 0 ? ld_flag(b + off[u]) : 0ull;
      for (;;) {
        bool done = true;
#pragma unroll
        for (int u = 0; u < kMaxW; u++)
          if (off[u] >= 0 && (uint32_t)(v[u] >> 32) != seq) done = false;
        if (done) break;
        if (mode == 2) __nanosleep(sleep_ns);
#pragma unroll
        for (int u = 0; u < kMaxW; u++)
          if (off[u] >= 0 && (uint32_t)(v[u] >> 32) != seq) v[u] = ld_flag(b + off[u]);
      }
    }
    float a = 0.0f;
#pragma unroll
    for (int u = 0; u < kMaxW; u++) if (off[u] >= 0) a += __uint_as_float((uint32_t)v[u]);
    sink[tid] = a;
    asm volatile("barrier.sync 0;" ::: "memory");
  }
  const long long t1 = clock64();
  if (tid == 0) out[c] = (t1 - t0) / iters;
  if (sink[(tid + 1) & 511] == -1.0f) out[0] = 0;
}

int main() {
  unsigned long long* buf; long long* d; int* err;
  cudaMalloc(&buf, 1 << 24); cudaMalloc(&d, 148 * 8); cudaMalloc(&err, 4);
  long long h[148];
  for (int R : {4, 17, 27}) {
    int ylog = 0; while ((1 << ylog) < (R < 16 ? 16 : R)) ylog++;
    for (int mode = 0; mode < 4; mode++)
      for (int s : {0, 32, 128, 512}) {
        if ((mode == 0 || mode == 1) && s != 0) continue;
        if ((mode == 2 || mode == 3) && s == 0) continue;
        cudaMemset(buf, 0, 1 << 24);
        k_vol<<<148, 512>>>(buf, R, ylog, 3000, mode, s, d, err);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        long long mx = 0; for (int i = 0; i < 148; i++) mx = h[i] > mx ? h[i] : mx;
        printf("R=%2d words=%4d mode=%d sleep=%3dns: %lld cycles/hop (%s)\n", R, 148 * R, mode, s,
               mx, cudaGetErrorString(e));
      }
  }
  return 0;
}
