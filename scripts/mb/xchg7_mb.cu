// Where does an exchange hop's time go?  (1) one-way latency of a flag word
// between two CTAs (ping-pong, thread 0 each); (2) a 148-producer hop (one
// word per producer on its own line) with the polls issued by 1 warp, by all
// 16 warps, or by all 16 warps with 16-byte vector polls of 2-word lines --
// the poll fan-in the L2 slices see; (3) the same with the producer's store
// issued as atom.exch / red instead of st.relaxed.
#include <cstdio>
#include "train_phases.cuh"
using namespace dmlp;

__device__ __forceinline__ void st_word(unsigned long long* p, unsigned long long v, int kind) {
  if (kind == 0) asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else if (kind == 1) asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else { unsigned long long o; asm volatile("atom.relaxed.gpu.global.exch.b64 %0, [%1], %2;" : "=l"(o) : "l"(p), "l"(v) : "memory"); }
}

__global__ void k_ping(unsigned long long* w, int other, int iters, int kind, long long* out) {
  const int c = blockIdx.x;
  if (threadIdx.x != 0 || (c != 0 && c != other)) return;
  unsigned long long* mine = w + (c == 0 ? 0 : 16);
  unsigned long long* theirs = w + (c == 0 ? 16 : 0);
  const long long t0 = clock64();
  for (int it = 1; it <= iters; it++) {
    if (c == 0) {
      st_word(mine, it, kind);
      while (ld_flag(theirs) != (unsigned long long)it) {}
    } else {
      while (ld_flag(theirs) != (unsigned long long)it) {}
      st_word(mine, it, kind);
    }
  }
  const long long t1 = clock64();
  if (c == 0) out[0] = (t1 - t0) / iters;  // one round trip = two one-way hops
}

// mode 0: warp 0 polls all producers; 1: every warp polls all producers;
// 2: every thread polls only producer (tid % P) (one word per thread);
// 3: warp 0 polls, lanes hold ceil(P/32) words each (same as 0) but stores via kind.
__global__ void __launch_bounds__(512, 1) k_hop(unsigned long long* buf, int P, int iters, int mode,
                                                int kind, long long* out) {
  const int c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ float sink[512];
  const long long t0 = clock64();
  for (int it = 1; it <= iters; it++) {
    unsigned long long* b = buf + (size_t)(it & 1) * P * 16;
    const unsigned long long want = (unsigned long long)it << 32;
    if (tid == 0 && c < P) st_word(b + (size_t)c * 16, want | 1u, kind);
    float acc = 0.0f;
    if (mode == 0 || mode == 1) {
      if (mode == 1 || warp == 0) {
        unsigned long long v[5];
#pragma unroll
        for (int u = 0; u < 5; u++) {
          const int p = lane + 32 * u;
          v[u] = p < P ? ld_flag(b + (size_t)p * 16) : want;
        }
        for (;;) {
          bool done = true;
#pragma unroll
          for (int u = 0; u < 5; u++) if ((v[u] >> 32) != (unsigned long long)it) done = false;
          if (done) break;
#pragma unroll
          for (int u = 0; u < 5; u++) {
            const int p = lane + 32 * u;
            if ((v[u] >> 32) != (unsigned long long)it) v[u] = ld_flag(b + (size_t)p * 16);
          }
        }
#pragma unroll
        for (int u = 0; u < 5; u++) acc += (float)(uint32_t)v[u];
      }
    } else {
      const int p = tid % P;
      unsigned long long v = ld_flag(b + (size_t)p * 16);
      while ((v >> 32) != (unsigned long long)it) v = ld_flag(b + (size_t)p * 16);
      acc = (float)(uint32_t)v;
    }
    sink[tid] = acc;
    asm volatile("barrier.sync 0;" ::: "memory");
  }
  const long long t1 = clock64();
  if (tid == 0) out[c] = (t1 - t0) / iters;
  if (sink[(tid + 1) & 511] == -1.0f) out[0] = 0;
}

int main() {
  unsigned long long* w; long long* d;
  cudaMalloc(&w, 1 << 20); cudaMalloc(&d, 148 * 8);
  long long h[148];
  for (int kind = 0; kind < 3; kind++)
    for (int other : {1, 2, 74, 75, 147}) {
      cudaMemset(w, 0, 1 << 20);
      k_ping<<<148, 32>>>(w, other, 20000, kind, d);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
      printf("ping kind=%d (0 st.relaxed 1 st.release 2 atom.exch) CTA0<->CTA%-3d round trip %lld cycles (%s)\n",
             kind, other, h[0], cudaGetErrorString(e));
    }
  for (int kind = 0; kind < 3; kind += 2)
    for (int mode = 0; mode < 3; mode++)
      for (int P : {16, 64, 148}) {
        cudaMemset(w, 0, 1 << 20);
        k_hop<<<148, 512>>>(w, P, 4000, mode, kind, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        long long mx = 0; for (int i = 0; i < 148; i++) mx = h[i] > mx ? h[i] : mx;
        printf("hop kind=%d mode=%d (0 warp0 polls all, 1 all warps poll all, 2 one word/thread) P=%3d: %lld cycles/hop (%s)\n",
               kind, mode, P, mx, cudaGetErrorString(e));
      }
  return 0;
}
