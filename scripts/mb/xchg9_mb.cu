// One-way latency of a flag word between two CTAs (ping-pong of thread 0 of
// CTA 0 and CTA k) for several store and poll flavours: is the ~1K-cycle hop
// of st.relaxed.gpu -> ld.relaxed.gpu (xchg7_mb) the store's drain, the
// poll, or the fabric?
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void store(unsigned long long* p, unsigned long long v, int kind) {
  switch (kind) {
    case 0: asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory"); break;
    case 1: asm volatile("st.volatile.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory"); break;
    case 2: asm volatile("st.global.cg.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory"); break;
    case 3: asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(p) : "memory"); break;
    case 4:
      asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      break;
    case 5: asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory"); break;
    default: asm volatile("st.global.wt.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory"); break;
  }
}
__device__ __forceinline__ unsigned long long load(const unsigned long long* p, int kind) {
  unsigned long long v;
  switch (kind) {
    case 0: asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); break;
    case 1: asm volatile("ld.volatile.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); break;
    case 2: asm volatile("ld.global.cv.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); break;
    default: asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); break;
  }
  return v;
}

__global__ void k_ping(unsigned long long* w, int other, int iters, int sk, int lk, long long* out) {
  const int c = blockIdx.x;
  if (threadIdx.x != 0 || (c != 0 && c != other)) return;
  unsigned long long* mine = w + (c == 0 ? 0 : 32);
  unsigned long long* theirs = w + (c == 0 ? 32 : 0);
  const long long t0 = clock64();
  for (int it = 1; it <= iters; it++) {
    const unsigned long long want = (unsigned long long)it;
    if (c == 0) {
      store(mine, want, sk);
      while (load(theirs, lk) < want) {}
    } else {
      while (load(theirs, lk) < want) {}
      store(mine, want, sk);
    }
  }
  const long long t1 = clock64();
  if (c == 0) out[0] = (t1 - t0) / iters;
}

// dependent load latency of the poll flavours on a line another SM wrote
__global__ void k_lat(unsigned long long* w, int lk, long long* out) {
  if (threadIdx.x != 0) return;
  unsigned long long v = 0;
  const long long t0 = clock64();
  for (int i = 0; i < 1000; i++) v = load(w + (v & 1), lk);
  const long long t1 = clock64();
  out[1] = (t1 - t0) / 1000 + (v == 12345 ? 1 : 0);
}

int main() {
  unsigned long long* w; long long* d;
  cudaMalloc(&w, 1 << 16); cudaMalloc(&d, 64);
  long long h[2];
  const char* sn[] = {"st.relaxed.gpu", "st.volatile", "st.cg", "red.add", "st+fence.acq_rel", "st.relaxed.sys", "st.wt"};
  const char* ln[] = {"ld.relaxed.gpu", "ld.volatile", "ld.cv", "ld.acquire.gpu"};
  for (int lk = 0; lk < 4; lk++) {
    cudaMemset(w, 0, 1 << 16);
    k_lat<<<1, 32>>>(w, lk, d);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("dependent %-15s latency %lld cycles\n", ln[lk], h[1]);
  }
  for (int sk = 0; sk < 7; sk++)
    for (int lk = 0; lk < 4; lk++) {
      long long best = 1LL << 60, worst = 0;
      for (int other : {1, 37, 74, 111, 147}) {
        cudaMemset(w, 0, 1 << 16);
        k_ping<<<148, 32>>>(w, other, 10000, sk, lk, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        best = h[0] < best ? h[0] : best;
        worst = h[0] > worst ? h[0] : worst;
      }
      printf("%-17s -> %-15s one-way %5lld .. %5lld cycles\n", sn[sk], ln[lk], best / 2, worst / 2);
    }
  return 0;
}
