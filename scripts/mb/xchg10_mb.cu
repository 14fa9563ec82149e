// One-way flag latency vs (producer SM, consumer SM, home of the word):
// ping-pong between CTA 0 and CTA k (thread 0 each) on two words in one 2-KB
// granule g, for every k and 16 granules.  Prints the %smid of every CTA and
// the one-way latency matrix [k][g], to tell whether the hop cost depends on
// which die holds the line (xchg9_mb: 490..1060 cycles across pairs).
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ unsigned long long ldr(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void str(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void k_ping(unsigned long long* w, int other, int iters, long long* out, int* smid) {
  const int c = blockIdx.x;
  if (threadIdx.x == 0) {
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    smid[c] = (int)s;
  }
  if (threadIdx.x != 0 || (c != 0 && c != other)) return;
  unsigned long long* mine = w + (c == 0 ? 0 : 16);
  unsigned long long* theirs = w + (c == 0 ? 16 : 0);
  const long long t0 = clock64();
  for (int it = 1; it <= iters; it++) {
    if (c == 0) {
      str(mine, it);
      while (ldr(theirs) < (unsigned long long)it) {}
    } else {
      while (ldr(theirs) < (unsigned long long)it) {}
      str(mine, it);
    }
  }
  const long long t1 = clock64();
  if (c == 0) out[0] = (t1 - t0) / iters;
}

int main() {
  const int NG = 16;
  unsigned long long* w; long long* d; int* sm;
  cudaMalloc(&w, NG * 2048 + 4096); cudaMalloc(&d, 64); cudaMalloc(&sm, 148 * 4);
  int hsm[148];
  static long long lat[148][NG];
  for (int g = 0; g < NG; g++)
    for (int k = 1; k < 148; k++) {
      unsigned long long* wg = w + (size_t)g * 256;  // 2 KB granules
      cudaMemset(wg, 0, 256);
      k_ping<<<148, 32>>>(wg, k, 1500, d, sm);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      lat[k][g] = h / 2;
    }
  cudaMemcpy(hsm, sm, sizeof hsm, cudaMemcpyDeviceToHost);
  printf("smid:");
  for (int k = 0; k < 148; k++) printf(" %d", hsm[k]);
  printf("\n");
  for (int k = 1; k < 148; k++) {
    printf("k=%3d sm=%3d:", k, hsm[k]);
    for (int g = 0; g < NG; g++) printf(" %5lld", lat[k][g]);
    printf("\n");
  }
  return 0;
}
