// Microbenchmark: forward dot of one owned row block (R rows x pitch) from smem,
// variants of the access path. One CTA per SM, 512 threads, clock64 per call.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int T = 512;
template <int CH>
__device__ __forceinline__ float xpose_reduce(float (&a)[CH], int lane) {
  int off = 16;
#pragma unroll
  for (int h = CH / 2; h >= 1; h >>= 1, off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < h; i++) {
      const float send = up ? a[i] : a[i + h];
      const float keep = up ? a[i + h] : a[i];
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
#pragma unroll
  for (int o = 16 / CH; o >= 1; o >>= 1) a[0] += __shfl_xor_sync(0xffffffffu, a[0], o);
  return a[0];
}
__device__ __forceinline__ float lds(unsigned a) { float v; asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a)); return v; }

// MODE 0: generic pointer, runtime C loop;  1: shared asm, runtime C;  2: shared asm, C unrolled (template)
template <int MODE, int CH, int CC>
__device__ __noinline__ float fwd(const float* W, unsigned Ws, int pitch, int C, int nr, const float* v, float* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float acc[CH];
#pragma unroll
  for (int j = 0; j < CH; j++) acc[j] = 0.f;
  if (MODE == 2) {
#pragma unroll
    for (int m = 0; m < CC; m++) {
      const int col = tid + m * T;
      if (col < pitch) {
        const float x = v[col];
#pragma unroll
        for (int j = 0; j < CH; j++) if (j < nr) acc[j] = fmaf(lds(Ws + 4u * (j * pitch + col)), x, acc[j]);
      }
    }
  } else {
    for (int m = 0; m < C; m++) {
      const int col = tid + m * T;
      if (col < pitch) {
        const float x = v[col];
#pragma unroll
        for (int j = 0; j < CH; j++) if (j < nr) {
          const float w = MODE == 0 ? W[j * pitch + col] : lds(Ws + 4u * (j * pitch + col));
          acc[j] = fmaf(w, x, acc[j]);
        }
      }
    }
  }
  const float s = xpose_reduce<CH>(acc, lane);
  if ((lane & (32 / CH - 1)) == 0) red[warp * CH + lane / (32 / CH)] = s;
  __syncthreads();
  float a = 0.f;
  if (tid < nr) for (int w = 0; w < 16; w++) a += red[w * CH + tid];
  __syncthreads();
  return a;
}

template <int MODE, int CH, int CC>
__global__ void __launch_bounds__(512, 1) k(int R, int pitch, int iters, long long* out, float* sink) {
  extern __shared__ float sm[];
  float* v = sm; float* red = sm + pitch; float* W = red + 16 * 32;
  for (int i = threadIdx.x; i < pitch + R * pitch + 512; i += T) sm[i] = 0.001f * (i % 97);
  __syncthreads();
  const unsigned Ws = (unsigned)__cvta_generic_to_shared(W);
  const int C = (pitch + T - 1) / T;
  float acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) acc += fwd<MODE, CH, CC>(W, Ws, pitch, C, R, v, red);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
  if (acc == 12345.f) sink[0] = acc;
}

template <int MODE, int CH, int CC>
void run(const char* name, int R, int pitch) {
  long long* d; float* s; cudaMalloc(&d, 148 * 8); cudaMalloc(&s, 4);
  int smem = (pitch + 512 + R * pitch) * 4;
  cudaFuncSetAttribute(k<MODE, CH, CC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<MODE, CH, CC><<<148, T, smem>>>(R, pitch, 2000, d, s);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < 148; i++) mx = h[i] > mx ? h[i] : mx;
  double bytes = 4.0 * R * pitch;
  printf("%-28s R=%2d pitch=%4d cycles/call=%6lld  smem B/clk=%.1f  %s\n", name, R, pitch, mx, bytes / mx, cudaGetErrorString(e));
  cudaFree(d); cudaFree(s);
}
int main() {
  run<0, 16, 5>("generic ptr, loop C", 14, 2504);
  run<1, 16, 5>("ld.shared asm, loop C", 14, 2504);
  run<2, 16, 5>("ld.shared asm, unrolled C", 14, 2504);
  run<0, 16, 2>("generic ptr, loop C", 17, 844);
  run<0, 16, 2>("generic ptr, loop C (16r)", 16, 844);
  run<1, 16, 2>("ld.shared, loop C (16r)", 16, 844);
  run<2, 16, 2>("ld.shared unrolled (16r)", 16, 844);
  run<0, 8, 2>("generic ptr, loop C", 7, 844);
  run<2, 8, 2>("ld.shared unrolled", 7, 844);
  run<0, 16, 4>("generic, loop", 11, 2004);
  run<2, 16, 4>("ld.shared unrolled", 11, 2004);
  return 0;
}
