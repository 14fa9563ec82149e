// The kernel's own forward of one smem-resident row block (fwd_rows from
// train_phases.cuh, with its sub-profile), in isolation: 148 CTAs x 512
// threads, C4 layer shapes.  Compares with the in-kernel per-layer profile
// (bench line: profile_cycles_per_layer) to separate the phase's own cost
// from contention / instruction fetch inside the persistent kernel.
#include <cstdio>
#include "train_phases.cuh"
using namespace dmlp;

template <int CH>
__global__ void __launch_bounds__(512, 1) k_f(int R, int pitch, int gs, int iters,
                                              unsigned long long* slots, long long* out) {
  extern __shared__ __align__(16) float sm[];
  float* W = sm;
  float* v = W + R * pitch;
  float* red = v + pitch;
  float* tc = red + 2 * kWarps * 32;
  for (int i = threadIdx.x; i < R * pitch; i += 512) W[i] = 1e-3f * ((i * 7) % 13 - 6);
  for (int i = threadIdx.x; i < pitch; i += 512) v[i] = 1e-2f * ((i * 5) % 11 - 5);
  __syncthreads();
  __shared__ long long sub[4];
  if (threadIdx.x < 4) sub[threadIdx.x] = 0;
  __syncthreads();
  long long* sp = threadIdx.x == 0 ? sub : nullptr;
  const long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    fwd_rows<true, CH>(reinterpret_cast<const float4*>(W), pitch / 4, gs, R,
                       reinterpret_cast<const float4*>(v), red + (it & 1) * kWarps * 32, tc,
                       nullptr, slots + (size_t)blockIdx.x * 64, (uint32_t)it, sp);
    __syncthreads();
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 3 + 0] = (t1 - t0) / iters;
    out[blockIdx.x * 3 + 1] = sub[0] / iters;
    out[blockIdx.x * 3 + 2] = sub[1] / iters;
  }
}

template <int CH>
void run(const char* name, int R, int pitch, int gs) {
  unsigned long long* slots; long long* d;
  cudaMalloc(&slots, 148 * 64 * 8); cudaMalloc(&d, 148 * 3 * 8);
  const int smem = (R * pitch + pitch + 2 * kWarps * 32 + 64) * 4;
  cudaFuncSetAttribute(k_f<CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_f<CH><<<148, 512, smem>>>(R, pitch, gs, 2000, slots, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148 * 3]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  long long a = 0, b = 0, c = 0;
  for (int i = 0; i < 148; i++) { a += h[3 * i]; b += h[3 * i + 1]; c += h[3 * i + 2]; }
  printf("%-22s R=%2d pitch=%4d G=%d CH=%2d: %5lld cycles/layer (dot+reduce+barrier %5lld, tree+tanh+publish %5lld) %s\n",
         name, R, pitch, 1 << gs, CH, a / 148, b / 148, c / 148, cudaGetErrorString(e));
}


// The tail alone: tree over the warp partials, scaled tanh, publish.
// MODE 0: as fwd_rows; 1: no tanh (y = a); 2: no tree (a = red[tid]).
template <int CH, int MODE>
__global__ void __launch_bounds__(512, 1) k_tail(int nr, int iters, unsigned long long* slots,
                                                 long long* out) {
  __shared__ float red[2 * kWarps * 32], tc[64];
  for (int i = threadIdx.x; i < 2 * kWarps * 32; i += 512) red[i] = 1e-3f * (i % 7);
  __syncthreads();
  long long acc = 0;
  const int tid = threadIdx.x;
  for (int it = 0; it < iters; it++) {
    const long long t0 = clock64();
    if (tid < nr) {
      const float a = MODE == 2 ? red[tid + (it & 1)] : tree_sum<CH>(red + (it & 1) * 32 + tid, kWarps);
      float t = a;
      const float y = MODE == 1 ? a * 1.5f : tanh_scaled_noinline(a, &t);
      tc[tid] = t;
      st_flag(slots + (size_t)blockIdx.x * 64 + tid, y, (uint32_t)it);
    }
    const long long t1 = clock64();
    acc += t1 - t0;
    __syncthreads();
  }
  if (tid == 0) out[blockIdx.x] = acc / iters;
}

template <int CH, int MODE>
void run_tail(const char* name, int nr) {
  unsigned long long* slots; long long* d;
  cudaMalloc(&slots, 148 * 64 * 8); cudaMalloc(&d, 148 * 8);
  k_tail<CH, MODE><<<148, 512>>>(nr, 2000, slots, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  long long a = 0; for (int i = 0; i < 148; i++) a += h[i];
  printf("tail %-28s nr=%2d CH=%2d: %5lld cycles (thread 0) %s\n", name, nr, CH, a / 148, cudaGetErrorString(e));
}

int main() {
  run<16>("C4 L0 (smem)", 17, 844, 1);
  run<16>("C4 L2 (smem)", 11, 2004, 0);
  run<8>("C4 L3 (if smem)", 7, 1504, 0);
  run<4>("C4 L4 (smem)", 4, 1004, 0);
  run<4>("C1 L1 (smem)", 4, 1004, 0);
  run_tail<16, 0>("tree+tanh+publish", 17);
  run_tail<16, 1>("tree+publish (no tanh)", 17);
  run_tail<16, 2>("tanh+publish (no tree)", 17);
  run_tail<4, 0>("tree+tanh+publish", 4);
  return 0;
}
