#include <cstdio>
#include "dmlp_math.cuh"
using namespace dmlp;
template <int V>
__global__ void k(float x0, int n, float* out, long long* cyc) {
  float x = x0 + threadIdx.x * 1e-3f;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
    float t;
    if (V == 0) x = dev_tanhf(x) * 1.3f;
    else if (V == 1) x = dev_tanhf_branchy(x) * 1.3f;
    else x = dev_scaled_tanh(x, &t) * 0.9f;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / n;
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 8);
  for (float x0 : {0.05f, 0.3f, 0.8f, 2.0f}) for (int th : {1, 32}) {
    long long h[3];
    k<0><<<1, th>>>(x0, 1000, o, c); cudaMemcpy(&h[0], c, 8, cudaMemcpyDeviceToHost);
    k<1><<<1, th>>>(x0, 1000, o, c); cudaMemcpy(&h[1], c, 8, cudaMemcpyDeviceToHost);
    k<2><<<1, th>>>(x0, 1000, o, c); cudaMemcpy(&h[2], c, 8, cudaMemcpyDeviceToHost);
    printf("x0=%.2f threads=%d  select=%lld  branchy=%lld  scaled=%lld cycles/call\n", x0, th, h[0], h[1], h[2]);
  }
  return 0;
}
