// microbench.cu -- K6: roofline denominators and exchange-latency floor.
//
// * L2/HBM streaming read and read+write bandwidth with the persistent
//   kernel's geometry (one 512-thread CTA per SM, float4, .cg accesses),
//   for a buffer size chosen by the caller (L2-resident or not).
// * Shared-memory read+write bandwidth per SM.
// * Exchange hop latency: every CTA publishes one flag word per round and
//   polls all CTAs' words (the persistent kernel's gather pattern), so
//   cycles/round is the floor of one forward/backward exchange.
#include <cuda_runtime.h>

#include "dmlp_internal.h"
#include "dmlp_math.cuh"

namespace dmlp {

__global__ void __launch_bounds__(512, 1)
    k_bw(float4* buf, long long n4, int iters, int write, unsigned long long* cycles) {
  const long long start = clock64();
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (int it = 0; it < iters; it++) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n4; i += 8 * stride) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; u++) v[u] = __ldcg(buf + i + u * stride);
#pragma unroll
      for (int u = 0; u < 8; u++) {
        if (write) {
          v[u].x += 1.0f;
          __stcg(buf + i + u * stride, v[u]);
        } else {
          acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
        }
      }
    }
    for (; i < n4; i += stride) {
      float4 v = __ldcg(buf + i);
      if (write) { v.x += 1.0f; __stcg(buf + i, v); }
      else { acc.x += v.x; }
    }
  }
  if (acc.x == 12345.0f) buf[0] = acc;  // keep the loads alive
  if (threadIdx.x == 0) atomicMax(cycles, (unsigned long long)(clock64() - start));
}

__global__ void __launch_bounds__(512, 1) k_smem_bw(int iters, float* out, unsigned long long* cyc) {
  extern __shared__ __align__(16) float4 s4[];
  const int n4 = 8192;  // 128 KB
  for (int i = threadIdx.x; i < n4; i += blockDim.x) s4[i] = make_float4(i, 0, 0, 0);
  __syncthreads();
  const long long start = clock64();
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int it = 0; it < iters; it++) {
#pragma unroll 4
    for (int i = threadIdx.x; i < n4; i += blockDim.x) {
      float4 v = s4[i];
      acc.x += v.x; acc.y += v.y;
      v.z += 1.0f;
      s4[i] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(cyc, (unsigned long long)(clock64() - start));
  if (acc.x == 12345.0f) out[0] = acc.y;
}

__device__ __forceinline__ unsigned long long mb_ld(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mb_st(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long mb_ld_cg(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.global.cg.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// rounds of: publish {round} for this CTA; every thread tid < nct polls the
// word of CTA tid until it shows this round; __syncthreads.
// variant 0: contiguous words, ld.relaxed.gpu; 1: contiguous, ld.global.cg;
// 2: contiguous, relaxed + 64 ns backoff; 3: one 128-B line per producer;
// 4: 8 replicas (consumer c reads replica c%8), contiguous per replica;
// 5: 16 replicas.
__global__ void __launch_bounds__(512, 1)
    k_ping(unsigned long long* words, int rounds, unsigned base, int variant,
           unsigned long long* cyc) {
  const int c = blockIdx.x, n = gridDim.x;
  const int R = variant == 4 ? 8 : (variant == 5 ? 16 : 1);
  const int stride = (variant == 3 || variant == 6) ? 16 : 1;
  __syncthreads();
  const long long start = clock64();
  for (int r = 0; r < rounds; r++) {
    const unsigned seq = base + (unsigned)r;
    unsigned long long* w = words + (size_t)(seq & 1) * 16 * 148 * 148;
    const unsigned long long val = ((unsigned long long)seq << 32) | (unsigned)c;
    if (variant == 6) {  // mailbox: one line per (consumer, producer)
      if (threadIdx.x < n) mb_st(w + ((size_t)threadIdx.x * n + c) * 16, val);
    } else if (threadIdx.x < R) {
      mb_st(w + (size_t)threadIdx.x * 256 + (size_t)c * stride, val);
    }
    if (threadIdx.x < n) {
      const unsigned long long* p =
          variant == 6 ? w + ((size_t)c * n + threadIdx.x) * 16
                       : w + (size_t)(c % R) * 256 + (size_t)threadIdx.x * stride;
      unsigned long long v = variant == 1 ? mb_ld_cg(p) : mb_ld(p);
      while ((unsigned)(v >> 32) != seq) {
        if (variant == 2) __nanosleep(64);
        v = variant == 1 ? mb_ld_cg(p) : mb_ld(p);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicMax(cyc, (unsigned long long)(clock64() - start));
}

// Full exchange protocols at the kernel's volume: every CTA produces R values
// (one per warp, as the forward does) and needs all n*R values.  cycles/round.
//  A (0): per-word flag words, producer words written by R warps, consumer
//         thread t polls producer t's first word then reads the rest;
//  B (1): producer stages values in smem, ONE warp writes its flag-word line
//         (coalesced); consumer warps poll whole lines (16 lanes), ballot;
//  C (2): plain data stored coalesced by one warp, __threadfence, one flag
//         word per producer (own line); consumer warp 0 polls the n flags,
//         __syncthreads, everyone reads the data with .cg loads;
//  D (3): as C but the flag is a st.release.gpu (no explicit fence).
__global__ void __launch_bounds__(512, 1)
    k_xchg(unsigned long long* words, float* data, int rounds, int variant, int R,
           unsigned long long* cyc) {
  __shared__ float vals[32];
  __shared__ float got[148 * 32];
  const int c = blockIdx.x, n = gridDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int S = 32;  // slot words per producer (2 lines)
  if (R > 16) R = 16;
  __syncthreads();
  const long long start = clock64();
  for (int r = 0; r < rounds; r++) {
    const unsigned seq = 1u + (unsigned)r;
    unsigned long long* w = words + (size_t)(seq & 1) * n * S;
    float* d = data + (size_t)(seq & 1) * n * S;
    unsigned long long* f = words + (size_t)2 * n * S + (size_t)(seq & 1) * n * 16;
    const float myv = (float)(c * 100 + warp);
    if (variant == 0) {
      if (lane == 0 && warp < R)
        mb_st(w + (size_t)c * S + warp, ((unsigned long long)seq << 32) | __float_as_uint(myv));
      if (tid < n) {
        const unsigned long long* p = w + (size_t)tid * S;
        unsigned long long v = mb_ld(p);
        while ((unsigned)(v >> 32) != seq) v = mb_ld(p);
        got[tid * S] = __uint_as_float((unsigned)v);
        for (int k = 1; k < R; k++) {
          unsigned long long u = mb_ld(p + k);
          while ((unsigned)(u >> 32) != seq) u = mb_ld(p + k);
          got[tid * S + k] = __uint_as_float((unsigned)u);
        }
      }
    } else if (variant == 4 || variant == 5) {
      // E/F: line-aligned producer slots; every thread issues all its loads
      // (one producer line per warp instruction) and re-polls stragglers.
      if (variant == 4) {
        if (lane == 0 && warp < R) vals[warp] = myv;
        __syncthreads();
        if (warp == 0 && lane < R)
          mb_st(w + (size_t)c * S + lane,
                ((unsigned long long)seq << 32) | __float_as_uint(vals[lane]));
      } else if (lane == 0 && warp < R) {
        mb_st(w + (size_t)c * S + warp, ((unsigned long long)seq << 32) | __float_as_uint(myv));
      }
      constexpr int U = 10;  // ceil(148 / 16)
      unsigned long long v[U];
      const unsigned long long* pp[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int p = warp + 16 * u;
        const bool ok = p < n && lane < R;
        pp[u] = ok ? w + (size_t)p * S + lane : nullptr;
        v[u] = ok ? mb_ld(pp[u]) : 0ull;
      }
      for (;;) {
        bool done = true;
#pragma unroll
        for (int u = 0; u < U; u++)
          if (pp[u] && (unsigned)(v[u] >> 32) != seq) done = false;
        if (done) break;
#pragma unroll
        for (int u = 0; u < U; u++)
          if (pp[u] && (unsigned)(v[u] >> 32) != seq) v[u] = mb_ld(pp[u]);
      }
#pragma unroll
      for (int u = 0; u < U; u++)
        if (pp[u]) got[(warp + 16 * u) * S + lane] = __uint_as_float((unsigned)v[u]);
    } else if (variant == 1) {
      if (lane == 0 && warp < R) vals[warp] = myv;
      __syncthreads();
      if (warp == 0 && lane < R)
        mb_st(w + (size_t)c * S + lane, ((unsigned long long)seq << 32) | __float_as_uint(vals[lane]));
      for (int p = warp; p < n; p += 16) {
        const unsigned long long* q = w + (size_t)p * S + lane;
        bool ok;
        unsigned long long v = 0;
        do {
          v = lane < R ? mb_ld(q) : ((unsigned long long)seq << 32);
          ok = __all_sync(0xffffffffu, (unsigned)(v >> 32) == seq);
        } while (!ok);
        if (lane < R) got[p * S + lane] = __uint_as_float((unsigned)v);
      }
    } else {
      if (lane == 0 && warp < R) vals[warp] = myv;
      __syncthreads();
      if (warp == 0) {
        if (lane < R) __stcg(d + (size_t)c * S + lane, vals[lane]);
        __syncwarp();
        if (lane == 0) {
          if (variant == 2) {
            __threadfence();
            mb_st(f + (size_t)c * 16, seq);
          } else {
            asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(f + (size_t)c * 16),
                         "l"((unsigned long long)seq) : "memory");
          }
        }
        // poll all producers' flags
        for (int p0 = 0; p0 < n; p0 += 32) {
          const int p = p0 + lane;
          if (p < n) {
            unsigned long long v;
            do {
              if (variant == 2) v = mb_ld(f + (size_t)p * 16);
              else asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(f + (size_t)p * 16) : "memory");
            } while ((unsigned)v != seq);
          }
        }
        if (variant == 2) __threadfence();
      }
      __syncthreads();
      for (int i = tid; i < n * R; i += blockDim.x) {
        const int p = i / R, k = i - p * R;
        got[p * S + k] = __ldcg(d + (size_t)p * S + k);
      }
    }
    __syncthreads();
  }
  if (tid == 0) atomicMax(cyc, (unsigned long long)(clock64() - start));
  if (got[0] == -1.0f) data[0] = got[1];
}

// Latency of the primitives the sample loop chains (cycles per op, one CTA of
// 512 threads): out[0] __syncthreads, [1] exact scaled tanh (dependent
// chain), [2] __fdiv_rn chain, [3] 5-step warp shuffle reduction chain,
// [4] dependent L2 load chain (.cg), [5] dependent ld.relaxed.gpu chain,
// [6] smem load chain.
__global__ void __launch_bounds__(512, 1)
    k_prims(float* fbuf, unsigned long long* ubuf, double* out) {
  __shared__ int sidx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sidx[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  const int N = 1000;
  long long t0 = clock64();
  for (int i = 0; i < N; i++) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / N;
  float x = fbuf[threadIdx.x] * 1e-3f + 0.3f, t;
  t0 = clock64();
  for (int i = 0; i < N; i++) x = dev_scaled_tanh(x, &t) * 0.5f;
  t1 = clock64();
  if (threadIdx.x == 0) out[1] = (double)(t1 - t0) / N;
  float y = x + 1.5f;
  t0 = clock64();
  for (int i = 0; i < N; i++) y = __fdiv_rn(1.0f, y) + 1.0f;
  t1 = clock64();
  if (threadIdx.x == 0) out[2] = (double)(t1 - t0) / N;
  float z = y;
  t0 = clock64();
  for (int i = 0; i < N; i++) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) z += __shfl_xor_sync(0xffffffffu, z, s);
    z *= 1e-3f;
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[3] = (double)(t1 - t0) / N;
  // dependent global chains (thread 0 only)
  if (threadIdx.x == 0) {
    unsigned long long p = 0;
    t0 = clock64();
    for (int i = 0; i < 200; i++) p = __ldcg(ubuf + p);
    t1 = clock64();
    out[4] = (double)(t1 - t0) / 200;
    unsigned long long q = 0;
    t0 = clock64();
    for (int i = 0; i < 200; i++) {
      unsigned long long v;
      asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(ubuf + q) : "memory");
      q = v;
    }
    t1 = clock64();
    out[5] = (double)(t1 - t0) / 200;
    int k = 0;
    t0 = clock64();
    for (int i = 0; i < N; i++) k = sidx[k];
    t1 = clock64();
    out[6] = (double)(t1 - t0) / N;
    fbuf[0] = x + y + z + (float)(p + q + k);
  }
}

}  // namespace dmlp

using namespace dmlp;

namespace dmlp {
// Exhaustive check of the select-form tanhf against the branchy glibc
// restatement, over every 32-bit pattern [start, start + count).
__global__ void k_tanhf_check(unsigned long long start, unsigned long long count,
                              unsigned long long* bad, unsigned int* first) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
       i < count; i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint32_t u = (uint32_t)(start + i);
    const float x = u2f(u);
    const uint32_t a = f2u(dev_tanhf(x)), b = f2u(dev_tanhf_branchy(x));
    if (a != b && !((a & 0x7fffffffu) > 0x7f800000u && (b & 0x7fffffffu) > 0x7f800000u)) {
      atomicAdd(bad, 1ull);
      atomicMin(first, u);
    }
  }
}
// The training kernel's dev_tanhf_fast over every non-NaN float: st[0] inputs
// where it differs from the glibc restatement, st[1] the largest difference
// in ulp; st[2], st[3] the same against the correctly rounded tanh (CUDA's
// double tanh, rounded to float).
__global__ void k_tanhf_fast_check(unsigned long long* st) {
  unsigned long long dg = 0, dc = 0, mg = 0, mc = 0;
  for (unsigned long long u = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
       u < (1ull << 32); u += (unsigned long long)gridDim.x * blockDim.x) {
    const float x = u2f((uint32_t)u);
    if (x != x) continue;
    const long long a = (int32_t)f2u(dev_tanhf_fast(x)), g = (int32_t)f2u(dev_tanhf(x));
    const long long c = (int32_t)f2u(__double2float_rn(tanh((double)x)));
    const unsigned long long eg = (unsigned long long)(a > g ? a - g : g - a);
    const unsigned long long ec = (unsigned long long)(a > c ? a - c : c - a);
    dg += eg != 0;
    dc += ec != 0;
    mg = eg > mg ? eg : mg;
    mc = ec > mc ? ec : mc;
  }
  atomicAdd(st + 0, dg);
  atomicMax(st + 1, mg);
  atomicAdd(st + 2, dc);
  atomicMax(st + 3, mc);
}
__global__ void k_tanhf_fast_eval(const float* x, float* y, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = dev_tanhf_fast(x[i]);
}
__global__ void k_tanhf_eval(const float* x, float* y, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = dev_tanhf(x[i]);
}
}  // namespace dmlp

extern "C" {

int dmlp_tanhf_check(uint64_t* mismatches, uint32_t* first_bad) {
  unsigned long long* d = nullptr;
  unsigned int* f = nullptr;
  if (int rc = cuda_check(cudaMalloc(&d, 8), "cudaMalloc")) return rc;
  if (int rc = cuda_check(cudaMalloc(&f, 4), "cudaMalloc")) return rc;
  cudaMemset(d, 0, 8);
  cudaMemset(f, 0xff, 4);
  dmlp::k_tanhf_check<<<148 * 8, 256>>>(0ull, 1ull << 32, d, f);
  if (int rc = cuda_check(cudaGetLastError(), "k_tanhf_check")) return rc;
  if (int rc = cuda_check(cudaMemcpy(mismatches, d, 8, cudaMemcpyDeviceToHost), "cudaMemcpy"))
    return rc;
  if (int rc = cuda_check(cudaMemcpy(first_bad, f, 4, cudaMemcpyDeviceToHost), "cudaMemcpy"))
    return rc;
  cudaFree(d);
  cudaFree(f);
  return DMLP_OK;
}

int dmlp_tanhf_fast_check(uint64_t* stats) {
  unsigned long long* d = nullptr;
  if (int rc = cuda_check(cudaMalloc(&d, 32), "cudaMalloc")) return rc;
  cudaMemset(d, 0, 32);
  dmlp::k_tanhf_fast_check<<<148 * 8, 256>>>(d);
  int rc = cuda_check(cudaGetLastError(), "k_tanhf_fast_check");
  if (!rc) rc = cuda_check(cudaMemcpy(stats, d, 32, cudaMemcpyDeviceToHost), "cudaMemcpy");
  cudaFree(d);
  return rc;
}

int dmlp_tanhf_fast_eval(const float* x_dev, float* y_dev, int64_t n) {
  if (n <= 0) return DMLP_OK;
  dmlp::k_tanhf_fast_eval<<<148 * 4, 256>>>(x_dev, y_dev, n);
  return cuda_check(cudaGetLastError(), "k_tanhf_fast_eval");
}

int dmlp_tanhf_eval(const float* x_dev, float* y_dev, int64_t n) {
  if (n <= 0) return DMLP_OK;
  dmlp::k_tanhf_eval<<<148 * 4, 256>>>(x_dev, y_dev, n);
  return cuda_check(cudaGetLastError(), "k_tanhf_eval");
}

int dmlp_bench(int32_t kind, int64_t bytes, int32_t iters, int32_t n_ctas, double* seconds,
               double* cycles) {
  int dev = 0, sms = 148;
  if (int rc = cuda_check(cudaGetDevice(&dev), "cudaGetDevice")) return rc;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = n_ctas > 0 ? n_ctas : sms;
  unsigned long long* d_cyc = nullptr;
  if (int rc = cuda_check(cudaMalloc(&d_cyc, 8), "cudaMalloc")) return rc;
  cudaMemset(d_cyc, 0, 8);
  void* buf = nullptr;
  size_t alloc = kind <= 1 ? (size_t)bytes : (kind == 2 ? 64 : 2 * 16 * 148 * 148 * 8);
  if (int rc = cuda_check(cudaMalloc(&buf, alloc), "cudaMalloc")) {
    cudaFree(d_cyc);
    return rc;
  }
  cudaMemset(buf, 0, alloc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  if (kind <= 1) {  // warm the L2 then time
    k_bw<<<grid, 512>>>((float4*)buf, (long long)(bytes / 16), 1, kind, d_cyc);
    cudaMemset(d_cyc, 0, 8);
    cudaEventRecord(e0);
    k_bw<<<grid, 512>>>((float4*)buf, (long long)(bytes / 16), iters, kind, d_cyc);
    cudaEventRecord(e1);
  } else if (kind == 2) {
    cudaFuncSetAttribute(k_smem_bw, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    cudaEventRecord(e0);
    k_smem_bw<<<grid, 512, 131072>>>(iters, (float*)buf, d_cyc);
    cudaEventRecord(e1);
  } else if (kind == 5) {
    int variant = (int)(bytes & 0xff), R = (int)(bytes >> 8);
    float* data = nullptr;
    cudaMalloc(&data, (size_t)2 * 148 * 32 * 4);
    void* args[] = {&buf, &data, &iters, &variant, &R, &d_cyc};
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((const void*)k_xchg, dim3(grid), dim3(512), args, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaFree(data);
  } else {
    unsigned base = 1;
    int variant = (int)bytes;
    void* args[] = {&buf, &iters, &base, &variant, &d_cyc};
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((const void*)k_ping, dim3(grid), dim3(512), args, 0, 0);
    cudaEventRecord(e1);
  }
  cudaError_t e = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc = 0;
  cudaMemcpy(&cyc, d_cyc, 8, cudaMemcpyDeviceToHost);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  cudaFree(d_cyc);
  if (e != cudaSuccess) return cuda_check(e, "bench kernel");
  if (int rc = cuda_check(cudaGetLastError(), "bench launch")) return rc;
  if (seconds) *seconds = ms * 1e-3;
  if (cycles) *cycles = (double)cyc;
  return DMLP_OK;
}

int dmlp_bench_prims(double* out /* [8] */) {
  float* fb = nullptr;
  unsigned long long* ub = nullptr;
  double* d_out = nullptr;
  const int chase = 1 << 20;  // 8 MB pointer-chase table, stride 4 KB + 8 B
  if (int rc = cuda_check(cudaMalloc(&fb, 4096), "cudaMalloc")) return rc;
  cudaMalloc(&ub, (size_t)chase * 8);
  cudaMalloc(&d_out, 8 * sizeof(double));
  cudaMemset(fb, 0, 4096);
  cudaMemset(d_out, 0, 8 * sizeof(double));
  unsigned long long* h = new unsigned long long[chase];
  for (int i = 0; i < chase; i++) h[i] = (unsigned long long)((i + 513) % chase);
  cudaMemcpy(ub, h, (size_t)chase * 8, cudaMemcpyHostToDevice);
  delete[] h;
  k_prims<<<1, 512>>>(fb, ub, d_out);  // warm
  k_prims<<<1, 512>>>(fb, ub, d_out);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(out, d_out, 8 * sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(fb);
  cudaFree(ub);
  cudaFree(d_out);
  return cuda_check(e, "k_prims");
}

}  // extern "C"
