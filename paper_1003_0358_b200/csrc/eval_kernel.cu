// eval_kernel.cu -- batched evaluation forward on sm_100a.
//
// Replaces network.forward_batch (network.py:118-130), rank_outputs
// (network.py:133-135), trainer.error_percent (trainer.py:90-96) and the
// counting of eval_report.evaluate (eval_report.py:36-67).
//   * hidden layers: fp32 SIMT GEMM (128x128 CTA tile, 8x8 per thread,
//     double-buffered smem, float4 row loads transposed into k-major tiles)
//     with the bias add and the scaled tanh fused in the epilogue.  fp32 accumulation keeps argmax parity with the
//     reference's OpenBLAS sgemm; tensor-core tf32 would not.
//   * output layer: one warp per sample (10 rows, weights in smem), fused
//     with stable top-2 ranking and the {wrong, confusion, second-guess}
//     counters (block-aggregated, one atomic per counter per CTA).
// The samples are processed in chunks so the activation scratch stays
// bounded; chunks reuse the net's scratch buffers.
#include <cuda_runtime.h>

#include "dmlp_internal.h"
#include "dmlp_math.cuh"

namespace dmlp {

constexpr int BM = 128, BN = 128, BK = 16, GT = 256;

// Y[m][j] = A*tanh(B*(sum_k X[m][k] W[j][k] + W[j][K])), m < M, j < N.
// 128x128 CTA tile, 8x8 outer products per thread over k-major smem tiles
// (As[k][m], Bs[k][n]: one LDS.128 per 4 fragment values), double-buffered
// smem fed from registers.  The global loads are row-major float4s (VEC:
// rows 16-byte aligned, ld % 4 == 0; else scalar): thread t loads row
// t % 128, k-half t / 128 of both tiles, so every warp stores 32 consecutive
// m (or n) of one k row -- conflict-free transposes (C4 33.2 -> 36.7 TFLOP/s;
// a 3-stage pipeline of transposing 4-byte cp.async measured 27.8, and one
// CTA per SM with more registers 34.6).  Thread (ty, tx) owns rows
// ty*4 + {0..3, 64..67} and columns tx*4 + {0..3, 64..67}.
// Packed fp32 pairs for FFMA2 (fma.rn.f32x2: two independent round-to-nearest
// FMAs per instruction -- the same results as two fmaf).  On sm_100 a scalar
// FFMA issues at most every other cycle per SMSP, so the fp32 SIMT peak needs
// the packed form; the broadcast operand (a, a) becomes a scalar .F32
// operand in SASS, no extra moves.
__device__ __forceinline__ unsigned long long pack2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void fma2(unsigned long long& acc, unsigned long long a,
                                     unsigned long long b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}
__device__ __forceinline__ float2 unpack2(unsigned long long v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return make_float2(a, b);
}

template <bool VEC>
__global__ void __launch_bounds__(GT, 2)
    k_gemm_tanh(const float* __restrict__ X, long long ldx, const float* __restrict__ W, int ldw,
                int M, int N, int K, float* __restrict__ Y, int ldy) {
#ifndef DMLP_EVAL_KB
#define DMLP_EVAL_KB 16
#endif
  constexpr int KB = DMLP_EVAL_KB;  // k per smem tile
  constexpr int NL = KB / 8;        // float4 loads per thread per matrix per tile
  __shared__ __align__(16) float As[2][KB][BM];
  __shared__ __align__(16) float Bs[2][KB][BN];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int bm = blockIdx.y * BM, bn = blockIdx.x * BN;
  const int lr = tid & 127, lk = (tid >> 7) * 4;  // loader: row, first of 4 k (+ 8 r)
  const bool am = bm + lr < M, bnv = bn + lr < N;
  const float* xa = X + (long long)(am ? bm + lr : 0) * ldx;
  const float* wb = W + (long long)(bnv ? bn + lr : 0) * ldw;
  float4 ra[NL], rb[NL];
  auto load = [&](int k0) {
#pragma unroll
    for (int r = 0; r < NL; r++) {
      const int kb = k0 + lk + 8 * r;
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      if (VEC && kb + 4 <= K) {
        ra[r] = am ? *reinterpret_cast<const float4*>(xa + kb) : z;
        rb[r] = bnv ? __ldg(reinterpret_cast<const float4*>(wb + kb)) : z;
      } else {
        ra[r].x = (am && kb < K) ? xa[kb] : 0.f;
        ra[r].y = (am && kb + 1 < K) ? xa[kb + 1] : 0.f;
        ra[r].z = (am && kb + 2 < K) ? xa[kb + 2] : 0.f;
        ra[r].w = (am && kb + 3 < K) ? xa[kb + 3] : 0.f;
        rb[r].x = (bnv && kb < K) ? __ldg(wb + kb) : 0.f;
        rb[r].y = (bnv && kb + 1 < K) ? __ldg(wb + kb + 1) : 0.f;
        rb[r].z = (bnv && kb + 2 < K) ? __ldg(wb + kb + 2) : 0.f;
        rb[r].w = (bnv && kb + 3 < K) ? __ldg(wb + kb + 3) : 0.f;
      }
    }
  };
  auto store = [&](int b) {
#pragma unroll
    for (int r = 0; r < NL; r++) {
      const int k = lk + 8 * r;
      As[b][k + 0][lr] = ra[r].x; As[b][k + 1][lr] = ra[r].y;
      As[b][k + 2][lr] = ra[r].z; As[b][k + 3][lr] = ra[r].w;
      Bs[b][k + 0][lr] = rb[r].x; Bs[b][k + 1][lr] = rb[r].y;
      Bs[b][k + 2][lr] = rb[r].z; Bs[b][k + 3][lr] = rb[r].w;
    }
  };
  unsigned long long acc[8][4];  // (acc[i][2p], acc[i][2p+1]) packed for FFMA2
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j] = 0ull;
  // fragments double-buffered in registers: those of k+1 load while k multiplies
  float4 fa[2][2], fb[2][2];
  auto frag = [&](int b, int kk, int f) {
    fa[f][0] = *reinterpret_cast<const float4*>(&As[b][kk][ty * 4]);
    fa[f][1] = *reinterpret_cast<const float4*>(&As[b][kk][64 + ty * 4]);
    fb[f][0] = *reinterpret_cast<const float4*>(&Bs[b][kk][tx * 4]);
    fb[f][1] = *reinterpret_cast<const float4*>(&Bs[b][kk][64 + tx * 4]);
  };
  load(0);
  store(0);
  __syncthreads();
  frag(0, 0, 0);
  const int nk = (K + KB - 1) / KB;
  for (int kt = 0; kt < nk; kt++) {
    const int b = kt & 1;
    if (kt + 1 < nk) load((kt + 1) * KB);
#pragma unroll
    for (int kk = 0; kk < KB; kk++) {
      const int f = kk & 1;
      if (kk + 1 < KB) frag(b, kk + 1, f ^ 1);
      const float av[8] = {fa[f][0].x, fa[f][0].y, fa[f][0].z, fa[f][0].w,
                           fa[f][1].x, fa[f][1].y, fa[f][1].z, fa[f][1].w};
      const unsigned long long bp[4] = {pack2(fb[f][0].x, fb[f][0].y), pack2(fb[f][0].z, fb[f][0].w),
                                        pack2(fb[f][1].x, fb[f][1].y), pack2(fb[f][1].z, fb[f][1].w)};
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const unsigned long long aa = pack2(av[i], av[i]);
#pragma unroll
        for (int j = 0; j < 4; j++) fma2(acc[i][j], aa, bp[j]);
      }
    }
    if (kt + 1 < nk) {
      store(b ^ 1);
      __syncthreads();
      frag(b ^ 1, 0, 0);
    }
  }
  float bias[8];  // the bias column of this thread's 8 output columns, loaded once
#pragma unroll
  for (int j = 0; j < 8; j++) {
    const int n = bn + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
    bias[j] = n < N ? __ldg(W + (long long)n * ldw + K) : 0.0f;
  }
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const int m = bm + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const int n = bn + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (n >= N) continue;
      const float2 pr = unpack2(acc[i][j >> 1]);
      const float a = ((j & 1) ? pr.y : pr.x) + bias[j];
      float t;
      Y[(long long)m * ldy + n] = dev_scaled_tanh(a, &t);
    }
  }
}

constexpr int OT = 256;  // 8 warps, one sample per warp per iteration

// Output layer + ranking + counts.  W: (nout, ldw) rows with bias at column K.
__global__ void __launch_bounds__(OT)
    k_out_rank(const float* __restrict__ X, long long ldx, const float* __restrict__ W, int ldw,
               int M, int K, int nout, float* __restrict__ out, const uint8_t* __restrict__ labels,
               unsigned long long* __restrict__ counts, int* __restrict__ guess) {
  extern __shared__ __align__(16) float osm[];
  float* Ws = osm;  // nout * ldw
  unsigned* cnt = reinterpret_cast<unsigned*>(osm + nout * ldw);  // 102 counters
  for (int i = threadIdx.x; i < nout * ldw; i += OT) Ws[i] = W[i];
  for (int i = threadIdx.x; i < 102; i += OT) cnt[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int m = blockIdx.x * (OT / 32) + warp; m < M; m += gridDim.x * (OT / 32)) {
    float acc[kMaxOut];
#pragma unroll
    for (int j = 0; j < kMaxOut; j++) acc[j] = 0.0f;
    for (int k = lane; k < K; k += 32) {
      const float x = X[(long long)m * ldx + k];
#pragma unroll
      for (int j = 0; j < kMaxOut; j++)
        if (j < nout) acc[j] = fmaf(x, Ws[j * ldw + k], acc[j]);
    }
    float y[kMaxOut];
#pragma unroll
    for (int j = 0; j < kMaxOut; j++) {
      if (j < nout) {
        float s = acc[j];
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        float t;
        y[j] = dev_scaled_tanh(s + Ws[j * ldw + K], &t);
      }
    }
    if (lane == 0) {
      if (out)
        for (int j = 0; j < nout; j++) out[(long long)m * nout + j] = y[j];
      // stable argsort(-y): ties keep the smaller digit; NaN ranks last
      int g1 = -1, g2 = -1;
      for (int j = 0; j < nout; j++) {
        const float v = y[j];
        if (v != v) continue;
        if (g1 < 0 || v > y[g1]) { g2 = g1; g1 = j; }
        else if (g2 < 0 || v > y[g2]) { g2 = j; }
      }
      if (g1 < 0) { g1 = 0; g2 = nout > 1 ? 1 : 0; }
      else if (g2 < 0) { g2 = (g1 == 0 && nout > 1) ? 1 : 0; }
      if (guess) {
        guess[2 * (long long)m] = g1;
        guess[2 * (long long)m + 1] = g2;
      }
      if (labels && counts) {
        const int t = labels[m];
        if (g1 != t) {
          atomicAdd(&cnt[0], 1u);
          if (g2 == t) atomicAdd(&cnt[101], 1u);
        }
        if (t < 10 && g1 < 10) atomicAdd(&cnt[1 + t * 10 + g1], 1u);
      }
    }
  }
  __syncthreads();
  if (labels && counts)
    for (int i = threadIdx.x; i < 102; i += OT)
      if (cnt[i]) atomicAdd(&counts[i], (unsigned long long)cnt[i]);
}

// Rows of n_in floats (any stride) -> rows of `ld` floats, 16-byte aligned,
// so the first layer's GEMM can use float4 loads (padding is never read).
__global__ void k_pad_rows(const float* __restrict__ x, long long ldx, int M, int n_in,
                           float* __restrict__ y, int ld) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)M * n_in;
       t += (long long)gridDim.x * blockDim.x) {
    const long long m = t / n_in;
    const int k = (int)(t - m * n_in);
    y[m * ld + k] = x[m * ldx + k];
  }
}

static int ensure_act(dmlp_net* net, size_t rows, int ld) {
  if (net->act_rows >= rows && net->act_ld >= ld) return DMLP_OK;
  for (int b = 0; b < 3; b++) cudaFree(net->d_act[b]);
  net->d_act[0] = net->d_act[1] = net->d_act[2] = nullptr;
  net->act_rows = 0;
  for (int b = 0; b < 3; b++)
    if (int rc = cuda_check(cudaMalloc(&net->d_act[b], rows * ld * sizeof(float)), "cudaMalloc"))
      return rc;
  net->act_rows = rows;
  net->act_ld = ld;
  return DMLP_OK;
}

static int run_eval(dmlp_net* net, const float* x, long long n, float* out, const uint8_t* labels,
                    long long* counts, int* guess, cudaStream_t st) {
  if (n <= 0) return DMLP_OK;
  DeviceGuard dg(net->device);
  if (int rc = cuda_check(dg.err, "cudaSetDevice")) return rc;
  const int L = net->dev.L;
  int maxld = net->hl[0].pitch;  // activation row stride = input pitch of the consuming layer
  for (int l = 1; l < L; l++) maxld = maxld > net->hl[l].pitch ? maxld : net->hl[l].pitch;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, net->device);
  // a full chunk is one BM-row tile per SM: every layer's grid is then (column
  // tiles) x sms CTAs, whole waves at 2 CTAs per SM for an even number of
  // column tiles (C4: 20/16/12/8/4), where 16384 rows left partial last waves
  const long long cmax = (long long)BM * sms;
  const long long chunk = n < cmax ? n : cmax;
  if (int rc = ensure_act(net, (size_t)chunk, maxld)) return rc;
  const HostLayer& ho = net->hl[L - 1];
  const int osmem = (ho.fo * ho.pitch + 128) * (int)sizeof(float);
  if (int rc = cuda_check(
          cudaFuncSetAttribute(k_out_rank, cudaFuncAttributeMaxDynamicSharedMemorySize, osmem),
          "cudaFuncSetAttribute"))
    return rc;
  if (int rc = net_begin(net, st)) return rc;
  for (long long m0 = 0; m0 < n; m0 += chunk) {
    const int M = (int)((n - m0) < chunk ? (n - m0) : chunk);
    const float* in = x + m0 * net->sizes[0];
    long long ldin = net->sizes[0];
    if (L > 1 && (ldin % 4 != 0 || (reinterpret_cast<uintptr_t>(in) & 15) != 0)) {
      k_pad_rows<<<sms * 4, 256, 0, st>>>(in, ldin, M, net->sizes[0], net->d_act[2],
                                          net->hl[0].pitch);
      in = net->d_act[2];
      ldin = net->hl[0].pitch;
    }
    int b = 0;
    for (int l = 0; l < L - 1; l++) {
      const HostLayer& h = net->hl[l];
      float* y = net->d_act[b];
      const int ldy = net->hl[l + 1].pitch;
      dim3 grid((h.fo + BN - 1) / BN, (M + BM - 1) / BM);
      const bool vec = ldin % 4 == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0;
      (vec ? k_gemm_tanh<true> : k_gemm_tanh<false>)<<<grid, GT, 0, st>>>(
          in, ldin, net->d_w + h.w_off, h.pitch, M, h.fo, h.fi, y, ldy);
      in = y;
      ldin = ldy;
      b ^= 1;
    }
    const int blocks = (int)((M + (OT / 32) - 1) / (OT / 32)) < sms * 4
                           ? (int)((M + (OT / 32) - 1) / (OT / 32))
                           : sms * 4;
    k_out_rank<<<blocks, OT, osmem, st>>>(in, ldin, net->d_w + ho.w_off, ho.pitch, M, ho.fi,
                                          ho.fo, out ? out + m0 * ho.fo : nullptr,
                                          labels ? labels + m0 : nullptr,
                                          reinterpret_cast<unsigned long long*>(counts),
                                          guess ? guess + 2 * m0 : nullptr);
    if (int rc = cuda_check(cudaGetLastError(), "eval kernels")) return rc;
  }
  return net_end(net, st);
}

}  // namespace dmlp

using namespace dmlp;

extern "C" {

int dmlp_forward_batch(dmlp_net* net, const float* x_dev, int64_t n, float* out_dev,
                       void* stream) {
  if (!net) return set_error(DMLP_EINVAL, "null net");
  if (n > 0 && (!x_dev || !out_dev)) return set_error(DMLP_EINVAL, "null argument");
  return run_eval(net, x_dev, n, out_dev, nullptr, nullptr, nullptr, (cudaStream_t)stream);
}

int dmlp_eval_counts(dmlp_net* net, const float* x_dev, const uint8_t* labels_dev, int64_t n,
                     int64_t* counts_dev, int32_t* guess_dev, void* stream) {
  if (!net) return set_error(DMLP_EINVAL, "null net");
  if (n > 0 && (!x_dev || !labels_dev || !counts_dev))
    return set_error(DMLP_EINVAL, "null argument");
  return run_eval(net, x_dev, n, nullptr, labels_dev, (long long*)counts_dev, guess_dev,
                  (cudaStream_t)stream);
}

}  // extern "C"
