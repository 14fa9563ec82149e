// train_kernel.cu -- persistent on-line back-propagation kernel (sm_100a).
//
// Replaces trainer.train_epoch's per-sample Python loop (trainer.py:104-123)
// and kernels.train_step (kernels.py:329-361): ONE launch trains a whole
// sequence of samples.  Design:
//
//  * Row ownership.  CTA c owns rows [fo*c/nct, fo*(c+1)/nct) of every hidden
//    layer.  Forward a_j = W_j . y is CTA-local (fused with bias and the
//    scaled tanh).  The 10-row output layer is replicated: every CTA keeps its
//    own copy and computes the output, the output delta and the delta of the
//    last hidden layer redundantly, so they cost no inter-CTA exchange.
//  * Backward + update in one pass: for each owned row j the CTA reads W_j
//    once, accumulates the column partials P_c[i] = sum_j w_ji*delta_j with
//    the OLD weight and writes w_ji + (eta*delta_j)*y_i back (mul then add,
//    no FMA -- kernels.py:174,182).  Owners of layer l-1's rows then sum the
//    nct partials in fixed CTA order (deterministic).
//  * No grid barrier.  Every cross-CTA value travels as a 64-bit word
//    {float value, u32 sample-sequence flag} written with one st.relaxed.gpu
//    and polled with ld.relaxed.gpu until the flag matches: data and its
//    readiness arrive in the same single-copy-atomic access, so an exchange
//    costs one L2 round trip.  Buffers alternate by sample parity.
//  * Weights are either streamed from the L2-persisting HBM copy every
//    sample (RES=false) or kept in shared memory for the whole launch
//    (RES=true) and written back at the end.
#include <cuda_runtime.h>

#include "dmlp_internal.h"
#include "dmlp_math.cuh"

namespace dmlp {

constexpr long long kSpinTimeoutCycles = 40000000000LL;  // ~20 s: fail loudly, never hang

__device__ __forceinline__ unsigned long long ld_flag(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_flag(unsigned long long* p, float x, uint32_t seq) {
  const unsigned long long v = ((unsigned long long)seq << 32) | __float_as_uint(x);
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __noinline__ void spin_fail(int* err) {
  atomicExch(err, 1);
  __trap();
}
// After the call, lane k holds sum over the warp's lanes of v[k] (k < 32).
__device__ __forceinline__ float warp_transpose_reduce32(float (&v)[32], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int k = 0; k < s; k++) {
      const float send = upper ? v[k] : v[k + s];
      const float keep = upper ? v[k + s] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) x += __shfl_xor_sync(0xffffffffu, x, s);
  return x;
}

__device__ __forceinline__ void own_rows(int fo, int c, int nct, int& r0, int& r1) {
  r0 = (int)(((long long)fo * c) / nct);
  r1 = (int)(((long long)fo * (c + 1)) / nct);
}

// Pre-activations of rows [0, nr) of W (row stride pitch floats) against the
// smem vector v (pitch floats: inputs, then 1.0 for the bias column, then 0).
// Thread t owns column quads t, t+kThreads, ...; per-row sums are reduced
// across the CTA in a fixed order.  dst[k] = a_k.
__device__ __forceinline__ void fwd_rows(const float* __restrict__ W, int pitch, int nr,
                                         const float* __restrict__ v, float* red,
                                         float* dst) {
  const int nq = pitch >> 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float4* v4 = reinterpret_cast<const float4*>(v);
  for (int rb = 0; rb < nr; rb += 32) {
    const int n = min(32, nr - rb);
    float acc[32];
#pragma unroll
    for (int k = 0; k < 32; k++) acc[k] = 0.0f;
    const float4* wrow = reinterpret_cast<const float4*>(W + (size_t)rb * pitch);
    for (int q = tid; q < nq; q += kThreads) {
      const float4 x4 = v4[q];
#pragma unroll
      for (int k = 0; k < 32; k++) {
        if (k < n) {
          const float4 w4 = wrow[(size_t)k * nq + q];
          float a = acc[k];
          a = fmaf(w4.x, x4.x, a);
          a = fmaf(w4.y, x4.y, a);
          a = fmaf(w4.z, x4.z, a);
          a = fmaf(w4.w, x4.w, a);
          acc[k] = a;
        }
      }
    }
    const float s = warp_transpose_reduce32(acc, lane);
    red[warp * 32 + lane] = s;
    __syncthreads();
    if (tid < n) {
      float t = 0.0f;
#pragma unroll
      for (int w = 0; w < kWarps; w++) t += red[w * 32 + tid];
      dst[rb + tid] = t;
    }
    __syncthreads();
  }
}

// Fused backward + update over rows [0, nr) of W with owned deltas delta[k]
// and dsc[k] = f32(eta)*delta[k] (kernels.py:174).  Column partials of the
// OLD weights go to pll (flag words, may be null); input vector v as above.
__device__ __forceinline__ void bp_update_rows(float* __restrict__ W, int pitch, int fi, int nr,
                                               const float* __restrict__ v,
                                               const float* __restrict__ delta,
                                               const float* __restrict__ dsc,
                                               unsigned long long* pll, uint32_t seq) {
  const int nq = pitch >> 2;
  const float4* v4 = reinterpret_cast<const float4*>(v);
  float4* W4 = reinterpret_cast<float4*>(W);
  for (int q = threadIdx.x; q < nq; q += kThreads) {
    const float4 x4 = v4[q];
    float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
    float4* wp = W4 + q;
#pragma unroll 4
    for (int k = 0; k < nr; k++) {
      float4 w4 = wp[(size_t)k * nq];
      const float dj = delta[k], dd = dsc[k];
      p.x = fmaf(w4.x, dj, p.x);
      p.y = fmaf(w4.y, dj, p.y);
      p.z = fmaf(w4.z, dj, p.z);
      p.w = fmaf(w4.w, dj, p.w);
      w4.x = __fadd_rn(w4.x, __fmul_rn(dd, x4.x));
      w4.y = __fadd_rn(w4.y, __fmul_rn(dd, x4.y));
      w4.z = __fadd_rn(w4.z, __fmul_rn(dd, x4.z));
      w4.w = __fadd_rn(w4.w, __fmul_rn(dd, x4.w));
      wp[(size_t)k * nq] = w4;
    }
    if (pll != nullptr) {
      const int c0 = q * 4;
      if (c0 + 0 < fi) st_flag(pll + c0 + 0, p.x, seq);
      if (c0 + 1 < fi) st_flag(pll + c0 + 1, p.y, seq);
      if (c0 + 2 < fi) st_flag(pll + c0 + 2, p.z, seq);
      if (c0 + 3 < fi) st_flag(pll + c0 + 3, p.w, seq);
    }
  }
}

// Poll a batch of U flag words per thread in rounds: every round re-issues
// the loads of all words that are not ready yet, so a late producer costs
// one L2 round trip per round, not one per word.
template <int U>
__device__ __forceinline__ void poll_batch(const unsigned long long* const (&ptr)[U],
                                           unsigned long long (&v)[U], uint32_t seq,
                                           int* err) {
  long long t0 = 0;
  for (int round = 0;; round++) {
    bool done = true;
#pragma unroll
    for (int u = 0; u < U; u++)
      if (ptr[u] != nullptr && (uint32_t)(v[u] >> 32) != seq) done = false;
    if (done) return;
    if (round == 0) t0 = clock64();
    else if (clock64() - t0 > kSpinTimeoutCycles) spin_fail(err);
#pragma unroll
    for (int u = 0; u < U; u++)
      if (ptr[u] != nullptr && (uint32_t)(v[u] >> 32) != seq) v[u] = ld_flag(ptr[u]);
  }
}

// dst[i] = value of flag words src[i], i < n, once their flag equals seq.
__device__ __forceinline__ void gather_vec(const unsigned long long* src, int n, float* dst,
                                           uint32_t seq, int* err) {
  constexpr int U = 4;
  for (int ib = 0; ib < n; ib += kThreads * U) {
    const unsigned long long* ptr[U];
    unsigned long long v[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int i = ib + u * kThreads + threadIdx.x;
      ptr[u] = i < n ? src + i : nullptr;
      v[u] = i < n ? ld_flag(src + i) : 0ull;
    }
    poll_batch<U>(ptr, v, seq, err);
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int i = ib + u * kThreads + threadIdx.x;
      if (i < n) dst[i] = __uint_as_float((uint32_t)v[u]);
    }
  }
}

// Owned rows [0, nr) of layer l-1: delta_i = hidden_delta(sum_c P_c[i], t_i),
// P_c[i] = src[c*pitch + r0 + i].  Summation order is fixed.
__device__ __forceinline__ void gather_partials(const unsigned long long* src, int pitch,
                                                int nct, int r0, int nr,
                                                const float* __restrict__ tcache,
                                                float* delta, float* dsc, float eta,
                                                uint32_t seq, int* err) {
  constexpr int U = 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = warp; k < nr; k += kWarps) {
    const unsigned long long* col = src + r0 + k;
    float acc = 0.0f;
    for (int cb = 0; cb < nct; cb += 32 * U) {
      const unsigned long long* ptr[U];
      unsigned long long v[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int c = cb + u * 32 + lane;
        ptr[u] = c < nct ? col + (size_t)c * pitch : nullptr;
        v[u] = c < nct ? ld_flag(col + (size_t)c * pitch) : 0ull;
      }
      poll_batch<U>(ptr, v, seq, err);
#pragma unroll
      for (int u = 0; u < U; u++)
        if (cb + u * 32 + lane < nct) acc += __uint_as_float((uint32_t)v[u]);
    }
    acc = warp_sum(acc);
    if (lane == 0) {
      const float d = dev_hidden_delta(acc, tcache[k]);
      delta[k] = d;
      dsc[k] = __fmul_rn(eta, d);
    }
  }
}

__device__ __forceinline__ void cp_async4(float* smem_dst, const float* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

template <bool RES>
__global__ void __launch_bounds__(kThreads, 1)
    k_train(const NetDev net, const float* __restrict__ X, long long ldx,
            const uint8_t* __restrict__ labels, const int32_t* __restrict__ order,
            long long n, float eta, uint32_t seq0, unsigned long long* wrong_out,
            float* y_last) {
  extern __shared__ __align__(16) float sm[];
  const int c = blockIdx.x, tid = threadIdx.x;
  const int L = net.L, nct = net.nct;
  float* red = sm + net.red_off;
  float* outv = sm + net.out_off;  // a[32] | y[32] | delta[32] | dsc[32]
  const LayerDev& lo = net.ly[L - 1];

  // Constant tails of every input vector: 1.0 in the bias column, zeros after.
  for (int b = 0; b < 2; b++) {
    float* v = sm + net.in0_off[b];
    for (int i = net.ly[0].fi + tid; i < net.ly[0].pitch; i += kThreads)
      v[i] = (i == net.ly[0].fi) ? 1.0f : 0.0f;
  }
  for (int l = 1; l < L; l++) {
    float* v = sm + net.ly[l].in_off;
    for (int i = net.ly[l].fi + tid; i < net.ly[l].pitch; i += kThreads)
      v[i] = (i == net.ly[l].fi) ? 1.0f : 0.0f;
  }

  // Per-layer weight views (rows relative to the CTA's first owned row).
  float* Wv[kMaxLayers];
  int R0[kMaxLayers], NR[kMaxLayers];
  {
    int woff = net.wsm_off;
    for (int l = 0; l < L; l++) {
      const LayerDev& ly = net.ly[l];
      int r0 = 0, r1 = ly.fo;
      float* g = ly.w + (size_t)c * ly.fo * ly.pitch;  // replicated output copy
      if (l < L - 1) {
        own_rows(ly.fo, c, nct, r0, r1);
        g = ly.w + (size_t)r0 * ly.pitch;
      }
      R0[l] = r0;
      NR[l] = r1 - r0;
      if (RES) {
        float* s = sm + woff;
        const int cnt4 = NR[l] * ly.pitch / 4;
        for (int i = tid; i < cnt4; i += kThreads)
          reinterpret_cast<float4*>(s)[i] = reinterpret_cast<const float4*>(g)[i];
        Wv[l] = s;
        woff += NR[l] * ly.pitch;
      } else {
        Wv[l] = g;
      }
    }
  }

  // Stage sample 0's input; image indices are loaded two samples ahead so
  // no dependent global load sits at the head of a sample.
  long long img_cur = n > 0 ? (order ? order[0] : 0) : 0;
  long long img_nxt = n > 1 ? (order ? order[1] : 1) : -1;
  if (n > 0) {
    for (int i = tid; i < net.ly[0].fi; i += kThreads)
      cp_async4(sm + net.in0_off[0] + i, X + img_cur * ldx + i);
    cp_async_commit();
  }
  unsigned long long wrong = 0;
  // optional in-kernel profile: cycles inside the exchange waits vs the whole loop
  const bool prof = net.prof != nullptr && tid == 0;
  long long t_loop0 = prof ? clock64() : 0, t_xchg = 0, t_mark = 0;
#define DMLP_XCHG_BEGIN() \
  if (prof) t_mark = clock64();
#define DMLP_XCHG_END() \
  if (prof) t_xchg += clock64() - t_mark;

  for (long long s = 0; s < n; s++) {
    const uint32_t seq = seq0 + (uint32_t)s;
    const int buf = seq & 1;
    const long long img_nn = (s + 2 < n) ? (order ? order[s + 2] : s + 2) : -1;
    const int digit = labels[img_cur];
    float* in0 = sm + net.in0_off[s & 1];
    cp_async_wait_all();
    __syncthreads();
    if (img_nxt >= 0) {  // prefetch the next sample's input under this sample
      float* nx = sm + net.in0_off[(s + 1) & 1];
      for (int i = tid; i < net.ly[0].fi; i += kThreads)
        cp_async4(nx + i, X + img_nxt * ldx + i);
      cp_async_commit();
    }
    img_cur = img_nxt;
    img_nxt = img_nn;

    // ---------------- forward: hidden layers ----------------
    for (int l = 0; l < L - 1; l++) {
      const LayerDev& ly = net.ly[l];
      const float* v = (l == 0) ? in0 : sm + ly.in_off;
      float* tc = sm + ly.t_off;
      fwd_rows(Wv[l], ly.pitch, NR[l], v, red, tc);  // tc temporarily holds a_j
      unsigned long long* yb = ly.yll + (size_t)buf * ly.fo;
      for (int k = tid; k < NR[l]; k += kThreads) {
        float t;
        const float y = dev_scaled_tanh(tc[k], &t);
        tc[k] = t;
        st_flag(yb + R0[l] + k, y, seq);
      }
      DMLP_XCHG_BEGIN();
      gather_vec(yb, ly.fo, sm + net.ly[l + 1].in_off, seq, net.err);
      __syncthreads();
      DMLP_XCHG_END();
    }

    // ---------------- output layer (replicated in every CTA) ----------------
    {
      const float* v = (L == 1) ? in0 : sm + lo.in_off;
      fwd_rows(Wv[L - 1], lo.pitch, lo.fo, v, red, outv);
      if (tid < lo.fo) {
        const float a = outv[tid];
        float t;
        const float y = dev_scaled_tanh(a, &t);
        const float d = dev_output_delta(y, a, tid == digit ? 1.0f : -1.0f);
        outv[kMaxOut + tid] = y;
        outv[2 * kMaxOut + tid] = d;
        outv[3 * kMaxOut + tid] = __fmul_rn(eta, d);
      }
      __syncthreads();
      if (c == 0 && tid == 0) {  // np.argmax: first maximum (NaN counts as maximum)
        int best = 0;
        float bv = outv[kMaxOut];
        for (int k = 1; k < lo.fo && !(bv != bv); k++) {
          const float yk = outv[kMaxOut + k];
          if (yk > bv || yk != yk) { bv = yk; best = k; }
        }
        wrong += (best != digit);
      }
      if (c == 0 && s == n - 1 && y_last != nullptr && tid < lo.fo)
        y_last[tid] = outv[kMaxOut + tid];
    }

    int cur = 0;
    if (L >= 2) {
      // delta of the last hidden layer's owned rows from the (old) output weights,
      // sequential over the <=32 output rows == the reference's single-tile order.
      const LayerDev& lh = net.ly[L - 2];
      float* delta = sm + net.delta_off[cur];
      float* dsc = sm + net.dsc_off[cur];
      const float* tc = sm + lh.t_off;
      const float* Wo = Wv[L - 1];
      for (int k = tid; k < NR[L - 2]; k += kThreads) {
        const int i = R0[L - 2] + k;
        float acc = 0.0f;
        for (int j = 0; j < lo.fo; j++)
          acc = __fadd_rn(acc, __fmul_rn(Wo[(size_t)j * lo.pitch + i], outv[2 * kMaxOut + j]));
        const float d = dev_hidden_delta(acc, tc[k]);
        delta[k] = d;
        dsc[k] = __fmul_rn(eta, d);
      }
      __syncthreads();
    }
    // update the replicated output layer
    bp_update_rows(Wv[L - 1], lo.pitch, lo.fi, lo.fo, (L == 1) ? in0 : sm + lo.in_off,
                   outv + 2 * kMaxOut, outv + 3 * kMaxOut, nullptr, seq);

    // ---------------- backward + update: hidden layers L-2 .. 1 ----------------
    for (int l = L - 2; l >= 1; l--) {
      const LayerDev& ly = net.ly[l];
      unsigned long long* pb = ly.pll + (size_t)buf * nct * ly.pitch;
      bp_update_rows(Wv[l], ly.pitch, ly.fi, NR[l], sm + ly.in_off, sm + net.delta_off[cur],
                     sm + net.dsc_off[cur], pb + (size_t)c * ly.pitch, seq);
      const int nxt = cur ^ 1;
      DMLP_XCHG_BEGIN();
      gather_partials(pb, ly.pitch, nct, R0[l - 1], NR[l - 1], sm + net.ly[l - 1].t_off,
                      sm + net.delta_off[nxt], sm + net.dsc_off[nxt], eta, seq, net.err);
      __syncthreads();
      DMLP_XCHG_END();
      cur = nxt;
    }
    if (L >= 2) {
      const LayerDev& l0 = net.ly[0];
      bp_update_rows(Wv[0], l0.pitch, l0.fi, NR[0], in0, sm + net.delta_off[cur],
                     sm + net.dsc_off[cur], nullptr, seq);
    }
    __syncthreads();
  }

  if (RES) {  // write the resident rows back
    for (int l = 0; l < L; l++) {
      const LayerDev& ly = net.ly[l];
      float* g = (l < L - 1) ? ly.w + (size_t)R0[l] * ly.pitch
                             : ly.w + (size_t)c * ly.fo * ly.pitch;
      const int cnt4 = NR[l] * ly.pitch / 4;
      for (int i = tid; i < cnt4; i += kThreads)
        reinterpret_cast<float4*>(g)[i] = reinterpret_cast<const float4*>(Wv[l])[i];
    }
  }
  if (prof) {
    atomicAdd(net.prof + 2 * c, (unsigned long long)(clock64() - t_loop0));
    atomicAdd(net.prof + 2 * c + 1, (unsigned long long)t_xchg);
  }
#undef DMLP_XCHG_BEGIN
#undef DMLP_XCHG_END
  if (c == 0 && tid == 0 && wrong_out != nullptr) atomicAdd(wrong_out, wrong);
}

cudaError_t set_train_attributes(int smem_bytes) {
  cudaError_t e = cudaFuncSetAttribute(k_train<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_train<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              smem_bytes);
}

cudaError_t train_occupancy(int smem_bytes, int* blocks_per_sm) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_train<false>, kThreads,
                                                       smem_bytes);
}

cudaError_t launch_train(const dmlp_net* net, const float* x, long long ldx,
                         const uint8_t* labels, const int32_t* order, long long n, float eta,
                         uint32_t seq0, long long* wrong, float* y_last, cudaStream_t st) {
  NetDev nd = net->dev;
  unsigned long long* w = reinterpret_cast<unsigned long long*>(wrong);
  void* args[] = {&nd, &x, &ldx, &labels, &order, &n, &eta, &seq0, &w, &y_last};
  const void* fn = nd.resident ? (const void*)k_train<true> : (const void*)k_train<false>;
  return cudaLaunchCooperativeKernel(fn, dim3(nd.nct), dim3(kThreads), args,
                                     (size_t)net->smem_bytes, st);
}

}  // namespace dmlp
