// train_kernel.cu -- persistent on-line back-propagation kernel (sm_100a).
//
// Replaces trainer.train_epoch's per-sample Python loop (trainer.py:104-123)
// and kernels.train_step (kernels.py:329-361): ONE launch trains a whole
// sequence of samples.  Design:
//
//  * Row ownership.  CTA c owns the row block [c*R, c*R+R) of every hidden
//    layer.  Forward a_j = W_j . y is CTA-local: one warp per row, fused with
//    the bias and the scaled tanh; its lane 0 publishes y_j.  The <=32-row
//    output layer is replicated: every CTA keeps its own copy and computes
//    the output, the output delta and the delta of the last hidden layer
//    redundantly, so they cost no inter-CTA exchange.
//  * Backward + update in one pass: each owned weight is read once, feeds the
//    column partial P_c[i] = sum_j w_ji*delta_j with its OLD value and is
//    written back as w_ji + (eta*delta_j)*y_i (mul then add, no FMA --
//    kernels.py:174,182).  Owners of layer l-1's rows then sum the partials
//    in fixed CTA order (deterministic, independent of timing).
//  * No grid barrier.  Every cross-CTA value travels as a 64-bit word
//    {float value, u32 sample-sequence flag} written with one st.relaxed.gpu
//    and polled with ld.relaxed.gpu until the flag matches: data and its
//    readiness arrive in one single-copy-atomic access.  Each producer's
//    words start on their own 128-byte line (one writer per polled line --
//    measured 3.8x cheaper than shared lines on B200).  Buffers alternate by
//    sample parity.
//  * Per layer, the owned rows are either kept in shared memory for the whole
//    launch (resident) or streamed from the L2-persisting HBM copy every
//    sample; the host picks the resident set that fits.
#include <cuda_runtime.h>

#include "dmlp_internal.h"
#include "dmlp_math.cuh"

namespace dmlp {

constexpr int kProfSlots = kProfWords;
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
// Four consecutive flag words (16-byte aligned), the first `valid` of them.
__device__ __forceinline__ void st_flag4(unsigned long long* p, float4 x, int valid,
                                         uint32_t seq) {
  const unsigned long long h = (unsigned long long)seq << 32;
  const unsigned long long a = h | __float_as_uint(x.x), b = h | __float_as_uint(x.y);
  const unsigned long long c = h | __float_as_uint(x.z), d = h | __float_as_uint(x.w);
  if (valid >= 4) {
    asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
    asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p + 2), "l"(c), "l"(d)
                 : "memory");
  } else {
    if (valid > 0) st_flag(p, x.x, seq);
    if (valid > 1) st_flag(p + 1, x.y, seq);
    if (valid > 2) st_flag(p + 2, x.z, seq);
  }
}

__device__ __noinline__ void spin_fail(int* err) {
  atomicExch(err, 1);
  __trap();
}
__device__ __noinline__ float tanh_scaled_noinline(float a, float* t) {
  return dev_scaled_tanh(a, t);
}

// Weight access: shared memory (resident) or global through L2 only (.cg).
template <bool RES>
__device__ __forceinline__ float4 ldw(const float4* p) {
  if constexpr (RES) return *p;
  else return __ldcg(p);
}
template <bool RES>
__device__ __forceinline__ void stw(float4* p, float4 v) {
  if constexpr (RES) *p = v;
  else __stcg(p, v);
}

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) x += __shfl_xor_sync(0xffffffffu, x, s);
  return x;
}
__device__ __forceinline__ float dot4(float4 w, float4 x, float a) {
  a = fmaf(w.x, x.x, a);
  a = fmaf(w.y, x.y, a);
  a = fmaf(w.z, x.z, a);
  return fmaf(w.w, x.w, a);
}
__device__ __forceinline__ float4 upd4(float4 w, float d, float4 x) {  // w + d*x, unfused
  w.x = __fadd_rn(w.x, __fmul_rn(d, x.x));
  w.y = __fadd_rn(w.y, __fmul_rn(d, x.y));
  w.z = __fadd_rn(w.z, __fmul_rn(d, x.z));
  w.w = __fadd_rn(w.w, __fmul_rn(d, x.w));
  return w;
}

// Pre-activation of one row by one warp: lanes stride over float4 columns,
// 8 loads in flight per lane, fixed-order shuffle reduction.  All lanes
// return the sum.
template <bool RES>
__device__ __forceinline__ float warp_row_dot(const float4* __restrict__ w4,
                                              const float4* __restrict__ v4, int nq, int lane) {
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  int q = lane;
  for (; q + 7 * 32 < nq; q += 8 * 32) {
    float4 w[8];
#pragma unroll
    for (int u = 0; u < 8; u++) w[u] = ldw<RES>(w4 + q + 32 * u);
#pragma unroll
    for (int u = 0; u < 8; u++) acc[u & 3] = dot4(w[u], v4[q + 32 * u], acc[u & 3]);
  }
  for (; q < nq; q += 32) acc[0] = dot4(ldw<RES>(w4 + q), v4[q], acc[0]);
  return warp_sum((acc[0] + acc[1]) + (acc[2] + acc[3]));
}

// Update-only pass (layer 0 and the replicated output layer): every
// (row, float4) item is independent, spread over all threads.
template <bool RES>
__device__ __forceinline__ void update_rows(float* W, int pitch, int nr,
                                            const float* __restrict__ v,
                                            const float* __restrict__ dsc) {
  const int nq = pitch >> 2;
  const int total = nr * nq;
  float4* W4 = reinterpret_cast<float4*>(W);
  const float4* v4 = reinterpret_cast<const float4*>(v);
  int k = 0, q = threadIdx.x;  // (row, quad) of item `it`, advanced without division
  while (q >= nq) { q -= nq; k++; }
  int it = threadIdx.x;
  for (; it + 3 * kThreads < total; it += 4 * kThreads) {
    float4 w[4], x[4];
    float d[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      w[u] = ldw<RES>(W4 + it + u * kThreads);
      x[u] = v4[q];
      d[u] = dsc[k];
      q += kThreads;
      while (q >= nq) { q -= nq; k++; }
    }
#pragma unroll
    for (int u = 0; u < 4; u++) stw<RES>(W4 + it + u * kThreads, upd4(w[u], d[u], x[u]));
  }
  for (; it < total; it += kThreads) {
    stw<RES>(W4 + it, upd4(ldw<RES>(W4 + it), dsc[k], v4[q]));
    q += kThreads;
    while (q >= nq) { q -= nq; k++; }
  }
}

// Fused backward + update of a hidden layer l >= 1 over its owned rows:
// thread (g, q) walks rows g, g+G, ... of float4 column q; per-group partials
// are combined in fixed group order and published as flag words.
template <bool RES>
__device__ __forceinline__ void bp_update_rows(float* W, int pitch, int fi, int nr,
                                               const float* __restrict__ v,
                                               const float* __restrict__ delta,
                                               const float* __restrict__ dsc, float* pbuf,
                                               unsigned long long* pll, uint32_t seq) {
  const int nq = pitch >> 2;
  float4* W4 = reinterpret_cast<float4*>(W);
  const float4* v4 = reinterpret_cast<const float4*>(v);
  int G = kThreads / nq;  // row groups when all quads fit in one pass
  if (G < 1) G = 1;
  if (G > nr) G = nr;
  if (G <= 1) {
    for (int q = threadIdx.x; q < nq; q += kThreads) {
      const float4 x4 = v4[q];
      float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
      int k = 0;
      for (; k + 3 < nr; k += 4) {
        float4 w[4];
#pragma unroll
        for (int u = 0; u < 4; u++) w[u] = ldw<RES>(W4 + (size_t)(k + u) * nq + q);
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const float dj = delta[k + u];
          p.x = fmaf(w[u].x, dj, p.x);
          p.y = fmaf(w[u].y, dj, p.y);
          p.z = fmaf(w[u].z, dj, p.z);
          p.w = fmaf(w[u].w, dj, p.w);
          stw<RES>(W4 + (size_t)(k + u) * nq + q, upd4(w[u], dsc[k + u], x4));
        }
      }
      for (; k < nr; k++) {
        const float4 w4 = ldw<RES>(W4 + (size_t)k * nq + q);
        const float dj = delta[k];
        p.x = fmaf(w4.x, dj, p.x);
        p.y = fmaf(w4.y, dj, p.y);
        p.z = fmaf(w4.z, dj, p.z);
        p.w = fmaf(w4.w, dj, p.w);
        stw<RES>(W4 + (size_t)k * nq + q, upd4(w4, dsc[k], x4));
      }
      st_flag4(pll + 4 * q, p, fi - 4 * q, seq);
    }
    return;
  }
  const int g = threadIdx.x / nq, q = threadIdx.x - g * nq;
  if (g < G) {
    const float4 x4 = v4[q];
    float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int k = g; k < nr; k += G) {
      const float4 w4 = ldw<RES>(W4 + (size_t)k * nq + q);
      const float dj = delta[k];
      p.x = fmaf(w4.x, dj, p.x);
      p.y = fmaf(w4.y, dj, p.y);
      p.z = fmaf(w4.z, dj, p.z);
      p.w = fmaf(w4.w, dj, p.w);
      stw<RES>(W4 + (size_t)k * nq + q, upd4(w4, dsc[k], x4));
    }
    reinterpret_cast<float4*>(pbuf)[g * nq + q] = p;
  }
  __syncthreads();
  for (int col = threadIdx.x; col < fi; col += kThreads) {
    float s = pbuf[col];
    for (int h = 1; h < G; h++) s += pbuf[h * 4 * nq + col];
    st_flag(pll + col, s, seq);
  }
}

// Poll a batch of U flag words per thread in rounds: every round re-issues
// the loads of all words not ready yet, so a late producer costs one L2
// round trip per round, not one per word.
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

// Gather y of a hidden layer (protocol "E").  Producer p's
// rows sit in its own line-aligned slot; each warp instruction reads one
// producer's slot (lane = row within the block, 32-row segments when R > 32)
// and every thread keeps all of its loads in flight, re-polling only the
// words whose flag is not yet this sample's.  Measured: a 148-producer
// all-to-all exchange in ~2.2K cycles, the single-word ping floor.
constexpr int kGatherU = 10;  // producer lines per warp per batch (16 warps x 10 >= 148)

__device__ __forceinline__ void gather_y(const unsigned long long* src, const LayerDev& ly,
                                         float* dst, uint32_t seq, int* err) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nseg = (ly.R + 31) >> 5, V = ly.P * nseg;
  for (int vb = 0; vb < V; vb += kWarps * kGatherU) {
    const unsigned long long* ptr[kGatherU];
    unsigned long long v[kGatherU];
    int row[kGatherU];
#pragma unroll
    for (int u = 0; u < kGatherU; u++) {
      const int vi = vb + warp + kWarps * u;
      const int p = nseg == 1 ? vi : vi / nseg;
      const int k = (vi - p * nseg) * 32 + lane;
      row[u] = p * ly.R + k;
      const bool ok = vi < V && k < ly.R && row[u] < ly.fo;
      ptr[u] = ok ? src + ((size_t)p << ly.ylog) + k : nullptr;
      v[u] = ok ? ld_flag(ptr[u]) : 0ull;
    }
    poll_batch<kGatherU>(ptr, v, seq, err);
#pragma unroll
    for (int u = 0; u < kGatherU; u++)
      if (ptr[u] != nullptr) dst[row[u]] = __uint_as_float((uint32_t)v[u]);
  }
}

// Owned rows [0, nr) of layer l-1: delta_i = hidden_delta(sum_c P_c[i], t_i)
// with P_c[i] = src[c*pstride + r0 + i] over the P producers of layer l.
// Same protocol: each warp instruction reads one producer's nr contiguous
// words into xbuf[i*P + c]; then one warp per row sums over producers in
// fixed order (lane-strided, then a butterfly) -- deterministic.
__device__ __forceinline__ void gather_partials(const unsigned long long* src, int pstride,
                                                int P, int r0, int nr,
                                                const float* __restrict__ tcache, float* xbuf,
                                                float* delta, float* dsc, float eta,
                                                uint32_t seq, int* err) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nseg = (nr + 31) >> 5, V = P * nseg;
  for (int vb = 0; vb < V; vb += kWarps * kGatherU) {
    const unsigned long long* ptr[kGatherU];
    unsigned long long v[kGatherU];
    int slot[kGatherU];
#pragma unroll
    for (int u = 0; u < kGatherU; u++) {
      const int vi = vb + warp + kWarps * u;
      const int p = nseg == 1 ? vi : vi / nseg;
      const int k = (vi - p * nseg) * 32 + lane;
      slot[u] = k * P + p;
      const bool ok = vi < V && k < nr;
      ptr[u] = ok ? src + (size_t)p * pstride + r0 + k : nullptr;
      v[u] = ok ? ld_flag(ptr[u]) : 0ull;
    }
    poll_batch<kGatherU>(ptr, v, seq, err);
#pragma unroll
    for (int u = 0; u < kGatherU; u++)
      if (ptr[u] != nullptr) xbuf[slot[u]] = __uint_as_float((uint32_t)v[u]);
  }
  __syncthreads();
  for (int k = warp; k < nr; k += kWarps) {
    float acc = 0.0f;
    for (int c = lane; c < P; c += 32) acc += xbuf[k * P + c];
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

// Forward of the owned rows of a hidden layer: one warp per row; lane 0
// applies the scaled tanh to the (bias-included) pre-activation and caches
// t; the CTA's y values are staged in smem and published by ONE coalesced
// warp store of flag words into this CTA's line-aligned slot.
template <bool RES>
__device__ __forceinline__ void fwd_hidden(const float* W, const LayerDev& ly, int nr,
                                           const float* v, float* tc, float* ystage,
                                           unsigned long long* yslot, uint32_t seq) {
  const int nq = ly.pitch >> 2, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = warp; k < nr; k += kWarps) {
    const float a = warp_row_dot<RES>(reinterpret_cast<const float4*>(W + (size_t)k * ly.pitch),
                                      reinterpret_cast<const float4*>(v), nq, lane);
    if (lane == 0) {
      float t;
      ystage[k] = tanh_scaled_noinline(a, &t);
      tc[k] = t;
    }
  }
  __syncthreads();
  if (warp == 0)
    for (int k = lane; k < nr; k += 32) st_flag(yslot + k, ystage[k], seq);
}

// Output layer forward (all rows, one warp per row): a -> outv[0..fo).
template <bool RES>
__device__ __forceinline__ void fwd_out(const float* W, const LayerDev& lo, const float* v,
                                        float* outv) {
  const int nq = lo.pitch >> 2, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = warp; k < lo.fo; k += kWarps) {
    const float a = warp_row_dot<RES>(reinterpret_cast<const float4*>(W + (size_t)k * lo.pitch),
                                      reinterpret_cast<const float4*>(v), nq, lane);
    if (lane == 0) outv[k] = a;
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    k_train(const NetDev net, const float* __restrict__ X, long long ldx,
            const uint8_t* __restrict__ labels, const int32_t* __restrict__ order,
            long long n, float eta, uint32_t seq0, unsigned long long* wrong_out,
            float* y_last) {
  extern __shared__ __align__(16) float sm[];
  __shared__ int g_r0[kMaxLayers], g_nr[kMaxLayers];
  __shared__ float* g_w[kMaxLayers];  // this CTA's rows of each layer (smem or global)
  const int c = blockIdx.x, tid = threadIdx.x;
  const int L = net.L;
  float* pbuf = sm + net.pbuf_off;
  float* outv = sm + net.out_off;  // a | y | delta | eta*delta
  const LayerDev& lo = net.ly[L - 1];

  // Geometry of the rows this CTA works on.
  if (tid < L) {
    const LayerDev& ly = net.ly[tid];
    int r0 = 0, nr = ly.fo;
    float* g = ly.w + (size_t)c * ly.fo * ly.pitch;  // replicated output copy
    if (tid < L - 1) {
      r0 = min(c * ly.R, ly.fo);
      nr = min(ly.R, ly.fo - r0);
      g = ly.w + (size_t)r0 * ly.pitch;
    }
    g_r0[tid] = r0;
    g_nr[tid] = nr;
    g_w[tid] = ly.res ? sm + ly.wsm_off : g;
  }
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
  __syncthreads();
  for (int l = 0; l < L; l++) {  // resident layers: load the rows once
    const LayerDev& ly = net.ly[l];
    if (!ly.res) continue;
    const float4* g = reinterpret_cast<const float4*>(
        l < L - 1 ? ly.w + (size_t)g_r0[l] * ly.pitch : ly.w + (size_t)c * ly.fo * ly.pitch);
    float4* s = reinterpret_cast<float4*>(sm + ly.wsm_off);
    for (int i = tid; i < g_nr[l] * ly.pitch / 4; i += kThreads) s[i] = g[i];
  }

  // Sample indices and labels are loaded ahead so no dependent global load
  // sits at the head of a sample.
  long long img_cur = n > 0 ? (order ? order[0] : 0) : 0;
  long long img_nxt = n > 1 ? (order ? order[1] : 1) : -1;
  int digit_cur = n > 0 ? labels[img_cur] : 0;
  if (n > 0) {
    for (int i = tid; i < net.ly[0].fi; i += kThreads)
      cp_async4(sm + net.in0_off[0] + i, X + img_cur * ldx + i);
    cp_async_commit();
  }
  unsigned long long wrong = 0;  // counted by the last thread of CTA 0
  const bool counter = (c == 0 && tid == kThreads - 1);
  // optional in-kernel profile (thread 0 of every CTA): per-phase cycles.
  // slot 0 loop total, 1 exchange waits; 2.. per phase (device.py names them).
  const bool prof = net.prof != nullptr && tid == 0;
  long long t_loop0 = prof ? clock64() : 0, t_xchg = 0, t_mark = 0;
  long long ph[kProfSlots] = {0};
  long long t_ph = t_loop0;
#define PH(slot)                    \
  if (prof) {                       \
    const long long _t = clock64(); \
    ph[slot] += _t - t_ph;          \
    t_ph = _t;                      \
  }
  // optional one-sample timeline: CTA-synchronised %globaltimer marks.
  // mark 0 sample start; for exchange e: 1+2e producer side done, 2+2e
  // gather done (forward exchanges e = 0..L-2, backward e = L-1..).
#define TRACE(mark)                                                          \
  if (net.trace != nullptr && s == net.trace_sample) {                      \
    __syncthreads();                                                          \
    if (tid == 0) {                                                           \
      unsigned long long _g;                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_g));                \
      net.trace[(size_t)c * 64 + (mark)] = _g;                                \
    }                                                                         \
  }

  for (long long s = 0; s < n; s++) {
    const uint32_t seq = seq0 + (uint32_t)s;
    const int buf = seq & 1;
    const long long img_nn = (s + 2 < n) ? (order ? order[s + 2] : s + 2) : -1;
    const int digit = digit_cur;
    const int digit_nxt = img_nxt >= 0 ? labels[img_nxt] : 0;
    float* in0 = sm + net.in0_off[s & 1];
    cp_async_wait_all();
    __syncthreads();
    PH(2);
    TRACE(0);
    if (img_nxt >= 0) {  // prefetch the next sample's input under this sample
      float* nx = sm + net.in0_off[(s + 1) & 1];
      for (int i = tid; i < net.ly[0].fi; i += kThreads)
        cp_async4(nx + i, X + img_nxt * ldx + i);
      cp_async_commit();
    }

    // ---------------- forward: hidden layers ----------------
    for (int l = 0; l < L - 1; l++) {
      const LayerDev& ly = net.ly[l];
      unsigned long long* yb = ly.yll + ((size_t)buf * ly.P << ly.ylog);
      const float* v = l == 0 ? in0 : sm + ly.in_off;
      if (c < ly.P) {
        unsigned long long* mine = yb + ((size_t)c << ly.ylog);
        if (ly.res) fwd_hidden<true>(g_w[l], ly, g_nr[l], v, sm + ly.t_off, pbuf, mine, seq);
        else fwd_hidden<false>(g_w[l], ly, g_nr[l], v, sm + ly.t_off, pbuf, mine, seq);
      }
      PH(3);
      TRACE(1 + 2 * l);
      if (prof) t_mark = clock64();
      gather_y(yb, ly, sm + net.ly[l + 1].in_off, seq, net.err);
      __syncthreads();
      if (prof) t_xchg += clock64() - t_mark;
      PH(5);
      TRACE(2 + 2 * l);
    }

    // ---------------- output layer (replicated in every CTA) ----------------
    const float* vout = (L == 1) ? in0 : sm + lo.in_off;
    float* Wo = g_w[L - 1];
    if (lo.res) fwd_out<true>(Wo, lo, vout, outv);
    else fwd_out<false>(Wo, lo, vout, outv);
    __syncthreads();
    PH(6);
    if (tid < lo.fo) {
      const float a = outv[tid];
      float t;
      const float y = tanh_scaled_noinline(a, &t);
      const float d = dev_output_delta(y, a, tid == digit ? 1.0f : -1.0f);
      outv[kMaxOut + tid] = y;
      outv[2 * kMaxOut + tid] = d;
      outv[3 * kMaxOut + tid] = __fmul_rn(eta, d);
    }
    __syncthreads();
    if (counter) {  // np.argmax: first maximum (NaN counts as maximum)
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
    PH(7);

    int cur = 0;
    if (L >= 2) {
      // delta of the last hidden layer's owned rows through the OLD output
      // weights, sequential over the <=32 output rows: the reference's
      // single-tile order (kernels.py:149-153) exactly.  All loads first.
      const LayerDev& lh = net.ly[L - 2];
      const int rh0 = g_r0[L - 2], nrh = g_nr[L - 2];
      const float* tc = sm + lh.t_off;
      for (int k = tid; k < nrh; k += kThreads) {
        float w[kMaxOut];
#pragma unroll
        for (int j = 0; j < kMaxOut; j++)
          if (j < lo.fo)
            w[j] = lo.res ? Wo[(size_t)j * lo.pitch + rh0 + k]
                          : __ldcg(Wo + (size_t)j * lo.pitch + rh0 + k);
        float acc = 0.0f;
#pragma unroll
        for (int j = 0; j < kMaxOut; j++)
          if (j < lo.fo) acc = __fadd_rn(acc, __fmul_rn(w[j], outv[2 * kMaxOut + j]));
        const float d = dev_hidden_delta(acc, tc[k]);
        sm[net.delta_off[cur] + k] = d;
        sm[net.dsc_off[cur] + k] = __fmul_rn(eta, d);
      }
      __syncthreads();
    }
    PH(8);
    if (lo.res) update_rows<true>(Wo, lo.pitch, lo.fo, vout, outv + 3 * kMaxOut);
    else update_rows<false>(Wo, lo.pitch, lo.fo, vout, outv + 3 * kMaxOut);
    PH(9);

    // ---------------- backward + update: hidden layers L-2 .. 1 ----------------
    for (int l = L - 2; l >= 1; l--) {
      const LayerDev& ly = net.ly[l];
      unsigned long long* pb = ly.pll + (size_t)buf * ly.P * ly.pstride;
      if (c < ly.P) {
        if (ly.res)
          bp_update_rows<true>(g_w[l], ly.pitch, ly.fi, g_nr[l], sm + ly.in_off,
                               sm + net.delta_off[cur], sm + net.dsc_off[cur], pbuf,
                               pb + (size_t)c * ly.pstride, seq);
        else
          bp_update_rows<false>(g_w[l], ly.pitch, ly.fi, g_nr[l], sm + ly.in_off,
                                sm + net.delta_off[cur], sm + net.dsc_off[cur], pbuf,
                                pb + (size_t)c * ly.pstride, seq);
      }
      PH(10);
      TRACE(1 + 2 * (L - 1 + (L - 2 - l)));
      const int nxt = cur ^ 1;
      if (prof) t_mark = clock64();
      gather_partials(pb, ly.pstride, ly.P, g_r0[l - 1], g_nr[l - 1], sm + net.ly[l - 1].t_off,
                      sm + net.xbuf_off, sm + net.delta_off[nxt], sm + net.dsc_off[nxt], eta,
                      seq, net.err);
      __syncthreads();
      if (prof) t_xchg += clock64() - t_mark;
      PH(11);
      TRACE(2 + 2 * (L - 1 + (L - 2 - l)));
      cur = nxt;
    }
    if (L >= 2) {
      if (net.ly[0].res)
        update_rows<true>(g_w[0], net.ly[0].pitch, g_nr[0], in0, sm + net.dsc_off[cur]);
      else
        update_rows<false>(g_w[0], net.ly[0].pitch, g_nr[0], in0, sm + net.dsc_off[cur]);
    }
    PH(12);
    TRACE(63);
    img_cur = img_nxt;
    img_nxt = img_nn;
    digit_cur = digit_nxt;
  }
  __syncthreads();

  for (int l = 0; l < L; l++) {  // write the resident rows back
    const LayerDev& ly = net.ly[l];
    if (!ly.res) continue;
    float4* g = reinterpret_cast<float4*>(
        l < L - 1 ? ly.w + (size_t)g_r0[l] * ly.pitch : ly.w + (size_t)c * ly.fo * ly.pitch);
    const float4* s = reinterpret_cast<const float4*>(sm + ly.wsm_off);
    for (int i = tid; i < g_nr[l] * ly.pitch / 4; i += kThreads) g[i] = s[i];
  }
  if (prof) {
    ph[0] = clock64() - t_loop0;
    ph[1] = t_xchg;
    for (int k = 0; k < kProfSlots; k++)
      atomicAdd(net.prof + kProfSlots * c + k, (unsigned long long)ph[k]);
  }
#undef PH
#undef TRACE
  if (counter && wrong_out != nullptr) atomicAdd(wrong_out, wrong);
}

cudaError_t set_train_attributes(int smem_bytes) {
  return cudaFuncSetAttribute(k_train, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
}

cudaError_t train_occupancy(int smem_bytes, int* blocks_per_sm) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_train, kThreads,
                                                       smem_bytes);
}

cudaError_t launch_train(const dmlp_net* net, const float* x, long long ldx,
                         const uint8_t* labels, const int32_t* order, long long n, float eta,
                         uint32_t seq0, long long* wrong, float* y_last, cudaStream_t st) {
  NetDev nd = net->dev;
  unsigned long long* w = reinterpret_cast<unsigned long long*>(wrong);
  void* args[] = {&nd, &x, &ldx, &labels, &order, &n, &eta, &seq0, &w, &y_last};
  return cudaLaunchCooperativeKernel((const void*)k_train, dim3(nd.nct), dim3(kThreads), args,
                                     (size_t)net->smem_bytes, st);
}

}  // namespace dmlp
