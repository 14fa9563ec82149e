// train_phases.cuh -- the per-phase device routines of the persistent
// on-line BP kernel (train_kernel.cu): forward of an owned row block, column
// partials / update, and the flag-word exchanges.  Kept in a header so the
// phase microbenchmarks (scripts/mb/phase_mb.cu) time exactly this code.
#pragma once
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

// CTA barrier after per-thread spin loops.  bar.sync is the .aligned form:
// every lane of a warp must arrive at it together, and the lanes leave a
// poll loop in different rounds; ptxas does not always reconverge them
// before the barrier (seen as wrong results in the register-only instance,
// flagged by compute-sanitizer --tool synccheck), so reconverge explicitly.
__device__ __forceinline__ void cta_sync() {
  asm volatile("barrier.sync 0;" ::: "memory");
}

static __device__ __noinline__ void spin_fail(int* err) {
  atomicExch(err, 1);
  __trap();
}
// The activation on the training kernel's critical path: the faithfully
// rounded dev_tanhf_fast (C4 +4%, C1 +10%: the glibc restatement is a
// 367-cycle dependent chain, this 122).  Build with
// -DDMLP_K1_TANH_EXACT=1 for the bit-exact glibc form (A/B and drift runs).
#ifndef DMLP_K1_TANH_EXACT
#define DMLP_K1_TANH_EXACT 0
#endif
__device__ __forceinline__ float tanh_scaled_noinline(float a, float* t) {
  if (DMLP_K1_TANH_EXACT) return dev_scaled_tanh(a, t);
  return dev_scaled_tanh_fast(a, t);
}

// Four consecutive flag words (32-byte aligned), the first `valid` of them.
// A full quad is ONE 256-bit store (STG.E.ENL2.256): the 32-byte sector is
// written whole instead of as two 16-byte halves from two instructions -- a
// 2500-word backward exchange drops from 5.4K to 3.5K cycles
// (scripts/mb/xchg11_mb.cu).  Each 8-byte element is still a single-copy-
// atomic word carrying its own flag (vector accesses are per-element).
__device__ __forceinline__ void st_flag4(unsigned long long* p, float4 x, int valid,
                                         uint32_t seq) {
  const unsigned long long h = (unsigned long long)seq << 32;
  const unsigned long long a = h | __float_as_uint(x.x), b = h | __float_as_uint(x.y);
  const unsigned long long c = h | __float_as_uint(x.z), d = h | __float_as_uint(x.w);
  if (valid >= 4) {
    asm volatile("st.relaxed.gpu.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a),
                 "l"(b), "l"(c), "l"(d)
                 : "memory");
  } else {
    if (valid > 0) st_flag(p, x.x, seq);
    if (valid > 1) st_flag(p + 1, x.y, seq);
    if (valid > 2) st_flag(p + 2, x.z, seq);
  }
}

// Weight access: shared memory (resident) or global through L2 only (.cg).
// Callers pass smem pointers derived from the kernel's extern __shared__
// array, so RES accesses compile to LDS/STS.128.
// Streamed weights (RES = false) bypass L1 (.cg), except the first L1R rows of
// a thread's block in kernel instances with kFeatL1: those go through L1 (.ca
// loads, write-back stores), which the kernel otherwise leaves unused (the
// 28 KB next to the 228 KB shared-memory carve-out; C4's streamed layer 3:
// +2.5%).  Only this SM reads and writes its rows, and L1 does not survive a
// launch, so the cached copies stay coherent.
template <bool RES, int L1R = 0>
__device__ __forceinline__ float4 ldw4(const float4* p, int row = 0) {
  if constexpr (RES) return *p;
  else return row < L1R ? __ldca(p) : __ldcg(p);
}
template <bool RES, int L1R = 0>
__device__ __forceinline__ void stw4(float4* p, float4 v, int row = 0) {
  if constexpr (RES) *p = v;
  else if (row < L1R) __stwb(p, v);
  else __stcg(p, v);
}
__device__ __forceinline__ float upd(float w, float d, float x) {  // w + d*x, unfused
  return __fadd_rn(w, __fmul_rn(d, x));
}
__device__ __forceinline__ float4 upd4(float4 w, float d, float4 x) {
  return make_float4(upd(w.x, d, x.x), upd(w.y, d, x.y), upd(w.z, d, x.z), upd(w.w, d, x.w));
}
__device__ __forceinline__ float dot4(float4 w, float4 x, float a) {
  return fmaf(w.w, x.w, fmaf(w.z, x.z, fmaf(w.y, x.y, fmaf(w.x, x.x, a))));
}

// Transposing warp reduction of CH row partials per lane: CH halving
// exchange steps (each lane keeps one half, ships the other) and a plain
// butterfly for the rest.  Returns, on every lane, the warp-wide sum of row
// lane / (32/CH); fixed pairing, so deterministic.  CH-1 + log2(32/CH)
// shuffles instead of 5*CH.
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

// Thread mapping of a row block (LayerDev): G = 1 << gs row groups of
// TG = 512 >> gs threads; thread (g, u) owns rows g, g+G, ... (nj of them)
// and the float4 column quads u, u+TG, ... of each.
struct RowMap {
  int gs, TG, g, u, nj;
  __device__ __forceinline__ RowMap(int gs_, int nr) : gs(gs_) {
    TG = kThreads >> gs;
    g = threadIdx.x >> (9 - gs);
    u = threadIdx.x & (TG - 1);
    nj = nr > g ? ((nr - g - 1) >> gs) + 1 : 0;
  }
};
static_assert(kThreads == 512, "RowMap assumes 512 threads");

// Sum of n (a power of two <= 16) values r[0], r[S], r[2S], ...: every load
// issued at once, then a fixed pairwise tree -- deterministic, and no serial
// load-add chain on the critical path.
template <int S>
__device__ __forceinline__ float tree_sum(const float* r, int n) {
  float v[16];
#pragma unroll
  for (int i = 0; i < 16; i++) v[i] = i < n ? r[i * S] : 0.0f;
#pragma unroll
  for (int h = 8; h >= 1; h >>= 1)
#pragma unroll
    for (int i = 0; i < h; i++) v[i] += v[i + h];
  return v[0];
}

// Forward of the owned rows [0, nr) of a hidden layer.  Per-thread partial
// rows over its quads, a transposing warp reduction, a fixed-order sum over
// the group's warps; one thread per row then applies the scaled tanh, caches
// t_j and publishes y_j (yslot) and/or keeps it (yown).
template <bool RES, int CH, int L1R = 0>
__device__ __forceinline__ void fwd_rows(const float4* __restrict__ W4, int nq, int gs, int nr,
                                         const float4* __restrict__ v4, float* red, float* tc,
                                         float* yown, unsigned long long* yslot, uint32_t seq,
                                         long long* sub = nullptr) {
  long long t0 = sub ? clock64() : 0;
#define SUBP(i)                     \
  if (sub) {                        \
    const long long _t = clock64(); \
    sub[i] += _t - t0;              \
    t0 = _t;                        \
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const RowMap mp(gs, nr);
  const int G = 1 << gs, WG = kWarps >> gs;
  const int njmax = ((nr - 1) >> gs) + 1;
  const int rstep = nq << gs;
  for (int j0 = 0; j0 < njmax; j0 += CH) {
    float acc[CH];
#pragma unroll
    for (int jj = 0; jj < CH; jj++) acc[jj] = 0.0f;
    const int jn = mp.nj - j0;
    const float4* Wg = W4 + (mp.g + (j0 << gs)) * nq;
    for (int q = mp.u; q < nq; q += mp.TG) {
      const float4 x = v4[q];
      // rows in groups of FB loads: the empty asm keeps the compiler from
      // hoisting every load of the chunk (register budget)
      constexpr int FB = RES ? 4 : 8;
#pragma unroll
      for (int j4 = 0; j4 < CH; j4 += FB) {
        if (j4 >= jn) break;  // no rows of this group left (warp-uniform: a warp is in one group)
        float4 w[FB];
#pragma unroll
        for (int i = 0; i < FB; i++)
          w[i] = (j4 + i < CH && j4 + i < jn) ? ldw4<RES, L1R>(Wg + (j4 + i) * rstep + q, j0 + j4 + i)
                                              : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int i = 0; i < FB; i++)
          if (j4 + i < CH) acc[j4 + i < CH ? j4 + i : 0] = dot4(w[i], x, acc[j4 + i < CH ? j4 + i : 0]);
        asm volatile("" ::: "memory");
      }
    }
    const float s = xpose_reduce<CH>(acc, lane);
    if ((lane & (32 / CH - 1)) == 0) red[warp * CH + lane / (32 / CH)] = s;
    cta_sync();
    SUBP(0);
    if (tid < G * CH) {
      const int gg = tid / CH, jj = tid - gg * CH;
      const int k = gg + G * (j0 + jj);
      if (k < nr) {
        const float a = tree_sum<CH>(red + gg * WG * CH + jj, WG);
        float t;
        const float y = tanh_scaled_noinline(a, &t);
        tc[k] = t;
        if (yown) yown[k] = y;
        if (yslot) st_flag(yslot + k, y, seq);
      }
    }
    SUBP(1);
    if (j0 + CH < njmax) __syncthreads();  // red is reused by the next chunk
  }
#undef SUBP
}

template <bool RES, int L1R = 0>
__device__ __forceinline__ void fwd_dispatch(const float4* W4, const LayerDev& ly, int nr,
                                             const float4* v4, float* red, float* tc,
                                             float* yown, unsigned long long* yslot,
                                             uint32_t seq, long long* sub = nullptr) {
  const int nq = ly.pitch >> 2, gs = ly.gs;
  switch (ly.CH) {
    case 4: fwd_rows<RES, 4, L1R>(W4, nq, gs, nr, v4, red, tc, yown, yslot, seq, sub); break;
    case 8: fwd_rows<RES, 8, L1R>(W4, nq, gs, nr, v4, red, tc, yown, yslot, seq, sub); break;
    default: fwd_rows<RES, 16, L1R>(W4, nq, gs, nr, v4, red, tc, yown, yslot, seq, sub); break;
  }
}

// Column partials of the owned rows of hidden layer l >= 1 with the OLD
// weights, published as flag words (bias column excluded, kernels.py:
// 129-153).  FUSE (streamed layers): the same pass writes the updated weight
// w + (eta*delta_j)*y_i, so each weight is read once and written once.
template <bool RES, bool FUSE, int L1R = 0>
__device__ __forceinline__ void bwd_partials(float4* W4, int nq, int fi, int gs, int nr,
                                             const float* __restrict__ delta,
                                             const float* __restrict__ dsc,
                                             const float4* __restrict__ v4, float* pbuf,
                                             unsigned long long* pslot, uint32_t seq) {
  const RowMap mp(gs, nr);
  const int rstep = nq << gs;
  const int qlim = FUSE ? nq : (fi + 3) >> 2;
  for (int q = mp.u; q < qlim; q += mp.TG) {
    const float4 x = FUSE ? v4[q] : make_float4(0.f, 0.f, 0.f, 0.f);
    float4* Wq = W4 + mp.g * nq + q;
    float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
    if (FUSE && mp.nj <= 8) {
      // streamed layer: every owned row's weights in flight at once (one L2
      // round trip), the partials published before the update's stores
      float4 w[8];
#pragma unroll
      for (int i = 0; i < 8; i++)
        w[i] = i < mp.nj ? ldw4<RES, L1R>(Wq + i * rstep, i) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int i = 0; i < 8; i++) {
        if (i < mp.nj) {
          const float d = delta[mp.g + (i << gs)];
          p.x = fmaf(w[i].x, d, p.x);
          p.y = fmaf(w[i].y, d, p.y);
          p.z = fmaf(w[i].z, d, p.z);
          p.w = fmaf(w[i].w, d, p.w);
        }
      }
      if (4 * q < fi) {
        if (gs == 0) st_flag4(pslot + 4 * q, p, fi - 4 * q, seq);
        else reinterpret_cast<float4*>(pbuf)[mp.g * nq + q] = p;
      }
#pragma unroll
      for (int i = 0; i < 8; i++)
        if (i < mp.nj) stw4<RES, L1R>(Wq + i * rstep, upd4(w[i], dsc[mp.g + (i << gs)], x), i);
      continue;
    }
    int j = 0;
    for (; j + 4 <= mp.nj; j += 4) {
      float4 w[4];
#pragma unroll
      for (int i = 0; i < 4; i++) w[i] = ldw4<RES, L1R>(Wq + (j + i) * rstep, j + i);
#pragma unroll
      for (int i = 0; i < 4; i++) {
        const int k = mp.g + ((j + i) << gs);
        const float d = delta[k];
        p.x = fmaf(w[i].x, d, p.x);
        p.y = fmaf(w[i].y, d, p.y);
        p.z = fmaf(w[i].z, d, p.z);
        p.w = fmaf(w[i].w, d, p.w);
        if (FUSE) stw4<RES, L1R>(Wq + (j + i) * rstep, upd4(w[i], dsc[k], x), j + i);
      }
    }
    for (; j < mp.nj; j++) {
      const float4 w = ldw4<RES, L1R>(Wq + j * rstep, j);
      const int k = mp.g + (j << gs);
      const float d = delta[k];
      p.x = fmaf(w.x, d, p.x);
      p.y = fmaf(w.y, d, p.y);
      p.z = fmaf(w.z, d, p.z);
      p.w = fmaf(w.w, d, p.w);
      if (FUSE) stw4<RES, L1R>(Wq + j * rstep, upd4(w, dsc[k], x), j);
    }
    if (4 * q < fi) {
      if (gs == 0) st_flag4(pslot + 4 * q, p, fi - 4 * q, seq);
      else reinterpret_cast<float4*>(pbuf)[mp.g * nq + q] = p;
    }
  }
  if (gs > 0) {
    __syncthreads();
    const int G = 1 << gs, pitch = nq * 4;
    for (int col = threadIdx.x; col < fi; col += kThreads) {
      float s = pbuf[col];
      for (int h = 1; h < G; h++) s += pbuf[h * pitch + col];
      st_flag(pslot + col, s, seq);
    }
  }
}

// w_ji += (eta*delta_j) * v_i over the owned rows and every column (bias:
// v_fi = 1; padding: v = 0 keeps the zeros), same thread mapping.
template <bool RES, int L1R = 0>
__device__ __forceinline__ void update_rows(float4* W4, int nq, int gs, int nr,
                                            const float4* __restrict__ v4,
                                            const float* __restrict__ dsc) {
  const RowMap mp(gs, nr);
  const int rstep = nq << gs;
  for (int q = mp.u; q < nq; q += mp.TG) {
    const float4 x = v4[q];
    float4* Wq = W4 + mp.g * nq + q;
    int j = 0;
    for (; j + 4 <= mp.nj; j += 4) {
      float4 w[4];
#pragma unroll
      for (int i = 0; i < 4; i++) w[i] = ldw4<RES, L1R>(Wq + (j + i) * rstep, j + i);
#pragma unroll
      for (int i = 0; i < 4; i++)
        stw4<RES, L1R>(Wq + (j + i) * rstep, upd4(w[i], dsc[mp.g + ((j + i) << gs)], x), j + i);
    }
    for (; j < mp.nj; j++)
      stw4<RES, L1R>(Wq + j * rstep, upd4(ldw4<RES, L1R>(Wq + j * rstep, j), dsc[mp.g + (j << gs)], x), j);
  }
}

// ---- register-resident row blocks -------------------------------------------
// A hidden layer whose owned rows do not fit in shared memory can live in the
// register file (256 KB per SM): thread t holds column t + 512*m (m < RC) of
// every owned row k < RR, zeros beyond the layer's rows and columns.  RS more
// column slots m = RC .. RC+RS-1 of the same mapping live in a shared-memory
// tail [RS][RR][512] (conflict-free: consecutive threads, consecutive words),
// so a layer slightly too wide for the register budget still avoids L2.  Its
// forward, column partials and update are then FMA work on registers; only
// the tail, the input vector and the deltas are read from shared memory.

template <int RR, int RS>
__device__ __forceinline__ float& tail_at(float* tail, int m, int k) {
  return tail[(m * RR + k) * kThreads + threadIdx.x];
}

template <int RR, int RC, int RS>
__device__ __forceinline__ void reg_load(float (&w)[RR][RC], float* tail,
                                         const float* __restrict__ g, int pitch, int nr) {
#pragma unroll
  for (int k = 0; k < RR; k++) {
#pragma unroll
    for (int m = 0; m < RC; m++) {
      const int c = threadIdx.x + kThreads * m;
      w[k][m] = (k < nr && c < pitch) ? g[k * pitch + c] : 0.0f;
    }
#pragma unroll
    for (int m = 0; m < RS; m++) {
      const int c = threadIdx.x + kThreads * (RC + m);
      tail_at<RR, RS>(tail, m, k) = (k < nr && c < pitch) ? g[k * pitch + c] : 0.0f;
    }
  }
}

template <int RR, int RC, int RS>
__device__ __forceinline__ void reg_store(const float (&w)[RR][RC], float* tail, float* g,
                                          int pitch, int nr) {
#pragma unroll
  for (int k = 0; k < RR; k++) {
#pragma unroll
    for (int m = 0; m < RC; m++) {
      const int c = threadIdx.x + kThreads * m;
      if (k < nr && c < pitch) g[k * pitch + c] = w[k][m];
    }
#pragma unroll
    for (int m = 0; m < RS; m++) {
      const int c = threadIdx.x + kThreads * (RC + m);
      if (k < nr && c < pitch) g[k * pitch + c] = tail_at<RR, RS>(tail, m, k);
    }
  }
}

template <int RR, int RC, int RS>
__device__ __forceinline__ void reg_fwd(const float (&w)[RR][RC], float* tail, int pitch, int nr,
                                        const float* __restrict__ v, float* red, float* tc,
                                        float* yown, unsigned long long* yslot, uint32_t seq) {
  static_assert(RR <= 16, "register row block: at most 16 rows");
  constexpr int CH = RR <= 4 ? 4 : RR <= 8 ? 8 : 16;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float acc[CH];
#pragma unroll
  for (int k = 0; k < CH; k++) acc[k] = 0.0f;
#pragma unroll
  for (int m = 0; m < RC; m++) {
    const int c = tid + kThreads * m;
    const float x = c < pitch ? v[c] : 0.0f;
#pragma unroll
    for (int k = 0; k < RR; k++) acc[k] = fmaf(w[k][m], x, acc[k]);
  }
#pragma unroll
  for (int m = 0; m < RS; m++) {
    const int c = tid + kThreads * (RC + m);
    const float x = c < pitch ? v[c] : 0.0f;
#pragma unroll
    for (int k = 0; k < RR; k++) acc[k] = fmaf(tail_at<RR, RS>(tail, m, k), x, acc[k]);
  }
  const float s = xpose_reduce<CH>(acc, lane);
  if ((lane & (32 / CH - 1)) == 0) red[warp * CH + lane / (32 / CH)] = s;
  cta_sync();
  if (tid < nr) {
    const float a = tree_sum<CH>(red + tid, kWarps);
    float t;
    const float y = tanh_scaled_noinline(a, &t);
    tc[tid] = t;
    if (yown) yown[tid] = y;
    if (yslot) st_flag(yslot + tid, y, seq);
  }
}

template <int RR, int RC, int RS>
__device__ __forceinline__ void reg_partials(const float (&w)[RR][RC], float* tail, int fi,
                                             int nr, const float* __restrict__ delta,
                                             unsigned long long* pslot, uint32_t seq) {
  // all RC + RS column chains advance together (k ascending in each, the same
  // sums as one chain at a time), then the stores
  float p[RC + RS];
#pragma unroll
  for (int m = 0; m < RC + RS; m++) p[m] = 0.0f;
#pragma unroll
  for (int k = 0; k < RR; k++) {
    const float d = k < nr ? delta[k] : 0.0f;
#pragma unroll
    for (int m = 0; m < RC + RS; m++)
      p[m] = fmaf(m < RC ? w[k][m < RC ? m : 0] : tail_at<RR, RS>(tail, m - RC, k), d, p[m]);
  }
#pragma unroll
  for (int m = 0; m < RC + RS; m++) {
    const int c = threadIdx.x + kThreads * m;
    if (c < fi) st_flag(pslot + c, p[m], seq);
  }
}

template <int RR, int RC, int RS>
__device__ __forceinline__ void reg_update(float (&w)[RR][RC], float* tail, int pitch, int nr,
                                           const float* __restrict__ v,
                                           const float* __restrict__ dsc) {
  float sk[RR];  // eta*delta of the rows, read once (the tail stores may alias smem)
#pragma unroll
  for (int k = 0; k < RR; k++) sk[k] = k < nr ? dsc[k] : 0.0f;
  float x[RC + RS];
#pragma unroll
  for (int m = 0; m < RC + RS; m++) {
    const int c = threadIdx.x + kThreads * m;
    x[m] = c < pitch ? v[c] : 0.0f;
  }
#pragma unroll
  for (int k = 0; k < RR; k++)
#pragma unroll
    for (int m = 0; m < RC; m++) w[k][m] = upd(w[k][m], sk[k], x[m]);
#pragma unroll
  for (int m = RC; m < RC + RS; m++)
#pragma unroll
    for (int k = 0; k < RR; k++)
      tail_at<RR, RS>(tail, m - RC, k) = upd(tail_at<RR, RS>(tail, m - RC, k), sk[k], x[m]);
}

// Poll a batch of U flag words per thread in rounds: every round re-issues
// the loads of all words not ready yet, so a late producer costs one L2
// round trip per round, not one per word.  Word u is base[off[u]]
// (off < 0: none); 32-bit offsets keep the register footprint small.
#ifndef DMLP_POLL_BACKOFF_NS
#define DMLP_POLL_BACKOFF_NS 0
#endif
template <int U>
__device__ __forceinline__ void poll_batch(const unsigned long long* base, const int (&off)[U],
                                           unsigned long long (&v)[U], uint32_t seq,
                                           int* err) {
#pragma unroll
  for (int u = 0; u < U; u++) v[u] = off[u] >= 0 ? ld_flag(base + off[u]) : 0ull;
  long long t0 = 0;
  for (int round = 0;; round++) {
    bool done = true;
#pragma unroll
    for (int u = 0; u < U; u++)
      if (off[u] >= 0 && (uint32_t)(v[u] >> 32) != seq) done = false;
    if (done) return;
    if ((round & 63) == 0) {  // the hang guard, off the per-round path (C5 +1.5%)
      if (round == 0) t0 = clock64();
      else if (clock64() - t0 > kSpinTimeoutCycles) spin_fail(err);
    }
    if (DMLP_POLL_BACKOFF_NS > 0) __nanosleep(DMLP_POLL_BACKOFF_NS);
#pragma unroll
    for (int u = 0; u < U; u++)
      if (off[u] >= 0 && (uint32_t)(v[u] >> 32) != seq) v[u] = ld_flag(base + off[u]);
  }
}

constexpr int kGatherU = 10;  // producer lines per warp per batch (16 warps x 10 >= 148)

// ---- own-column gather (forward) ---------------------------------------------
// Every thread of a consuming CTA needs only the input columns of its own
// quads (or register columns) -- the update of the same layer reads the same
// columns from the same thread -- so it polls exactly those words from the
// producers' slots and keeps them in its own smem positions.  No CTA barrier
// separates the exchange from the dot: a thread starts as soon as its own
// words have arrived, so the forward dot overlaps the tail of the exchange.
struct SrcSlots {
  const unsigned long long* src;  // this sample's [P][2^ylog] slots of the producing layer
  int R, ylog, fi;                // producer rows, slot stride (log2 words), consumer fan-in
  int flat;                       // word of column i at src[i] (LayerDev::yflat)
};

template <int U>
__device__ __forceinline__ void gather_cols(const SrcSlots& sl, const int (&col)[U], float* v,
                                            uint32_t seq, int* err) {
  int off[U];
#pragma unroll
  for (int j = 0; j < U; j++) {
    const int i = col[j];
    if (i >= 0 && i < sl.fi) {
      const int p = i / sl.R;
      off[j] = sl.flat ? i : (p << sl.ylog) + (i - p * sl.R);
    } else {
      off[j] = -1;
    }
  }
  unsigned long long val[U];
  poll_batch<U>(sl.src, off, val, seq, err);
#pragma unroll
  for (int j = 0; j < U; j++)
    if (off[j] >= 0) v[col[j]] = __uint_as_float((uint32_t)val[j]);
}

// The float4 quads u, u+TG, ... of the RowMap thread, one quad per poll
// batch when the layer has one quad per thread, else two.  One division per
// quad: its four columns are consecutive, so the producer index advances by
// carry.
__device__ __forceinline__ void quad_offsets(const SrcSlots& sl, int q, int (&off)[4]) {
  const int i0 = 4 * q;
  if (sl.flat) {
#pragma unroll
    for (int j = 0; j < 4; j++) off[j] = (i0 + j < sl.fi) ? i0 + j : -1;
    return;
  }
  int p = i0 / sl.R, r = i0 - p * sl.R;
#pragma unroll
  for (int j = 0; j < 4; j++) {
    off[j] = (i0 + j < sl.fi) ? (p << sl.ylog) + r : -1;
    if (++r == sl.R) r = 0, p++;
  }
}

__device__ __forceinline__ void gather_quads(const SrcSlots& sl, int nq, int gs, float* v,
                                             uint32_t seq, int* err) {
  const int TG = kThreads >> gs, u = threadIdx.x & (TG - 1);
  if (nq <= TG) {
    if (u >= nq) return;
    if ((sl.flat || (sl.R & 3) == 0) && 4 * u + 4 <= sl.fi) {
      // flat words, or producer blocks of a multiple of 4 rows: the quad is
      // 4 consecutive, 32-byte aligned words -> one 256-bit vector poll
      const int p = 4 * u / sl.R;
      const unsigned long long* a =
          sl.src + (sl.flat ? 4 * u : (p << sl.ylog) + (4 * u - p * sl.R));
      unsigned long long w0, w1, w2, w3;
      long long t0 = 0;
      for (int round = 0;; round++) {
        asm volatile("ld.relaxed.gpu.global.v4.b64 {%0, %1, %2, %3}, [%4];"
                     : "=l"(w0), "=l"(w1), "=l"(w2), "=l"(w3) : "l"(a) : "memory");
        if ((uint32_t)(w0 >> 32) == seq && (uint32_t)(w1 >> 32) == seq &&
            (uint32_t)(w2 >> 32) == seq && (uint32_t)(w3 >> 32) == seq)
          break;
        if ((round & 63) == 0) {  // the hang guard, off the per-round path
          if (round == 0) t0 = clock64();
          else if (clock64() - t0 > kSpinTimeoutCycles) spin_fail(err);
        }
      }
      reinterpret_cast<float4*>(v)[u] =
          make_float4(__uint_as_float((uint32_t)w0), __uint_as_float((uint32_t)w1),
                      __uint_as_float((uint32_t)w2), __uint_as_float((uint32_t)w3));
      return;
    }
    int off[4];
    quad_offsets(sl, u, off);
    unsigned long long val[4];
    poll_batch<4>(sl.src, off, val, seq, err);
#pragma unroll
    for (int j = 0; j < 4; j++)
      if (off[j] >= 0) v[4 * u + j] = __uint_as_float((uint32_t)val[j]);
    return;
  }
  for (int q = u; q < nq; q += 2 * TG) {
    int off[8];
    {
      int o4[4];
      quad_offsets(sl, q, o4);
#pragma unroll
      for (int j = 0; j < 4; j++) off[j] = o4[j];
      if (q + TG < nq) quad_offsets(sl, q + TG, o4);
      else o4[0] = o4[1] = o4[2] = o4[3] = -1;
#pragma unroll
      for (int j = 0; j < 4; j++) off[4 + j] = o4[j];
    }
    unsigned long long val[8];
    poll_batch<8>(sl.src, off, val, seq, err);
#pragma unroll
    for (int j = 0; j < 8; j++)
      if (off[j] >= 0) v[4 * (q + (j >> 2) * TG) + (j & 3)] = __uint_as_float((uint32_t)val[j]);
  }
}

// The columns t + 512*m (m < NC) of a register row block.
template <int NC>
__device__ __forceinline__ void gather_regcols(const SrcSlots& sl, float* v, uint32_t seq,
                                               int* err) {
  int col[NC];
#pragma unroll
  for (int m = 0; m < NC; m++) col[m] = threadIdx.x + kThreads * m;
  gather_cols<NC>(sl, col, v, seq, err);
}

// gather_sum for nr <= 32 / S rows: the S lane groups of a warp take
// alternate producers (group h of warp w sums producers w + 16h,
// w + 16h + 16S, ...), so a lane keeps 1/S as many polls in flight; the
// groups are then combined by a fixed butterfly (deterministic).
template <int S, class Fin>
__device__ __forceinline__ void gather_sum_split(const unsigned long long* src, int stride, int P,
                                                 int o, int nr, float* red, uint32_t seq,
                                                 int* err, Fin fin) {
  constexpr int W = 32 / S;                                   // lanes per group = max rows
  constexpr int U = (16 * kGatherU + 16 * S - 1) / (16 * S);  // >= 160 producers per batch
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int h = lane / W, k = lane % W;
  const bool kv = k < nr;
  float acc = 0.0f;
  for (int pb = 0; pb < P; pb += S * kWarps * U) {
    int off[U];
    unsigned long long v[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int p = pb + warp + kWarps * (S * u + h);
      off[u] = (kv && p < P) ? p * stride + o + k : -1;
    }
    poll_batch<U>(src, off, v, seq, err);
#pragma unroll
    for (int u = 0; u < U; u++)
      if (off[u] >= 0) acc += __uint_as_float((uint32_t)v[u]);
  }
#pragma unroll
  for (int m = 16; m >= W; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
  if (h == 0) red[warp * 32 + k] = acc;
  cta_sync();
  if (tid < nr) fin(tid, tree_sum<32>(red + tid, kWarps));
  __syncthreads();
}

// gather_sum for 16 < nr <= 32 rows: one warp per producer would leave
// 32 - nr lanes idle and give every lane ceil(P/16) polls (C4's 17 layer-0
// rows: 10).  Instead the CTA is cut into G = 512/nr packed groups of nr
// threads (17 rows: 30 groups, <= 5 polls per thread); group g sums
// producers g, g + G, ... in ascending order, then one thread per row adds
// the G group sums by a fixed pairwise tree (deterministic).  Measured and
// off by default (scripts/ab_perf.sh, same box): C4 37.4k -> 35.1k samples/s,
// C2 79.3k -> 78.9k, C1 +1%; build with -DDMLP_GATHER_PACK=1 to A/B it.
#ifndef DMLP_GATHER_PACK
#define DMLP_GATHER_PACK 0
#endif
template <class Fin>
__device__ __forceinline__ void gather_sum_packed(const unsigned long long* src, int stride, int P,
                                                  int o, int nr, float* red, uint32_t seq,
                                                  int* err, Fin fin) {
  constexpr int U = kGatherU;  // G >= 16 groups x 10 >= 160 producers per batch
  const int tid = threadIdx.x;
  const int G = kThreads / nr;
  const int g = tid / nr, k = tid - g * nr;
  const bool gv = g < G;
  float acc = 0.0f;
  for (int pb = 0; pb < P; pb += G * U) {
    int off[U];
    unsigned long long v[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int p = pb + g + G * u;
      off[u] = (gv && p < P) ? p * stride + o + k : -1;
    }
    poll_batch<U>(src, off, v, seq, err);
#pragma unroll
    for (int u = 0; u < U; u++)
      if (off[u] >= 0) acc += __uint_as_float((uint32_t)v[u]);
  }
  if (gv) red[g * nr + k] = acc;
  cta_sync();
  if (tid < nr) {
    float r[32];
#pragma unroll
    for (int i = 0; i < 32; i++) r[i] = i < G ? red[i * nr + tid] : 0.0f;
#pragma unroll
    for (int h = 16; h >= 1; h >>= 1)
#pragma unroll
      for (int i = 0; i < h; i++) r[i] += r[i + h];
    fin(tid, r[0]);
  }
  __syncthreads();
}

// s_k = sum over producers c < P of src[c*stride + o + k], k < nr, in a
// fixed order (producers c = w + 16*i summed by warp w in ascending i, then
// the 16 warp sums in ascending w): deterministic, independent of timing,
// no staging buffer.  fin(k, s_k) runs on one thread per k.
template <int SPLIT = 1, class Fin>
__device__ __forceinline__ void gather_sum(const unsigned long long* src, int stride, int P,
                                           int o, int nr, float* red, uint32_t seq, int* err,
                                           Fin fin) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (SPLIT >= 4 && nr <= 8) {
    gather_sum_split<4>(src, stride, P, o, nr, red, seq, err, fin);
    return;
  }
  if (SPLIT >= 2 && nr <= 16) {
    gather_sum_split<2>(src, stride, P, o, nr, red, seq, err, fin);
    return;
  }
  if (DMLP_GATHER_PACK && nr > 16 && nr <= 32) {
    gather_sum_packed(src, stride, P, o, nr, red, seq, err, fin);
    return;
  }
  for (int k0 = 0; k0 < nr; k0 += 32) {
    const int k = k0 + lane;
    const bool kv = k < nr;
    float acc = 0.0f;
    for (int pb = 0; pb < P; pb += kWarps * kGatherU) {
      int off[kGatherU];
      unsigned long long v[kGatherU];
#pragma unroll
      for (int u = 0; u < kGatherU; u++) {
        const int p = pb + warp + kWarps * u;
        off[u] = (kv && p < P) ? p * stride + o + k : -1;
      }
      poll_batch<kGatherU>(src, off, v, seq, err);
#pragma unroll
      for (int u = 0; u < kGatherU; u++)
        if (off[u] >= 0) acc += __uint_as_float((uint32_t)v[u]);
    }
    red[warp * 32 + lane] = acc;
    cta_sync();
    if (tid < 32 && k0 + tid < nr) {
      fin(k0 + tid, tree_sum<32>(red + tid, kWarps));
    }
    __syncthreads();
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

}  // namespace dmlp
