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

__device__ __noinline__ void spin_fail(int* err) {
  atomicExch(err, 1);
  __trap();
}
__device__ __noinline__ float tanh_scaled_noinline(float a, float* t) {
  return dev_scaled_tanh(a, t);
}

// Four consecutive flag words (16-byte aligned), the first `valid` of them.
__device__ __forceinline__ void st_flag4(unsigned long long* p, float4 x, int valid,
                                         uint32_t seq) {
  const unsigned long long h = (unsigned long long)seq << 32;
  const unsigned long long a = h | __float_as_uint(x.x), b = h | __float_as_uint(x.y);
  const unsigned long long c = h | __float_as_uint(x.z), d = h | __float_as_uint(x.w);
  if (valid >= 4) {
    asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b)
                 : "memory");
    asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p + 2), "l"(c), "l"(d)
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
template <bool RES>
__device__ __forceinline__ float4 ldw4(const float4* p) {
  if constexpr (RES) return *p;
  else return __ldcg(p);
}
template <bool RES>
__device__ __forceinline__ void stw4(float4* p, float4 v) {
  if constexpr (RES) *p = v;
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

// Forward of the owned rows [0, nr) of a hidden layer.  Per-thread partial
// rows over its quads, a transposing warp reduction, a fixed-order sum over
// the group's warps; one thread per row then applies the scaled tanh, caches
// t_j and publishes y_j (yslot) and/or keeps it (yown).
template <bool RES, int CH>
__device__ __forceinline__ void fwd_rows(const float4* __restrict__ W4, int nq, int gs, int nr,
                                         const float4* __restrict__ v4, float* red, float* tc,
                                         float* yown, unsigned long long* yslot, uint32_t seq) {
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
#pragma unroll
      for (int jj = 0; jj < CH; jj++)
        if (jj < jn) acc[jj] = dot4(ldw4<RES>(Wg + jj * rstep + q), x, acc[jj]);
    }
    const float s = xpose_reduce<CH>(acc, lane);
    if ((lane & (32 / CH - 1)) == 0) red[warp * CH + lane / (32 / CH)] = s;
    __syncthreads();
    if (tid < G * CH) {
      const int gg = tid / CH, jj = tid - gg * CH;
      const int k = gg + G * (j0 + jj);
      if (k < nr) {
        const float* r = red + gg * WG * CH + jj;
        float a = r[0];
        for (int w = 1; w < WG; w++) a += r[w * CH];
        float t;
        const float y = tanh_scaled_noinline(a, &t);
        tc[k] = t;
        if (yown) yown[k] = y;
        if (yslot) st_flag(yslot + k, y, seq);
      }
    }
    if (j0 + CH < njmax) __syncthreads();  // red is reused by the next chunk
  }
}

template <bool RES>
__device__ __forceinline__ void fwd_dispatch(const float4* W4, const LayerDev& ly, int nr,
                                             const float4* v4, float* red, float* tc,
                                             float* yown, unsigned long long* yslot,
                                             uint32_t seq) {
  const int nq = ly.pitch >> 2, gs = ly.gs;
  switch (ly.CH) {
    case 4: fwd_rows<RES, 4>(W4, nq, gs, nr, v4, red, tc, yown, yslot, seq); break;
    case 8: fwd_rows<RES, 8>(W4, nq, gs, nr, v4, red, tc, yown, yslot, seq); break;
    default: fwd_rows<RES, 16>(W4, nq, gs, nr, v4, red, tc, yown, yslot, seq); break;
  }
}

// Column partials of the owned rows of hidden layer l >= 1 with the OLD
// weights, published as flag words (bias column excluded, kernels.py:
// 129-153).  FUSE (streamed layers): the same pass writes the updated weight
// w + (eta*delta_j)*y_i, so each weight is read once and written once.
template <bool RES, bool FUSE>
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
    int j = 0;
    for (; j + 4 <= mp.nj; j += 4) {
      float4 w[4];
#pragma unroll
      for (int i = 0; i < 4; i++) w[i] = ldw4<RES>(Wq + (j + i) * rstep);
#pragma unroll
      for (int i = 0; i < 4; i++) {
        const int k = mp.g + ((j + i) << gs);
        const float d = delta[k];
        p.x = fmaf(w[i].x, d, p.x);
        p.y = fmaf(w[i].y, d, p.y);
        p.z = fmaf(w[i].z, d, p.z);
        p.w = fmaf(w[i].w, d, p.w);
        if (FUSE) stw4<RES>(Wq + (j + i) * rstep, upd4(w[i], dsc[k], x));
      }
    }
    for (; j < mp.nj; j++) {
      const float4 w = ldw4<RES>(Wq + j * rstep);
      const int k = mp.g + (j << gs);
      const float d = delta[k];
      p.x = fmaf(w.x, d, p.x);
      p.y = fmaf(w.y, d, p.y);
      p.z = fmaf(w.z, d, p.z);
      p.w = fmaf(w.w, d, p.w);
      if (FUSE) stw4<RES>(Wq + j * rstep, upd4(w, dsc[k], x));
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
template <bool RES>
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
      for (int i = 0; i < 4; i++) w[i] = ldw4<RES>(Wq + (j + i) * rstep);
#pragma unroll
      for (int i = 0; i < 4; i++)
        stw4<RES>(Wq + (j + i) * rstep, upd4(w[i], dsc[mp.g + ((j + i) << gs)], x));
    }
    for (; j < mp.nj; j++)
      stw4<RES>(Wq + j * rstep, upd4(ldw4<RES>(Wq + j * rstep), dsc[mp.g + (j << gs)], x));
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

constexpr int kGatherU = 10;  // producer lines per warp per batch (16 warps x 10 >= 148)

// Gather y of hidden layer `ly` into dst (protocol E).  Producer p's rows sit
// in its own line-aligned slot; each warp instruction reads one producer's
// slot (lane = row within the block, 32-row segments when R > 32) and every
// thread keeps all of its loads in flight, re-polling only the words whose
// flag is not yet this sample's.
__device__ __forceinline__ void gather_y(const unsigned long long* src, const LayerDev& ly,
                                         float* dst, uint32_t seq, int* err) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nseg = (ly.R + 31) >> 5, V = ly.P * nseg;
  for (int vb = 0; vb < V; vb += kWarps * kGatherU) {
    const unsigned long long* ptr[kGatherU];
    unsigned long long v[kGatherU];
#pragma unroll
    for (int u = 0; u < kGatherU; u++) {
      const int vi = vb + warp + kWarps * u;
      const int p = nseg == 1 ? vi : vi / nseg;
      const int k = (vi - p * nseg) * 32 + lane;
      const bool ok = vi < V && k < ly.R && p * ly.R + k < ly.fo;
      ptr[u] = ok ? src + ((size_t)p << ly.ylog) + k : nullptr;
      v[u] = ok ? ld_flag(ptr[u]) : 0ull;
    }
    poll_batch<kGatherU>(ptr, v, seq, err);
#pragma unroll
    for (int u = 0; u < kGatherU; u++)
      if (ptr[u] != nullptr) {
        const int vi = vb + warp + kWarps * u;
        const int p = nseg == 1 ? vi : vi / nseg;
        dst[p * ly.R + (vi - p * nseg) * 32 + lane] = __uint_as_float((uint32_t)v[u]);
      }
  }
}

// s_k = sum over producers c < P of src[c*stride + off + k], k < nr, in a
// fixed order (producers c = w + 16*i summed by warp w in ascending i, then
// the 16 warp sums in ascending w): deterministic, independent of timing,
// no staging buffer.  fin(k, s_k) runs on one thread per k.
template <class Fin>
__device__ __forceinline__ void gather_sum(const unsigned long long* src, int stride, int P,
                                           int off, int nr, float* red, uint32_t seq, int* err,
                                           Fin fin) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int k0 = 0; k0 < nr; k0 += 32) {
    const int k = k0 + lane;
    const bool kv = k < nr;
    float acc = 0.0f;
    for (int pb = 0; pb < P; pb += kWarps * kGatherU) {
      const unsigned long long* ptr[kGatherU];
      unsigned long long v[kGatherU];
#pragma unroll
      for (int u = 0; u < kGatherU; u++) {
        const int p = pb + warp + kWarps * u;
        const bool ok = kv && p < P;
        ptr[u] = ok ? src + (size_t)p * stride + off + k : nullptr;
        v[u] = ok ? ld_flag(ptr[u]) : 0ull;
      }
      poll_batch<kGatherU>(ptr, v, seq, err);
#pragma unroll
      for (int u = 0; u < kGatherU; u++)
        if (ptr[u] != nullptr) acc += __uint_as_float((uint32_t)v[u]);
    }
    red[warp * 32 + lane] = acc;
    __syncthreads();
    if (tid < 32 && k0 + tid < nr) {
      float s = red[tid];
      for (int w = 1; w < kWarps; w++) s += red[w * 32 + tid];
      fin(k0 + tid, s);
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
