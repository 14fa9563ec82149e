// train_kernel.cuh -- persistent on-line back-propagation kernel (sm_100a).
//
// The kernel template; train_inst_f*.cu instantiate it (one translation unit
// per feature set, compiled in parallel) and train_glue.cu launches it.
//
// Replaces trainer.train_epoch's per-sample Python loop (trainer.py:104-123)
// and kernels.train_step (kernels.py:329-361): ONE launch trains a whole
// sequence of samples.  Design:
//
//  * Row ownership.  CTA c owns the row block [c*R, c*R+R) of every hidden
//    layer.  Inside the CTA, thread (g, u) owns rows g, g+G, ... and columns
//    u, u+TG, ... of the block (LayerDev), so the forward dot, the column
//    partials and the update all run on every thread, lanes on consecutive
//    columns (conflict-free smem, 128-byte coalesced L2 lines).
//  * Forward a_j = W_j . y is CTA-local: per-thread partial rows, a
//    transposing warp reduction (one value per lane pair), a fixed-order sum
//    over the group's warps, then bias-included exact scaled tanh on one
//    thread per row, which publishes y_j straight away.
//  * Output layer by COLUMN ownership: CTA c keeps the columns of W_out that
//    match its rows of the last hidden layer and publishes the fo partial
//    pre-activations of those columns instead of its y; every CTA sums the
//    partials in fixed producer order.  The last hidden layer's y is never
//    exchanged, and the output delta, the deltas of the owned last-hidden
//    rows and the W_out update are all local.
//  * Backward of hidden layer l: column partials P_c[i] = sum_j w_ji*delta_j
//    with the OLD weights, published as soon as they are formed; the update
//    w_ji + (eta*delta_j)*y_i (mul then add, no FMA -- kernels.py:174,182)
//    runs while the partials travel (smem-resident layers) or in the same
//    pass (L2-streamed layers: one read, one write per weight).  The owners
//    of layer l-1's rows sum the partials over producers in a fixed order.
//  * No grid barrier.  Every cross-CTA value travels as a 64-bit word
//    {float value, u32 sample-sequence flag} written with one st.relaxed.gpu
//    and polled with ld.relaxed.gpu until the flag matches: data and its
//    readiness arrive in one single-copy-atomic access.  Each producer's
//    words start on their own 128-byte line (one writer per polled line),
//    buffers alternate by sample parity, and every consumer keeps all its
//    polls in flight (protocol E, profiles/r1_microbench.json).
#pragma once
#include <cuda_runtime.h>

#include "dmlp_internal.h"
#include "dmlp_math.cuh"
#include "train_phases.cuh"

namespace dmlp {

constexpr int kProfSlots = kProfWords;
// gather_sum lane groups per register plan (compile time: selecting at run
// time cost C4 ~4%): halves for <= 16 rows (C4 36.3k -> 37.4k samples/s, C5
// +3.6%), quarters for <= 8 rows with the 1000-wide plans (C1, C5), none
// without register rows (C2: halves -2.2%)
#ifndef DMLP_GATHER_SPLIT
#define DMLP_GATHER_SPLIT(NRL, RR) ((NRL) == 0 ? 1 : (RR) <= 8 ? 4 : 2)
#endif
// FEAT: which residency paths are compiled in (kFeatSmem: shared-memory
// hidden layers, kFeatL2: L2-streamed ones; register row blocks always):
// code a net never runs still costs registers and instruction fetch in the
// hot loop (C1, registers only: +8.8% without the smem/L2 paths).
// PROF: the in-kernel phase profile and the one-sample timeline are compiled
// in (selected only while profiling or tracing is enabled: the hooks cost
// 1.5-7.5% even when switched off at run time).
template <int NRL, int RR, int RC, int RS, int FEAT, bool PROF>
__global__ void __launch_bounds__(kThreads, 1)
    k_train(const NetDev net, const float* __restrict__ X, long long ldx,
            const uint8_t* __restrict__ labels, const int32_t* __restrict__ order,
            long long n, float eta, uint32_t seq0, unsigned long long* wrong_out,
            float* y_last, uint8_t* pred) {
  extern __shared__ __align__(16) float sm[];
  __shared__ int g_r0[kMaxLayers], g_nr[kMaxLayers];
  __shared__ int g_rb[kMaxLayers];  // forward reduction buffer offset per layer
#ifndef DMLP_CTA_ROT
#define DMLP_CTA_ROT 0  // experiments: logical CTA = (blockIdx + ROT) mod grid
#endif
  const int c = DMLP_CTA_ROT ? (blockIdx.x + DMLP_CTA_ROT) % gridDim.x : blockIdx.x;
  const int tid = threadIdx.x;
  const int L = net.L, H = L - 1;  // H hidden layers
  // streamed rows per thread cached in L1 (kFeatL1 instances: layer 0 is never
  // streamed there, and the one streamed layer has <= 8 rows per thread)
  constexpr int kL1R = (FEAT & kFeatL1) ? kL1Rows : 0;
  float* red = sm + net.red_off;
  float* pbuf = sm + net.pbuf_off;
  float* outv = sm + net.out_off;  // a | y | delta | eta*delta
  const LayerDev& lo = net.ly[L - 1];
  const int OT = lo.R + 1;  // output tile row stride: owned columns + bias column
  float* otile = sm + lo.wsm_off;
  float wr[NRL > 0 ? NRL : 1][RR][RC];  // register-resident row blocks (kResReg layers)

  if (tid < H) {
    const LayerDev& ly = net.ly[tid];
    const int r0 = min(c * ly.R, ly.fo);
    g_r0[tid] = r0;
    g_nr[tid] = min(ly.R, ly.fo - r0);
    int nown = 0;  // owned layers below this one: owned layers alternate buffers
    for (int j = 0; j < tid; j++) nown += c < net.ly[j].P;
    g_rb[tid] = (nown & 1) * kWarps * 32;
  }
  // Owned output columns: those of the CTA's last-hidden rows (all inputs
  // when there is no hidden layer; then the launch has one CTA).
  const int oc0 = H > 0 ? min(c * lo.R, lo.fi) : 0;
  const int onc = H > 0 ? min(lo.R, lo.fi - oc0) : lo.fi;
  const bool oown = onc > 0 || c == 0;
  // Constant tails of every input vector: 1.0 in the bias column, zeros after.
  for (int b = 0; b < 2; b++) {
    float* v = sm + net.in0_off[b];
    for (int i = net.ly[0].fi + tid; i < net.ly[0].pitch; i += kThreads)
      v[i] = (i == net.ly[0].fi) ? 1.0f : 0.0f;
  }
  for (int l = 1; l < H; l++) {
    float* v = sm + net.ly[l].in_off;
    for (int i = net.ly[l].fi + tid; i < net.ly[l].pitch; i += kThreads)
      v[i] = (i == net.ly[l].fi) ? 1.0f : 0.0f;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NRL; i++) {  // register-resident row blocks
    const int l = net.reg_layer[i];
    if (l < 0) {  // slot unused by this net's plan
#pragma unroll
      for (int k = 0; k < RR; k++)
#pragma unroll
        for (int m = 0; m < RC; m++) wr[i][k][m] = 0.0f;
      continue;
    }
    const LayerDev& ly = net.ly[l];
    const int r0 = min(c * ly.R, ly.fo), nr = min(ly.R, ly.fo - r0);
    reg_load<RR, RC, RS>(wr[i], sm + ly.wsm_off, ly.w + (size_t)r0 * ly.pitch, ly.pitch, nr);
  }
  for (int l = 0; l < H; l++) {  // smem-resident hidden layers: load the rows once
    const LayerDev& ly = net.ly[l];
    if (!(FEAT & kFeatSmem) || ly.res != kResSmem) continue;
    const float4* g = reinterpret_cast<const float4*>(ly.w + (size_t)g_r0[l] * ly.pitch);
    float4* s = reinterpret_cast<float4*>(sm + ly.wsm_off);
    for (int i = tid; i < g_nr[l] * ly.pitch / 4; i += kThreads) s[i] = g[i];
  }
  for (int i = tid; i < lo.fo * OT; i += kThreads) {  // output tile (+ bias column)
    const int j = i / OT, k = i - j * OT;
    float w = 0.0f;
    if (k < onc) w = lo.w[(size_t)j * lo.pitch + oc0 + k];
    else if (k == OT - 1 && c == 0) w = lo.w[(size_t)j * lo.pitch + lo.fi];
    otile[i] = w;
  }

  // Sample indices and labels are loaded ahead so no dependent global load
  // sits at the head of a sample.
  const int img_cur = n > 0 ? (order ? order[0] : 0) : 0;
  int img_nxt = n > 1 ? (order ? order[1] : 1) : -1;
  int digit_cur = n > 0 ? labels[img_cur] : 0;
  if (n > 0) {
    for (int i = tid; i < net.ly[0].fi; i += kThreads)
      cp_async4(sm + net.in0_off[0] + i, X + (long long)img_cur * ldx + i);
    cp_async_commit();
  }
  __shared__ unsigned long long s_wrong;  // counted by the last thread of CTA 0
  if (tid == 0) s_wrong = 0;
  const bool counter = (c == 0 && tid == kThreads - 1);
  // optional in-kernel profile (thread 0 of every CTA): per-phase cycles.
  // slot 0 loop total, 1 exchange waits; 2.. per phase (device.py names them).
  const bool prof = PROF && net.prof != nullptr && tid == 0;
  __shared__ long long ph[kProfSlots];  // per-phase cycles (thread 0 only)
  for (int i = tid; i < kProfSlots; i += kThreads) ph[i] = 0;
  // thread 0's clocks live in smem: no registers held across the loop
  __shared__ long long pt[4];  // loop start, exchange total, exchange mark, phase mark
  if (prof) pt[0] = pt[3] = clock64(), pt[1] = pt[2] = 0;
  if (prof) {  // slot 12: the SM this CTA ran on, + 1 (per-CTA readout: dmlp_net_read_profile_cta)
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    ph[12] = smid + 1;
  }
#define t_loop0 pt[0]
#define t_xchg pt[1]
#define t_mark pt[2]
#define t_ph pt[3]
#define PH(slot)                    \
  if (prof) {                       \
    const long long _t = clock64(); \
    ph[slot] += _t - t_ph;          \
    t_ph = _t;                      \
  }
  // PHL: the same, also booked to layer `ly_` under per-layer kind `k_`.
#define PHL(slot, ly_, k_)                                   \
  if (prof) {                                                \
    const long long _t = clock64();                          \
    ph[slot] += _t - t_ph;                                   \
    ph[kProfPhases + kProfKinds * (ly_) + (k_)] += _t - t_ph; \
    t_ph = _t;                                               \
  }
#define XB() \
  if (prof) t_mark = clock64();
#define XE() \
  if (prof) t_xchg += clock64() - t_mark;
  // optional one-sample timeline: CTA-synchronised %globaltimer marks.
  // mark 0 sample start; for exchange e: 1+2e producer side done, 2+2e
  // gather done (forward y exchanges e = 0..L-3, output partials e = L-2,
  // backward e = L-1..2L-4); 63 sample end.
#define TRACE(mark)                                                          \
  if (PROF && net.trace != nullptr && s == net.trace_sample) {              \
    __syncthreads();                                                          \
    if (tid == 0) {                                                           \
      unsigned long long _g;                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_g));                \
      net.trace[(size_t)c * 64 + (mark)] = _g;                                \
    }                                                                         \
  }

  for (int s = 0; s < n; s++) {
    const uint32_t seq = seq0 + (uint32_t)s;
    const int buf = seq & 1;
    const int img_nn = (s + 2 < n) ? (order ? order[s + 2] : s + 2) : -1;
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
        cp_async4(nx + i, X + (long long)img_nxt * ldx + i);
      cp_async_commit();
    }
    PH(13);

    // ---------------- forward: hidden layers ----------------
    for (int l = 0; l < H; l++) {
      const LayerDev& ly = net.ly[l];
      const bool mine = c < ly.P;
      if (l > 0) {  // y of layer l-1: each thread polls the columns it consumes
        const LayerDev& lp = net.ly[l - 1];
        XB();
        if (mine) {
          const SrcSlots sl{lp.yll + ((size_t)buf * lp.P << lp.ylog), lp.R, lp.ylog, ly.fi,
                           lp.yflat};
          if (ly.res == kResReg) gather_regcols<RC + RS>(sl, sm + ly.in_off, seq, net.err);
          else if (FEAT & (kFeatSmem | kFeatL2))
            gather_quads(sl, ly.pitch >> 2, ly.gs, sm + ly.in_off, seq, net.err);
        }
        XE();
        PHL(4, l, 1);
        TRACE(2 + 2 * (l - 1));
      }
      if (mine) {
        // consecutive OWNED layers alternate reduction buffers: the barrier
        // inside the forward of the owned layer between two users of one
        // buffer orders the later writes after the earlier reads (a CTA may
        // own layers l and l+2 but not l+1)
        float* redl = red + g_rb[l];
        const float4* v4 = reinterpret_cast<const float4*>(l == 0 ? in0 : sm + ly.in_off);
        unsigned long long* ys =
            (l < H - 1) ? ly.yll + ((size_t)buf * ly.P << ly.ylog) +
                              (ly.yflat ? (size_t)g_r0[l] : ((size_t)c << ly.ylog))
                        : nullptr;
        float* yo = (l == H - 1) ? sm + net.yown_off : nullptr;
        if (ly.res == kResReg) {
#pragma unroll
          for (int i = 0; i < NRL; i++)
            if (net.reg_layer[i] == l)
              reg_fwd<RR, RC, RS>(wr[i], sm + ly.wsm_off, ly.pitch, g_nr[l],
                                  reinterpret_cast<const float*>(v4), redl, sm + ly.t_off, yo,
                                  ys, seq);
        } else if ((FEAT & kFeatSmem) && ly.res == kResSmem)
          fwd_dispatch<true>(reinterpret_cast<const float4*>(sm + ly.wsm_off), ly, g_nr[l], v4,
                             redl, sm + ly.t_off, yo, ys, seq, (prof && l == 0) ? ph + 14 : nullptr);
        else if (FEAT & kFeatL2)
          fwd_dispatch<false, kL1R>(reinterpret_cast<const float4*>(ly.w + (size_t)g_r0[l] * ly.pitch),
                              ly, g_nr[l], v4, redl, sm + ly.t_off, yo, ys, seq);
      }
      PHL(3, l, 0);
      if (l < H - 1) TRACE(1 + 2 * l);
    }

    // np.argmax of the output (first maximum; NaN counts as maximum) by one
    // thread of CTA 0.  (Deferring it past the first backward publish or to
    // the end of the sample measured slower: scripts/ab_perf.sh.)
    auto count_error = [&]() {
      if (counter) {
        int best = 0;
        float bv = outv[kMaxOut];
        for (int k = 1; k < lo.fo && !(bv != bv); k++) {
          const float yk = outv[kMaxOut + k];
          if (yk > bv || yk != yk) { bv = yk; best = k; }
        }
        s_wrong += (best != digit);
        if (pred != nullptr) pred[s] = (uint8_t)best;
      }
    };

    // ---------------- output layer: partials of the owned columns ----------------
    const float* yin = H > 0 ? sm + net.yown_off : in0;
    __syncthreads();
    // fo partials, padded with zero words up to whole 32-byte sectors (the
    // slot is line aligned): no partially written sector
    if (oown && tid < ((lo.fo + 3) & ~3)) {
      float a = 0.0f;
      if (tid < lo.fo) {
        const float* wr = otile + tid * OT;
        for (int k = 0; k < onc; k++) a = fmaf(wr[k], yin[k], a);
        if (c == 0) a += wr[OT - 1];  // bias
      }
      st_flag(lo.yll + ((size_t)buf * lo.P << lo.ylog) + ((size_t)c << lo.ylog) + tid, a, seq);
    }
    PH(5);
    TRACE(1 + 2 * (L - 2));
    XB();
    // the output activation and delta are formed by the thread that finishes
    // the sum (gather_sum's closing barrier publishes them to the CTA)
    if (oown)
      gather_sum<DMLP_GATHER_SPLIT(NRL, RR)>(lo.yll + ((size_t)buf * lo.P << lo.ylog), 1 << lo.ylog, lo.P, 0, lo.fo, red, seq,
                 net.err, [&](int k, float a) {
                   float t;
                   const float y = tanh_scaled_noinline(a, &t);
                   const float d = dev_output_delta_t(y, t, k == digit ? 1.0f : -1.0f);
                   outv[k] = a;
                   outv[kMaxOut + k] = y;
                   outv[2 * kMaxOut + k] = d;
                   outv[3 * kMaxOut + k] = __fmul_rn(eta, d);
                 });
    else
      __syncthreads();
    XE();
    PH(6);
    TRACE(2 + 2 * (L - 2));
    if (oown) {
      count_error();
      if (c == 0 && s == n - 1 && y_last != nullptr && tid < lo.fo)
        y_last[tid] = outv[kMaxOut + tid];
      // Deltas of the owned last-hidden rows through the OLD output weights,
      // sequential over the output rows -- the reference's single-tile
      // order (kernels.py:149-153) exactly -- then this thread's column of
      // the output tile is updated (the same thread read it first).
      const float* dout = outv + 2 * kMaxOut;
      const float* sout = outv + 3 * kMaxOut;
      for (int k = tid; k < onc + (c == 0); k += kThreads) {
        if (k < onc) {
          const float yk = yin[k];
          float acc = 0.0f;
#pragma unroll 10
          for (int j = 0; j < lo.fo; j++) {
            const float w = otile[j * OT + k];
            acc = __fadd_rn(acc, __fmul_rn(w, dout[j]));
            otile[j * OT + k] = upd(w, sout[j], yk);
          }
          if (H > 0) {
            const float d = dev_hidden_delta(acc, sm[net.ly[H - 1].t_off + k]);
            sm[net.delta_off[0] + k] = d;
            sm[net.dsc_off[0] + k] = __fmul_rn(eta, d);
          }
        } else {  // bias column (CTA 0): w + (eta*delta)*1
#pragma unroll 10
          for (int j = 0; j < lo.fo; j++)
            otile[j * OT + OT - 1] = __fadd_rn(otile[j * OT + OT - 1], sout[j]);
        }
      }
    }
    __syncthreads();
    PH(7);

    // ---------------- backward + update: hidden layers H-1 .. 1 ----------------
    int cur = 0;
    for (int l = H - 1; l >= 1; l--) {
      const LayerDev& ly = net.ly[l];
      unsigned long long* pb = ly.pll + (size_t)buf * ly.P * ly.pstride;
      const float* dl = sm + net.delta_off[cur];
      const float* sl = sm + net.dsc_off[cur];
      const bool mine = c < ly.P;
      if (mine) {
        unsigned long long* ps = pb + (size_t)c * ly.pstride;
        const float4* v4 = reinterpret_cast<const float4*>(sm + ly.in_off);
        if (ly.res == kResReg) {
#pragma unroll
          for (int i = 0; i < NRL; i++)
            if (net.reg_layer[i] == l)
              reg_partials<RR, RC, RS>(wr[i], sm + ly.wsm_off, ly.fi, g_nr[l], dl, ps, seq);
        } else if ((FEAT & kFeatSmem) && ly.res == kResSmem) {
          // plans without register rows, <= 8 rows per thread group: the
          // update is fused into the same pass (every row's weights in flight,
          // the partials published before the updated weights are stored: one
          // read, one write per weight; C2 +2%).  Elsewhere it measured slower
          // (C4 -2 to -5%, C3 -3%): those layers update separately while the
          // partials travel
          if (NRL == 0 && (((g_nr[l] - 1) >> ly.gs) + 1) <= 8)
            bwd_partials<true, true>(reinterpret_cast<float4*>(sm + ly.wsm_off), ly.pitch >> 2,
                                     ly.fi, ly.gs, g_nr[l], dl, sl, v4, pbuf, ps, seq);
          else
            bwd_partials<true, false>(reinterpret_cast<float4*>(sm + ly.wsm_off), ly.pitch >> 2,
                                      ly.fi, ly.gs, g_nr[l], dl, sl, v4, pbuf, ps, seq);
        }
        else if (FEAT & kFeatL2)
          bwd_partials<false, true, kL1R>(
              reinterpret_cast<float4*>(ly.w + (size_t)g_r0[l] * ly.pitch), ly.pitch >> 2,
              ly.fi, ly.gs, g_nr[l], dl, sl, v4, pbuf, ps, seq);
      }
      PHL(8, l, 2);
      TRACE(1 + 2 * (L - 1 + (H - 1 - l)));
      if ((FEAT & kFeatSmem) && mine && ly.res == kResSmem &&
          !(NRL == 0 && (((g_nr[l] - 1) >> ly.gs) + 1) <= 8))
        update_rows<true>(reinterpret_cast<float4*>(sm + ly.wsm_off), ly.pitch >> 2, ly.gs,
                          g_nr[l], reinterpret_cast<const float4*>(sm + ly.in_off), sl);
      if (mine && ly.res == kResReg) {
#pragma unroll
        for (int i = 0; i < NRL; i++)
          if (net.reg_layer[i] == l)
            reg_update<RR, RC, RS>(wr[i], sm + ly.wsm_off, ly.pitch, g_nr[l], sm + ly.in_off,
                                   sl);
      }
      PHL(9, l, 3);
      const int nxt = cur ^ 1;
      const LayerDev& lb = net.ly[l - 1];
      float* dn = sm + net.delta_off[nxt];
      float* sn = sm + net.dsc_off[nxt];
      const float* tcb = sm + lb.t_off;
      XB();
      if (c < lb.P)
        gather_sum<DMLP_GATHER_SPLIT(NRL, RR)>(pb, ly.pstride, ly.P, g_r0[l - 1], g_nr[l - 1], red, seq, net.err,
                   [&](int k, float a) {
                     const float d = dev_hidden_delta(a, tcb[k]);
                     dn[k] = d;
                     sn[k] = __fmul_rn(eta, d);
                   });
      else
        __syncthreads();
      XE();
      PHL(10, l, 4);
      TRACE(2 + 2 * (L - 1 + (H - 1 - l)));
      cur = nxt;
    }
    if (H > 0 && c < net.ly[0].P) {
      const LayerDev& l0 = net.ly[0];
      const float4* x4 = reinterpret_cast<const float4*>(in0);
      if (l0.res == kResReg) {
#pragma unroll
        for (int i = 0; i < NRL; i++)
          if (net.reg_layer[i] == 0)
            reg_update<RR, RC, RS>(wr[i], sm + l0.wsm_off, l0.pitch, g_nr[0], in0,
                                   sm + net.dsc_off[cur]);
      } else if ((FEAT & kFeatSmem) && l0.res == kResSmem)
        update_rows<true>(reinterpret_cast<float4*>(sm + l0.wsm_off), l0.pitch >> 2, l0.gs,
                          g_nr[0], x4, sm + net.dsc_off[cur]);
      else if (FEAT & kFeatL2)
        update_rows<false, kL1R>(reinterpret_cast<float4*>(l0.w + (size_t)g_r0[0] * l0.pitch),
                           l0.pitch >> 2, l0.gs, g_nr[0], x4, sm + net.dsc_off[cur]);
    }
    PH(11);
    TRACE(63);
    img_nxt = img_nn;
    digit_cur = digit_nxt;
  }
  __syncthreads();

#pragma unroll
  for (int i = 0; i < NRL; i++) {
    const int l = net.reg_layer[i];
    if (l < 0) continue;
    const LayerDev& ly = net.ly[l];
    const int r0 = min(c * ly.R, ly.fo), nr = min(ly.R, ly.fo - r0);
    reg_store<RR, RC, RS>(wr[i], sm + ly.wsm_off, ly.w + (size_t)r0 * ly.pitch, ly.pitch, nr);
  }
  for (int l = 0; l < H; l++) {  // write the resident rows back
    const LayerDev& ly = net.ly[l];
    if (!(FEAT & kFeatSmem) || ly.res != kResSmem) continue;
    float4* g = reinterpret_cast<float4*>(ly.w + (size_t)g_r0[l] * ly.pitch);
    const float4* s = reinterpret_cast<const float4*>(sm + ly.wsm_off);
    for (int i = tid; i < g_nr[l] * ly.pitch / 4; i += kThreads) g[i] = s[i];
  }
  for (int i = tid; i < lo.fo * OT; i += kThreads) {
    const int j = i / OT, k = i - j * OT;
    if (k < onc) lo.w[(size_t)j * lo.pitch + oc0 + k] = otile[i];
    else if (k == OT - 1 && c == 0) lo.w[(size_t)j * lo.pitch + lo.fi] = otile[i];
  }
  if (prof) {
    ph[0] = clock64() - t_loop0;
    ph[1] = t_xchg;
    for (int k = 0; k < kProfSlots; k++)
      atomicAdd(net.prof + kProfSlots * c + k, (unsigned long long)ph[k]);
  }
#undef PH
#undef t_loop0
#undef t_xchg
#undef t_mark
#undef t_ph
#undef PHL
#undef XB
#undef XE
#undef TRACE
  if (counter && wrong_out != nullptr) atomicAdd(wrong_out, s_wrong);
}

// The compiled register plans (NRL, RR, RC, RS): none; one 14-row block of
// 4 register column slots + 1 shared-memory slot (the 2000x2501 hidden layer
// of C4: 14 rows x 2504 columns per CTA); up to four 7-row x 2-column blocks
// and three 8-row x 2-column blocks (1000-wide layers: C5, C1).
#define DMLP_REGISTER_PLANS(X) X(0, 1, 1, 0) X(1, 14, 4, 1) X(2, 7, 2, 0) X(4, 7, 2, 0) X(3, 8, 2, 0)
constexpr int kNumPlans = 5;

}  // namespace dmlp
