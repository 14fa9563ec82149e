// capi.cu -- the extern "C" boundary of libdmlp.so (see include/dmlp.h).
//
// Owns the network state that the reference keeps in network.Mlp
// (network.py:87-106): device weights in the kernel's padded row layout,
// the flag-word exchange buffers of the persistent kernel, and the sample
// sequence counter that tags every exchanged word.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "dmlp_internal.h"

namespace dmlp {

static thread_local std::string g_err;

int set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return DMLP_OK;
  return set_error(DMLP_ECUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

// Every operation on a net waits for the previous one (whatever stream it ran
// on) and records net->done when it is enqueued: weights are never read or
// written concurrently by two streams.
int net_begin(dmlp_net* net, cudaStream_t st) {
  return cuda_check(cudaStreamWaitEvent(st, net->done, 0), "cudaStreamWaitEvent");
}
int net_end(dmlp_net* net, cudaStream_t st) {
  return cuda_check(cudaEventRecord(net->done, st), "cudaEventRecord");
}

#define DMLP_CUDA(call)                                 \
  do {                                                  \
    int _rc = ::dmlp::cuda_check((call), #call);        \
    if (_rc != DMLP_OK) return _rc;                     \
  } while (0)

static int round_up(int x, int m) { return (x + m - 1) / m * m; }

// Plan-override knobs for A/B experiments (DMLP_YFLAT, DMLP_GS,
// DMLP_FORCE_VARIANT, DMLP_FEAT, DMLP_SMEM_EXCLUDE).  Read only in builds made with
// -DDMLP_EXPERIMENT_KNOBS (scripts/ab_perf.sh); the product library never
// lets the environment change a net's kernel plan.
static const char* knob(const char* name) {
#ifdef DMLP_EXPERIMENT_KNOBS
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

// Reference layout (fo, fi+1) row-major -> device rows of `pitch` floats.
__global__ void k_pack(const float* __restrict__ src, float* __restrict__ dst, int fo, int fi,
                       int pitch) {
  const long long total = (long long)fo * pitch;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(t / pitch), i = (int)(t % pitch);
    dst[t] = (i <= fi) ? src[(long long)j * (fi + 1) + i] : 0.0f;
  }
}

__global__ void k_unpack(const float* __restrict__ src, float* __restrict__ dst, int fo, int fi,
                         int pitch) {
  const long long total = (long long)fo * (fi + 1);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(t / (fi + 1)), i = (int)(t % (fi + 1));
    dst[t] = src[(long long)j * pitch + i];
  }
}

// Rows per CTA block: CTA c owns rows [c*R, min(c*R + R, fo)).
static int own_max_rows(int fo, int nct) { return (fo + nct - 1) / nct; }
static int ceil_log2(int x) {
  int l = 0;
  while ((1 << l) < x) l++;
  return l;
}

// Lay out dynamic shared memory for a resident-layer mask (hidden layers);
// returns bytes.
static int layout_smem(dmlp_net* net, unsigned mask, unsigned regmask = 0,
                       int reg_tail_floats = 0) {
  NetDev& d = net->dev;
  const int L = d.L, H = L - 1;
  int off = 0;
  auto take = [&](int floats) {
    const int o = off;
    off += round_up(floats > 0 ? floats : 1, 4);
    return o;
  };
  d.in0_off[0] = take(d.ly[0].pitch);
  d.in0_off[1] = take(d.ly[0].pitch);
  d.ly[0].in_off = d.in0_off[0];
  for (int l = 1; l < H; l++) d.ly[l].in_off = take(d.ly[l].pitch);
  int maxr = 1, pb = 1;
  for (int l = 0; l < H; l++) {
    d.ly[l].t_off = take(d.ly[l].R);
    if (d.ly[l].R > maxr) maxr = d.ly[l].R;
    const int G = 1 << d.ly[l].gs;  // column-partial staging: layers with a backward pass
    if (l >= 1 && !((regmask >> l) & 1u) && G > 1 && G * d.ly[l].pitch > pb)
      pb = G * d.ly[l].pitch;
  }
  d.yown_off = take(H > 0 ? d.ly[H - 1].R : 1);
  for (int b = 0; b < 2; b++) {
    d.delta_off[b] = take(maxr);
    d.dsc_off[b] = take(maxr);
  }
  d.red_off = take(2 * kWarps * 32);  // two: consecutive forward layers alternate
  d.pbuf_off = take(pb);
  d.out_off = take(4 * kMaxOut);
  LayerDev& lo = d.ly[L - 1];
  lo.res = 1;
  lo.wsm_off = take(lo.fo * (lo.R + 1));
  for (int l = 0; l < H; l++) {
    d.ly[l].res = ((regmask >> l) & 1u) ? kResReg : ((mask >> l) & 1u) ? kResSmem : kResL2;
    d.ly[l].wsm_off = d.ly[l].res == kResSmem ? take(d.ly[l].R * d.ly[l].pitch)
                      : d.ly[l].res == kResReg ? take(reg_tail_floats) : 0;
  }
  return off * (int)sizeof(float);
}

static long long resident_floats(const NetDev& d, unsigned mask) {
  long long f = 0;
  for (int l = 0; l < d.L - 1; l++)
    if ((mask >> l) & 1u) f += (long long)d.ly[l].R * d.ly[l].pitch;
  return f;
}

// Thread mapping of a hidden layer's row block (LayerDev): the row-group
// count G = 2^gs minimising the serial steps ceil(R/G) * ceil(quads/(512/G))
// (plus reduction chunks), and the reduction chunk CH >= rows per group
// (capped at 16: chunks beyond).
static void choose_mapping(LayerDev& ly, bool stages, int force_gs) {
  const int nq = ly.pitch / 4;
  int best = 1 << 30;
  for (int gs = 0; (1 << gs) <= kWarps; gs++) {
    const int G = 1 << gs, TG = kThreads / G;
    const int C = (nq + TG - 1) / TG, nj = (ly.R + G - 1) / G;
    // G > 1 stages G partial vectors in smem for the backward pass: only for
    // narrow layers, where the staging costs little shared memory (layer 0
    // has no backward pass and stages nothing)
    if (stages && G > 1 && G * ly.pitch > 2048) break;
    // without that limit (layer 0) the count model would trade rows for
    // quads down to one row per 32-thread group (C3: gs = 4, -4.8%): keep
    // one quad per thread
    if (!stages && G > 1 && C > 1) break;
    // G > 1 also costs a duplicated input gather and (backward) a staged
    // combine of the partials: only worth it for a clear win (layer 0 has
    // neither: C5's layer 0 with G = 2 instead of 1 is +0.8%, scripts/gs_ab.sh)
    const int cost = C * nj + (stages && G > 1 ? 4 : 0) + 8 * ((nj + 15) / 16 - 1);
    if (cost < best) {
      best = cost;
      ly.gs = gs;
    }
  }
  if (force_gs >= 0 && (1 << force_gs) <= kWarps) ly.gs = force_gs;
  const int nj = (ly.R + (1 << ly.gs) - 1) >> ly.gs;
  ly.CH = nj <= 4 ? 4 : nj <= 8 ? 8 : 16;
}

// Row blocks, thread mappings and exchange-buffer offsets for nct CTAs.
static void set_geometry(dmlp_net* net, int nct, size_t* yoff, size_t* poff, int rround = 1) {
  NetDev& d = net->dev;
  const int H = d.L - 1;
  d.nct = nct;
  // exchange buffers (line-aligned per producer): y words [2][P][1<<ylog] for
  // hidden layers but the last, output partials [2][P][1<<ylog], column
  // partial words [2][P][pstride] for hidden layers l >= 1
  size_t ll = 0;
  for (int l = 0; l < H; l++) {
    LayerDev& ly = d.ly[l];
    ly.R = own_max_rows(ly.fo, nct);
    if (rround > 1) ly.R = (ly.R + rround - 1) / rround * rround;
    ly.P = (ly.fo + ly.R - 1) / ly.R;
    ly.ylog = ceil_log2(ly.R < 16 ? 16 : ly.R);
    // flat y words: a consumer's quad is then always one 32-byte pair of
    // vector polls (per-producer slots only give that when R % 4 == 0)
    ly.yflat = (ly.R & 3) != 0;
    if (const char* yf = knob("DMLP_YFLAT")) ly.yflat = atoi(yf) == 2 ? 1 : atoi(yf) == 0 ? 0 : ly.yflat;
    ly.pstride = round_up(ly.fi, 16);
    int force_gs = -1;  // experiments: DMLP_GS="gs0,gs1,..." per hidden layer, -1 = auto
    if (const char* g = knob("DMLP_GS")) {
      for (int i = 0; i < l && g; i++) g = strchr(g, ',') ? strchr(g, ',') + 1 : nullptr;
      if (g) force_gs = atoi(g);
    }
    choose_mapping(ly, l >= 1, force_gs);
    yoff[l] = ll;
    if (l < H - 1) ll += 2 * (size_t)ly.P << ly.ylog;
    if (l >= 1) {
      poff[l] = ll;
      ll += 2 * (size_t)ly.P * ly.pstride;
    }
  }
  {
    LayerDev& lo = d.ly[d.L - 1];
    lo.R = H > 0 ? d.ly[H - 1].R : lo.fi;  // owned input columns per CTA
    lo.P = H > 0 ? d.ly[H - 1].P : 1;
    lo.ylog = ceil_log2(lo.fo < 16 ? 16 : lo.fo);
    lo.yflat = 0;
    lo.gs = 0;
    lo.CH = 1;
    lo.pstride = 0;
    yoff[d.L - 1] = ll;
    ll += 2 * (size_t)lo.P << lo.ylog;
  }
  net->ll_words = ll;

}

// DMLP_RES_AUTO: keep the most weight bytes on chip.  For every compiled
// register plan, put its row blocks on the largest layers that fit them, then
// pick the best shared-memory subset of the rest; ties go to the simpler
// plan.  Sets the plan on net; returns the fraction of the CTA's weight
// floats kept on chip (1.0: every hidden layer).
static double auto_plan(dmlp_net* net, bool noreg, int smem_cap, unsigned all) {
  NetDev& d = net->dev;
  const int H = d.L - 1;
  unsigned mask = 0;
  net->train_fn = nullptr;
  net->reg_mask = 0;
  net->reg_tail = 0;
  long long best = -1;
  const TrainVariant* vars = nullptr;
  const int nv = train_variants(&vars);
  for (int vi = 0; vi < nv; vi++) {
    const TrainVariant& tv = vars[vi];
    if (noreg && tv.n_reg > 0) continue;
    if (const char* fv = knob("DMLP_FORCE_VARIANT"))  // experiments: only plan `fv`
      if (atoi(fv) != vi) continue;
    unsigned regmask = 0;
    long long regf = 0;
    for (int i = 0; i < tv.n_reg; i++) {  // greedy: largest fitting layer not yet taken
      int pick = -1;
      long long pf = 0;
      for (int l = 0; l < H; l++) {
        const LayerDev& ly = d.ly[l];
        if (((regmask >> l) & 1u) || ly.R > tv.rr || ly.pitch > kThreads * (tv.rc + tv.rs))
          continue;
        const long long f = (long long)ly.R * ly.pitch;
        if (f > pf) { pf = f; pick = l; }
      }
      if (pick < 0) break;
      regmask |= 1u << pick;
      regf += pf;
    }
    if (tv.n_reg > 0 && regmask == 0) continue;
    unsigned excl = 0;  // experiments: hidden layers kept out of shared memory
    if (const char* ex = knob("DMLP_SMEM_EXCLUDE")) excl = (unsigned)atoi(ex);
    for (unsigned m = 0; m <= all; m++) {
      if (m & (regmask | excl)) continue;
      if (layout_smem(net, m, regmask, tv.rr * tv.rs * kThreads) > smem_cap) continue;
      const long long f = resident_floats(d, m) + regf;
      // ties go to the simpler plan, except that a plan holding every hidden
      // layer in registers beats shared memory (C1: +5%; CTA-count sweep)
      if (f > best || (f == best && regmask == all && net->reg_mask != all)) {
        best = f;
        mask = m;
        net->reg_mask = regmask;
        net->variant = vi;
        net->train_fn = tv.fn[3];
        net->reg_tail = tv.rr * tv.rs * kThreads;
        for (int k = 0; k < kMaxRegLayers; k++) d.reg_layer[k] = -1;
        int k = 0;
        for (int l = 0; l < H; l++)
          if ((regmask >> l) & 1u) d.reg_layer[k++] = l;
      }
    }
  }
  net->resident_mask = mask;
  long long tot = 0;
  for (int l = 0; l < H; l++) tot += (long long)d.ly[l].R * d.ly[l].pitch;
  const unsigned onchip = mask | net->reg_mask;
  if (onchip == all) return 1.0;
  return tot > 0 ? (double)(best > 0 ? best : 0) / (double)tot : 1.0;
}

}  // namespace dmlp

using namespace dmlp;

extern "C" {

const char* dmlp_last_error(void) { return g_err.c_str(); }

int dmlp_device_info(int device, int32_t* n_sms, int32_t* smem_per_block, int64_t* l2_bytes,
                     int64_t* persisting_l2_max) {
  cudaDeviceProp p;
  DMLP_CUDA(cudaGetDeviceProperties(&p, device));
  if (n_sms) *n_sms = p.multiProcessorCount;
  if (smem_per_block) *smem_per_block = (int32_t)p.sharedMemPerBlockOptin;
  if (l2_bytes) *l2_bytes = p.l2CacheSize;
  if (persisting_l2_max) *persisting_l2_max = p.persistingL2CacheMaxSize;
  return DMLP_OK;
}

int dmlp_net_create(int device, const int32_t* sizes, int32_t n_sizes, int32_t residency,
                    int32_t n_ctas, dmlp_net** out) {
  if (!out || !sizes) return set_error(DMLP_EINVAL, "null argument");
  *out = nullptr;
  if (n_sizes < 2) return set_error(DMLP_EINVAL, "architecture needs at least input and output sizes");
  if (n_sizes - 1 > kMaxLayers)
    return set_error(DMLP_EINVAL, "at most %d weight layers supported, got %d", kMaxLayers,
                     n_sizes - 1);
  for (int i = 0; i < n_sizes; i++)
    if (sizes[i] < 1) return set_error(DMLP_EINVAL, "layer sizes must be positive");
  if (sizes[n_sizes - 1] > kMaxOut)
    return set_error(DMLP_EINVAL, "output layer wider than %d is not supported", kMaxOut);
  const bool noreg = (residency & DMLP_RES_NOREG) != 0;
  const bool allpaths = (residency & DMLP_RES_ALLPATHS) != 0;
  residency &= ~(DMLP_RES_NOREG | DMLP_RES_ALLPATHS);
  if ((residency < DMLP_RES_AUTO || residency > DMLP_RES_SMEM) && !(residency & DMLP_RES_MASK))
    return set_error(DMLP_EINVAL, "unknown residency %d", residency);
  DeviceGuard dg(device);
  DMLP_CUDA(dg.err);
  cudaDeviceProp prop;
  DMLP_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    return set_error(DMLP_ECUDA, "device %d is sm_%d%d; libdmlp is built for sm_100a", device,
                     prop.major, prop.minor);

  dmlp_net* net = new dmlp_net();
  net->device = device;
  net->n_sizes = n_sizes;
  memcpy(net->sizes, sizes, sizeof(int32_t) * n_sizes);
  NetDev& d = net->dev;
  d.L = n_sizes - 1;
  int nct = n_ctas > 0 ? n_ctas : prop.multiProcessorCount;
  if (nct > prop.multiProcessorCount) nct = prop.multiProcessorCount;
  if (d.L == 1) nct = 1;  // no hidden layer: nothing to distribute
  d.nct = nct;
  const int H = d.L - 1;

  size_t woff = 0;
  for (int l = 0; l < d.L; l++) {
    HostLayer& h = net->hl[l];
    h.fi = sizes[l];
    h.fo = sizes[l + 1];
    h.pitch = round_up(h.fi + 1, 4);
    h.w_off = woff;
    woff += (size_t)h.fo * h.pitch;
    d.ly[l].fi = h.fi;
    d.ly[l].fo = h.fo;
    d.ly[l].pitch = h.pitch;
  }
  net->w_floats = woff;

  size_t yoff[kMaxLayers], poff[kMaxLayers];
  set_geometry(net, nct, yoff, poff);

  // residency: choose which layers keep their rows in shared memory
  const int smem_cap = (int)prop.sharedMemPerBlockOptin - 1024;  // keep room for static smem
  const unsigned all = (1u << H) - 1u;  // hidden layers (the output tile is always resident)
  unsigned mask = 0;
  if (residency & DMLP_RES_MASK) {
    mask = (unsigned)residency & all;
    if (layout_smem(net, mask) > smem_cap) {
      const int need = layout_smem(net, mask);
      delete net;
      return set_error(DMLP_EINVAL, "resident-layer mask needs %d bytes of smem (> %d)", need,
                       smem_cap);
    }
  } else if (residency == DMLP_RES_SMEM) {
    mask = all;
    if (layout_smem(net, mask) > smem_cap) {
      const int need = layout_smem(net, mask);
      delete net;
      return set_error(DMLP_EINVAL,
                       "net does not fit in shared memory: %d bytes per CTA needed, %d available",
                       need, smem_cap);
    }
  } else if (residency == DMLP_RES_AUTO) {
    // Grid and row blocks (CTA-count and rounding sweeps):
    //  1. 128 (then 136) CTAs when every weight fits on chip with that many:
    //     fewer producers per exchange (C1-C3: 6-10% faster than 148);
    //  2. else all SMs with rows per CTA rounded up to a multiple of 4
    //     (producer blocks polled as 16-byte vectors, fewer producers) when
    //     >= 90% of the weights stay on chip (C5: +4.4%);
    //  3. else all SMs, rows per CTA = ceil(fo / SMs), for capacity (C4).
    bool chosen = false;
    if (n_ctas <= 0 && H > 0) {
      for (int cand : {128, 136}) {
        if (cand > prop.multiProcessorCount) continue;
        set_geometry(net, cand, yoff, poff);
        if (auto_plan(net, noreg, smem_cap, all) >= 1.0) {  // fully on chip
          chosen = true;
          break;
        }
      }
    }
    if (!chosen && H > 0) {
      set_geometry(net, nct, yoff, poff, 4);
      chosen = auto_plan(net, noreg, smem_cap, all) >= 0.9;
    }
    if (!chosen) set_geometry(net, nct, yoff, poff);
    auto_plan(net, noreg, smem_cap, all);
    mask = net->resident_mask;
  }
  if (!net->train_fn) {
    const TrainVariant* vars = nullptr;
    train_variants(&vars);
    net->variant = 0;
    net->train_fn = vars[0].fn[3];
    for (int k = 0; k < kMaxRegLayers; k++) d.reg_layer[k] = -1;
  }
  if (layout_smem(net, 0) > smem_cap) {
    const int need = layout_smem(net, 0);
    delete net;
    return set_error(DMLP_EINVAL, "activation vectors need %d bytes of shared memory (> %d)",
                     need, smem_cap);
  }
  const unsigned onchip = mask | net->reg_mask;
  net->residency =
      onchip == all ? DMLP_RES_SMEM : (onchip == 0 ? DMLP_RES_L2 : DMLP_RES_HYBRID);
  net->smem_bytes = layout_smem(net, mask, net->reg_mask, net->reg_tail);
  net->resident_mask = mask;
  {  // the instance compiled with just the residency paths this plan uses
    const TrainVariant* vars = nullptr;
    train_variants(&vars);
    int feat = 0;
    for (int l = 0; l < H; l++)
      feat |= d.ly[l].res == kResSmem ? kFeatSmem : d.ly[l].res == kResL2 ? kFeatL2 : 0;
    // L1 for the one streamed layer l >= 1 (layer 0 resident, <= 8 rows per
    // thread, its first kL1Rows rows per thread within kL1Budget)
    int streamed = 0, l1ok = H > 0 && d.ly[0].res != kResL2;
    for (int l = 1; l < H; l++) {
      const LayerDev& ly = d.ly[l];
      if (ly.res != kResL2) continue;
      const int nj = (ly.R + (1 << ly.gs) - 1) >> ly.gs;
      streamed++;
      l1ok = l1ok && nj <= 8 && nj >= kL1Rows &&
             kL1Rows * (1 << ly.gs) * ly.pitch * (int)sizeof(float) <= kL1Budget;
    }
    if (streamed == 1 && l1ok) feat |= kFeatL1;
    if (allpaths) feat = kFeatSmem | kFeatL2;  // sanitizer runs: every residency path
    net->feat = feat;
    net->train_fn = train_instance(vars[net->variant], feat);
    net->train_fn_prof = vars[net->variant].fn_prof;
  }

  int rc = DMLP_OK;
  auto fail = [&](int code) {
    dmlp_net_destroy(net);
    return code;
  };
  if ((rc = cuda_check(set_train_attributes(net->train_fn, net->smem_bytes),
                       "cudaFuncSetAttribute")) ||
      (rc = cuda_check(set_train_attributes(net->train_fn_prof, net->smem_bytes),
                       "cudaFuncSetAttribute")))
    return fail(rc);
  int bps = 0;
  if ((rc = cuda_check(train_occupancy(net->train_fn, net->smem_bytes, &bps), "occupancy")))
    return fail(rc);
  if (bps < 1)
    return fail(set_error(DMLP_ECUDA, "persistent kernel cannot be resident (%d smem bytes)",
                          net->smem_bytes));

  if ((rc = cuda_check(cudaMalloc(&net->d_w, net->w_floats * sizeof(float)), "cudaMalloc weights")))
    return fail(rc);
  if ((rc = cuda_check(cudaMemset(net->d_w, 0, net->w_floats * sizeof(float)), "memset")))
    return fail(rc);
  if (const size_t ll = net->ll_words) {
    if ((rc = cuda_check(cudaMalloc(&net->d_ll, ll * 8), "cudaMalloc exchange"))) return fail(rc);
    if ((rc = cuda_check(cudaMemset(net->d_ll, 0, ll * 8), "memset"))) return fail(rc);
  }
  if ((rc = cuda_check(cudaMalloc(&net->d_err, sizeof(int)), "cudaMalloc"))) return fail(rc);
  if ((rc = cuda_check(cudaMemset(net->d_err, 0, sizeof(int)), "memset"))) return fail(rc);
  const int fi0 = sizes[0];
  if ((rc = cuda_check(cudaMalloc(&net->d_stage, (fi0 + 64) * sizeof(float)), "cudaMalloc")))
    return fail(rc);
  if ((rc = cuda_check(cudaMalloc(&net->d_stage_lab, 64), "cudaMalloc"))) return fail(rc);
  if ((rc = cuda_check(cudaMalloc(&net->d_stage_wrong, 64), "cudaMalloc"))) return fail(rc);
  if ((rc = cuda_check(cudaEventCreateWithFlags(&net->done, cudaEventDisableTiming),
                       "cudaEventCreate")))
    return fail(rc);
  if ((rc = cuda_check(cudaStreamCreateWithFlags(&net->stream, cudaStreamNonBlocking),
                       "cudaStreamCreate")))
    return fail(rc);
  for (int l = 0; l < d.L; l++) {
    d.ly[l].w = net->d_w + net->hl[l].w_off;
    d.ly[l].yll = (l < H - 1 || l == d.L - 1) ? net->d_ll + yoff[l] : nullptr;
    d.ly[l].pll = (l >= 1 && l < H) ? net->d_ll + poff[l] : nullptr;
  }
  d.err = net->d_err;
  d.prof = nullptr;
  d.trace = nullptr;
  d.trace_sample = -1;
  *out = net;
  return DMLP_OK;
}

int dmlp_net_destroy(dmlp_net* net) {
  if (!net) return DMLP_OK;
  DeviceGuard dg(net->device);
  cudaDeviceSynchronize();
  cudaFree(net->d_w);
  cudaFree(net->d_ll);
  cudaFree(net->d_err);
  cudaFree(net->d_stage);
  cudaFree(net->d_stage_lab);
  cudaFree(net->d_stage_wrong);
  cudaFree(net->d_act[0]);
  cudaFree(net->d_act[1]);
  cudaFree(net->d_act[2]);
  cudaFree(net->dev.prof);
  cudaFree(net->dev.trace);
  if (net->stream) cudaStreamDestroy(net->stream);
  if (net->done) cudaEventDestroy(net->done);
  delete net;
  return DMLP_OK;
}

int dmlp_net_info(dmlp_net* net, int32_t* residency, int32_t* n_ctas, int32_t* threads,
                  int32_t* smem_bytes) {
  if (!net) return set_error(DMLP_EINVAL, "null net");
  if (residency) *residency = net->residency;
  if (n_ctas) *n_ctas = net->dev.nct;
  if (threads) *threads = kThreads;
  if (smem_bytes) *smem_bytes = net->smem_bytes;
  return DMLP_OK;
}

int dmlp_net_layer_residency(dmlp_net* net, int32_t* where) {
  if (!net || !where) return set_error(DMLP_EINVAL, "null argument");
  for (int l = 0; l < net->dev.L; l++)
    where[l] = (l == net->dev.L - 1) ? kResSmem : net->dev.ly[l].res;
  return DMLP_OK;
}

int dmlp_net_layer_regcols(dmlp_net* net, int32_t* reg_cols, int32_t* tail_cols) {
  if (!net || !reg_cols || !tail_cols) return set_error(DMLP_EINVAL, "null argument");
  const TrainVariant* vars = nullptr;
  train_variants(&vars);
  const TrainVariant& tv = vars[net->variant];
  for (int l = 0; l < net->dev.L; l++) {
    const LayerDev& ly = net->dev.ly[l];
    const bool reg = l < net->dev.L - 1 && ly.res == kResReg;
    const int fi1 = ly.fi + 1;
    reg_cols[l] = reg ? min(fi1, kThreads * tv.rc) : 0;
    tail_cols[l] = reg ? min(fi1, kThreads * (tv.rc + tv.rs)) - reg_cols[l] : 0;
  }
  return DMLP_OK;
}

int dmlp_net_layer_l1rows(dmlp_net* net, int32_t* rows) {
  if (!net || !rows) return set_error(DMLP_EINVAL, "null argument");
  const int H = net->dev.L - 1;
  for (int l = 0; l < net->dev.L; l++) {
    const LayerDev& ly = net->dev.ly[l];
    rows[l] = ((net->feat & kFeatL1) && l >= 1 && l < H && ly.res == kResL2)
                  ? min(kL1Rows << ly.gs, ly.R) : 0;
  }
  return DMLP_OK;
}

int dmlp_net_profile(dmlp_net* net, int32_t enable) {
  if (!net) return set_error(DMLP_EINVAL, "null net");
  DeviceGuard dg(net->device);
  DMLP_CUDA(dg.err);
  DMLP_CUDA(cudaStreamSynchronize(net->stream));
  if (enable && !net->dev.prof) {
    unsigned long long* p = nullptr;
    DMLP_CUDA(cudaMalloc(&p, kProfWords * sizeof(unsigned long long) * net->dev.nct));
    DMLP_CUDA(cudaMemset(p, 0, kProfWords * sizeof(unsigned long long) * net->dev.nct));
    net->dev.prof = p;
  } else if (!enable && net->dev.prof) {
    DMLP_CUDA(cudaDeviceSynchronize());
    cudaFree(net->dev.prof);
    net->dev.prof = nullptr;
  }
  return DMLP_OK;
}

int dmlp_net_trace(dmlp_net* net, int64_t sample, uint64_t* marks /* [n_ctas][64] or NULL */) {
  if (!net) return set_error(DMLP_EINVAL, "null net");
  DeviceGuard dg(net->device);
  DMLP_CUDA(dg.err);
  DMLP_CUDA(cudaDeviceSynchronize());
  const size_t bytes = (size_t)net->dev.nct * 64 * sizeof(unsigned long long);
  if (marks && net->dev.trace) {  // read back the previous launch's marks
    DMLP_CUDA(cudaMemcpy(marks, net->dev.trace, bytes, cudaMemcpyDeviceToHost));
  }
  if (sample >= 0) {
    if (!net->dev.trace) DMLP_CUDA(cudaMalloc(&net->dev.trace, bytes));
    DMLP_CUDA(cudaMemset(net->dev.trace, 0, bytes));
    net->dev.trace_sample = sample;
  } else if (net->dev.trace) {
    cudaFree(net->dev.trace);
    net->dev.trace = nullptr;
  }
  return DMLP_OK;
}

int dmlp_net_read_profile_all(dmlp_net* net, int64_t* slots, int32_t n_slots) {
  if (!net || !slots) return set_error(DMLP_EINVAL, "null argument");
  if (!net->dev.prof) return set_error(DMLP_EINVAL, "profiling is not enabled");
  DeviceGuard dg(net->device);
  DMLP_CUDA(dg.err);
  DMLP_CUDA(cudaDeviceSynchronize());
  const int n = kProfWords * net->dev.nct;
  unsigned long long* h = new unsigned long long[n];
  cudaError_t e = cudaMemcpy(h, net->dev.prof, n * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    delete[] h;
    return cuda_check(e, "cudaMemcpy profile");
  }
  for (int k = 0; k < n_slots; k++) {
    long long a = 0;
    if (k < kProfWords)
      for (int c = 0; c < net->dev.nct; c++) a += (long long)h[kProfWords * c + k];
    slots[k] = a;
  }
  delete[] h;
  DMLP_CUDA(cudaMemset(net->dev.prof, 0, n * sizeof(unsigned long long)));
  return DMLP_OK;
}

int dmlp_net_read_profile_cta(dmlp_net* net, int64_t* slots) {
  if (!net || !slots) return set_error(DMLP_EINVAL, "null argument");
  if (!net->dev.prof) return set_error(DMLP_EINVAL, "profiling is not enabled");
  DeviceGuard dg(net->device);
  DMLP_CUDA(dg.err);
  DMLP_CUDA(cudaDeviceSynchronize());
  const int n = kProfWords * net->dev.nct;
  DMLP_CUDA(cudaMemcpy(slots, net->dev.prof, n * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost));
  DMLP_CUDA(cudaMemset(net->dev.prof, 0, n * sizeof(unsigned long long)));
  return DMLP_OK;
}

int dmlp_net_read_profile(dmlp_net* net, int64_t* slots) {
  return dmlp_net_read_profile_all(net, slots, kProfPhases);
}

int dmlp_net_set_layer(dmlp_net* net, int32_t layer, const float* w, int64_t n) {
  if (!net || !w) return set_error(DMLP_EINVAL, "null argument");
  if (layer < 0 || layer >= net->dev.L) return set_error(DMLP_EINVAL, "layer %d out of range", layer);
  const HostLayer& h = net->hl[layer];
  if (n != (int64_t)h.fo * (h.fi + 1))
    return set_error(DMLP_ESIZE, "layer %d holds %lld weights, got %lld", layer,
                     (long long)h.fo * (h.fi + 1), (long long)n);
  DeviceGuard dg(net->device);
  DMLP_CUDA(dg.err);
  float* tmp = nullptr;
  DMLP_CUDA(cudaStreamWaitEvent(net->stream, net->done, 0));
  DMLP_CUDA(cudaMallocAsync(&tmp, n * sizeof(float), net->stream));
  DMLP_CUDA(cudaMemcpyAsync(tmp, w, n * sizeof(float), cudaMemcpyDefault, net->stream));
  k_pack<<<296, 256, 0, net->stream>>>(tmp, net->d_w + h.w_off, h.fo, h.fi, h.pitch);
  DMLP_CUDA(cudaGetLastError());
  DMLP_CUDA(cudaFreeAsync(tmp, net->stream));
  DMLP_CUDA(cudaEventRecord(net->done, net->stream));
  DMLP_CUDA(cudaStreamSynchronize(net->stream));
  return DMLP_OK;
}

int dmlp_net_get_layer(dmlp_net* net, int32_t layer, float* w, int64_t n) {
  if (!net || !w) return set_error(DMLP_EINVAL, "null argument");
  if (layer < 0 || layer >= net->dev.L) return set_error(DMLP_EINVAL, "layer %d out of range", layer);
  const HostLayer& h = net->hl[layer];
  if (n != (int64_t)h.fo * (h.fi + 1))
    return set_error(DMLP_ESIZE, "layer %d holds %lld weights, got %lld", layer,
                     (long long)h.fo * (h.fi + 1), (long long)n);
  DeviceGuard dg(net->device);
  DMLP_CUDA(dg.err);
  float* tmp = nullptr;
  DMLP_CUDA(cudaStreamWaitEvent(net->stream, net->done, 0));
  DMLP_CUDA(cudaMallocAsync(&tmp, n * sizeof(float), net->stream));
  k_unpack<<<296, 256, 0, net->stream>>>(net->d_w + h.w_off, tmp, h.fo, h.fi, h.pitch);
  DMLP_CUDA(cudaGetLastError());
  DMLP_CUDA(cudaMemcpyAsync(w, tmp, n * sizeof(float), cudaMemcpyDefault, net->stream));
  DMLP_CUDA(cudaFreeAsync(tmp, net->stream));
  DMLP_CUDA(cudaEventRecord(net->done, net->stream));
  DMLP_CUDA(cudaStreamSynchronize(net->stream));
  return DMLP_OK;
}

static int check_kernel_error(dmlp_net* net, cudaError_t e) {
  if (e != cudaSuccess) {
    int flag = 0;
    cudaMemcpy(&flag, net->d_err, sizeof(int), cudaMemcpyDeviceToHost);
    return set_error(DMLP_ECUDA, "training kernel failed: %s%s", cudaGetErrorString(e),
                     flag ? " (exchange wait timed out)" : "");
  }
  return DMLP_OK;
}

static int run_epoch(dmlp_net* net, const float* x, long long ldx, const uint8_t* labels,
                     const int32_t* order, long long n, float eta, long long* wrong, float* y_last,
                     uint8_t* pred, cudaStream_t st) {
  if (n <= 0) return DMLP_OK;
  if (n > 0x7FFFFFFFLL) return set_error(DMLP_EINVAL, "at most 2^31-1 samples per launch");
  if (!(eta >= 0.0f)) return set_error(DMLP_EINVAL, "eta must be non-negative");
  if (ldx < net->sizes[0]) return set_error(DMLP_ESIZE, "row stride %lld < fan-in %d", ldx,
                                            net->sizes[0]);
  if ((unsigned long long)net->seq + (unsigned long long)n >= 0xFFFFFFF0ull) {
    // flag wrap-around: clear the exchange words and restart the sequence
    DMLP_CUDA(cudaStreamSynchronize(st));
    if (net->d_ll) DMLP_CUDA(cudaMemset(net->d_ll, 0, net->ll_words * 8));
    DMLP_CUDA(cudaDeviceSynchronize());
    net->seq = 1;
  }
  const uint32_t seq0 = net->seq;
  if (int rc = net_begin(net, st)) return rc;
  cudaError_t e = launch_train(net, x, ldx, labels, order, n, eta, seq0, wrong, y_last, pred, st);
  if (e != cudaSuccess) return check_kernel_error(net, e);
  if (int rc = net_end(net, st)) return rc;
  net->seq += (uint32_t)n;
  return DMLP_OK;
}

int dmlp_train_step(dmlp_net* net, const float* x, int32_t digit, float eta, float* y_out) {
  if (!net || !x) return set_error(DMLP_EINVAL, "null argument");
  const int nout = net->sizes[net->n_sizes - 1];
  if (digit < 0 || digit >= nout) return set_error(DMLP_EINVAL, "digit %d out of range", digit);
  DeviceGuard dg(net->device);
  DMLP_CUDA(dg.err);
  const int fi0 = net->sizes[0];
  uint8_t lab = (uint8_t)digit;
  DMLP_CUDA(cudaStreamWaitEvent(net->stream, net->done, 0));
  DMLP_CUDA(cudaMemcpyAsync(net->d_stage, x, fi0 * sizeof(float), cudaMemcpyDefault, net->stream));
  DMLP_CUDA(cudaMemcpyAsync(net->d_stage_lab, &lab, 1, cudaMemcpyHostToDevice, net->stream));
  float* ydev = net->d_stage + round_up(fi0, 32);
  int rc = run_epoch(net, net->d_stage, fi0, net->d_stage_lab, nullptr, 1, eta, nullptr, ydev,
                     nullptr, net->stream);
  if (rc) return rc;
  if (y_out)
    DMLP_CUDA(cudaMemcpyAsync(y_out, ydev, nout * sizeof(float), cudaMemcpyDefault, net->stream));
  return check_kernel_error(net, cudaStreamSynchronize(net->stream));
}

int dmlp_train_epoch(dmlp_net* net, const float* x_dev, int64_t ldx, const uint8_t* labels_dev,
                     const int32_t* order_dev, int64_t n, float eta, int64_t* wrong_dev,
                     float* y_last_dev, uint8_t* pred_dev, void* stream) {
  if (!net || (!x_dev && n > 0) || (!labels_dev && n > 0))
    return set_error(DMLP_EINVAL, "null argument");
  DeviceGuard dg(net->device);
  DMLP_CUDA(dg.err);
  return run_epoch(net, x_dev, ldx, labels_dev, order_dev, n, eta, (long long*)wrong_dev,
                   y_last_dev, pred_dev, (cudaStream_t)stream);
}

}  // extern "C"
