// mb_common.cuh -- shared helpers of the exchange microbenchmarks.
//
// gather_y: the CTA-wide "protocol E" slot gather the training kernel used
// before the own-column gather (train_phases.cuh: gather_quads): every warp
// instruction reads one producer's line and every thread keeps all its polls
// in flight.  Kept here as the exchange the xchg*_mb benchmarks time.
#pragma once
#include "train_phases.cuh"

namespace dmlp {

// Gather y of hidden layer `ly` into dst (protocol E).  Producer p's rows sit
// in its own line-aligned slot; each warp instruction reads one producer's
// slot (lane = row within the block, 32-row segments when R > 32) and every
// thread keeps all of its loads in flight, re-polling only the words whose
// flag is not yet this sample's.
__device__ __forceinline__ void gather_y(const unsigned long long* src, const LayerDev& ly,
                                         float* dst, uint32_t seq, int* err) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (ly.R <= 32) {  // one 32-row segment per producer (every BASELINE config): cheap indices
    const int R = ly.R, kmask = (1 << ly.ylog) - 1;
    const bool kv = lane < R;
    const int last = ly.fo - (ly.P - 1) * R;  // rows of the last producer
    for (int pb = 0; pb < ly.P; pb += kWarps * kGatherU) {
      int off[kGatherU];
      unsigned long long v[kGatherU];
#pragma unroll
      for (int u = 0; u < kGatherU; u++) {
        const int p = pb + warp + kWarps * u;
        const bool ok = kv && p < ly.P && (p < ly.P - 1 || lane < last);
        off[u] = ok ? (p << ly.ylog) + lane : -1;
      }
      poll_batch<kGatherU>(src, off, v, seq, err);
#pragma unroll
      for (int u = 0; u < kGatherU; u++)
        if (off[u] >= 0) dst[(off[u] >> ly.ylog) * R + (off[u] & kmask)] =
                             __uint_as_float((uint32_t)v[u]);
    }
    return;
  }
  const int nseg = (ly.R + 31) >> 5, V = ly.P * nseg;
  for (int vb = 0; vb < V; vb += kWarps * kGatherU) {
    int off[kGatherU];
    unsigned long long v[kGatherU];
#pragma unroll
    for (int u = 0; u < kGatherU; u++) {
      const int vi = vb + warp + kWarps * u;
      const int p = nseg == 1 ? vi : vi / nseg;
      const int k = (vi - p * nseg) * 32 + lane;
      const bool ok = vi < V && k < ly.R && p * ly.R + k < ly.fo;
      off[u] = ok ? (p << ly.ylog) + k : -1;
    }
    poll_batch<kGatherU>(src, off, v, seq, err);
    const int kmask = (1 << ly.ylog) - 1;
#pragma unroll
    for (int u = 0; u < kGatherU; u++)  // slot offset -> row: p * R + k
      if (off[u] >= 0)
        dst[(off[u] >> ly.ylog) * ly.R + (off[u] & kmask)] = __uint_as_float((uint32_t)v[u]);
  }
}

}  // namespace dmlp
