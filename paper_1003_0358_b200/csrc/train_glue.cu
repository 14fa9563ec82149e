// train_glue.cu -- host side of the training kernel: the table of compiled
// instances (register plan x feature set, train_inst_f*.cu), attributes and
// the cooperative launch.
#include <cuda_runtime.h>

#include "dmlp_internal.h"

namespace dmlp {

void train_fns_f0(const void** fns, const void** prof);
void train_fns_f1(const void** fns, const void** prof);
void train_fns_f3(const void** fns, const void** prof);
void train_fns_f7(const void** fns, const void** prof);

int train_variants(const TrainVariant** out) {
  static TrainVariant table[] = {
      {0, 1, 1, 0, {}, nullptr}, {1, 14, 4, 1, {}, nullptr}, {2, 7, 2, 0, {}, nullptr},
      {4, 7, 2, 0, {}, nullptr}, {3, 8, 2, 0, {}, nullptr},
  };
  constexpr int n = sizeof(table) / sizeof(table[0]);
  static bool ready = false;
  if (!ready) {  // one-time, on the first net creation (host side, no CUDA calls)
    const void* f0[n] = {};
    const void* f1[n] = {};
    const void* f3[n] = {};
    const void* f7[n] = {};
    const void* pr[n] = {};
    train_fns_f0(f0, nullptr);
    train_fns_f1(f1, nullptr);
    train_fns_f3(f3, pr);
    train_fns_f7(f7, nullptr);
    for (int k = 0; k < n; k++) {
      table[k].fn[0] = f0[k];
      table[k].fn[1] = f1[k];
      table[k].fn[2] = nullptr;  // L2 without shared memory: the full instance
      table[k].fn[3] = f3[k];
      table[k].fn[7] = f7[k];  // + L1-cached streamed rows
      table[k].fn_prof = pr[k];
    }
    ready = true;
  }
  *out = table;
  return n;
}

const void* train_instance(const TrainVariant& tv, int feat) {
  for (int f = feat; f < 8; f++)  // the smallest compiled superset of the features
    if ((f & feat) == feat && tv.fn[f]) return tv.fn[f];
  return tv.fn[3];
}

cudaError_t set_train_attributes(const void* fn, int smem_bytes) {
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
}

cudaError_t train_occupancy(const void* fn, int smem_bytes, int* blocks_per_sm) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, fn, kThreads, smem_bytes);
}

cudaError_t launch_train(const dmlp_net* net, const float* x, long long ldx,
                         const uint8_t* labels, const int32_t* order, long long n, float eta,
                         uint32_t seq0, long long* wrong, float* y_last, uint8_t* pred,
                         cudaStream_t st) {
  NetDev nd = net->dev;
  unsigned long long* w = reinterpret_cast<unsigned long long*>(wrong);
  void* args[] = {&nd, &x, &ldx, &labels, &order, &n, &eta, &seq0, &w, &y_last, &pred};
  const void* fn = (nd.prof || nd.trace) ? net->train_fn_prof : net->train_fn;
  return cudaLaunchCooperativeKernel(fn, dim3(nd.nct), dim3(kThreads), args,
                                     (size_t)net->smem_bytes, st);
}

}  // namespace dmlp
