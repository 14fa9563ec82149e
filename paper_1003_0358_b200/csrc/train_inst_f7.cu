// train_inst_f7.cu -- instances of the training kernel with feature set 7
// (train_kernel.cuh: bit 0 shared-memory layers, bit 1 L2-streamed layers,
// bit 2 the streamed layer's first rows cached in L1), one translation unit per
// feature set so the build compiles them in parallel.  Profiling launches use
// the feature-set-3 instance.
#include "train_kernel.cuh"

namespace dmlp {

void train_fns_f7(const void** fns, const void** prof) {
  int k = 0;
#define DMLP_INST(n, rr, rc, rs)                                   \
  fns[k] = (const void*)k_train<n, rr, rc, rs, 7, false>;          \
  if (prof) prof[k] = nullptr;                                     \
  k++;
  DMLP_REGISTER_PLANS(DMLP_INST)
#undef DMLP_INST
}

}  // namespace dmlp
