// train_inst_f1.cu -- instances of the training kernel with feature set 1
// (train_kernel.cuh: bit 0 shared-memory layers, bit 1 L2-streamed layers),
// one translation unit per feature set so the build compiles them in parallel.
#include "train_kernel.cuh"

namespace dmlp {

namespace {
template <int N, int RR, int RC, int RS>
const void* instance() {
  if constexpr (1 == 0 && N == 0) return nullptr;  // no register block and no features
  else return (const void*)k_train<N, RR, RC, RS, 1, false>;
}
template <int N, int RR, int RC, int RS>
const void* profiling_instance() {
  if constexpr (1 == 3) return (const void*)k_train<N, RR, RC, RS, 3, true>;
  else return nullptr;
}
}  // namespace

void train_fns_f1(const void** fns, const void** prof) {
  int k = 0;
#define DMLP_INST(n, rr, rc, rs)                                 \
  fns[k] = instance<n, rr, rc, rs>();                            \
  if (prof) prof[k] = profiling_instance<n, rr, rc, rs>();       \
  k++;
  DMLP_REGISTER_PLANS(DMLP_INST)
#undef DMLP_INST
}

}  // namespace dmlp
