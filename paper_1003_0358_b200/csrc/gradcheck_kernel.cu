// gradcheck_kernel.cu -- fp64 gradient-check oracle on the GPU (debug aid).
//
// Replaces kernels.backprop_gradients / kernels.gradient_check
// (kernels.py:374-418): the analytic dE/dw of the SSE
// loss with +-1 targets (kernels.py:367-371) through the naive fp64 kernels,
// and central finite differences of the loss for every weight, in fp64
// whatever the model dtype.  For small nets (every layer <= 1024 wide).
//
//  * k_gc_analytic (one CTA): forward (pre-activations and outputs of every
//    layer kept in global scratch), output and hidden deltas, gradients
//    g_ji = -delta_j * y_i, g_j,bias = -delta_j (kernels.py:374-389).
//  * k_gc_fd (one CTA per perturbed forward, two per weight): the forward of
//    the net with one weight moved by +-step.  Layers before the perturbed
//    one are unchanged, so each CTA starts from the stored output of the
//    layer below it.  The loss 0.5*sum((y - t)^2) (kernels.py:367-371).
#include <cuda_runtime.h>

#include <vector>

#include "dmlp_internal.h"

namespace dmlp {

constexpr int kGcMaxWidth = 1024;
constexpr int kGcThreads = 256;
constexpr double kAd = 1.7159, kBd = 0.6666;  // network.py:13-14 as float64

struct GcNet {
  int L;
  int fi[kMaxLayers], fo[kMaxLayers];
  long long woff[kMaxLayers + 1];  // weight offsets (reference layout, bias last)
  long long aoff[kMaxLayers + 1];  // activation offsets (pre / out scratch)
};

__device__ __forceinline__ double act(double a) { return kAd * tanh(kBd * a); }

// Forward of layers [l0, L) from input vector x (length fi[l0]); layer l of
// weight index `pw` (if any) has its weight shifted by `dw`.
__device__ double fwd_loss(const GcNet& g, const double* __restrict__ w, const double* xin,
                           int l0, long long pw, double dw, int digit, double* bufa,
                           double* bufb) {
  const int tid = threadIdx.x;
  for (int i = tid; i < g.fi[l0]; i += blockDim.x) bufa[i] = xin[i];
  __syncthreads();
  double* cur = bufa;
  double* nxt = bufb;
  for (int l = l0; l < g.L; l++) {
    const int fi = g.fi[l], fo = g.fo[l];
    const double* W = w + g.woff[l];
    for (int j = tid; j < fo; j += blockDim.x) {
      const long long row = g.woff[l] + (long long)j * (fi + 1);
      double a = 0.0;
      for (int i = 0; i < fi; i++) {
        double wv = W[(long long)j * (fi + 1) + i];
        if (row + i == pw) wv += dw;
        a += wv * cur[i];
      }
      double b = W[(long long)j * (fi + 1) + fi];
      if (row + fi == pw) b += dw;
      nxt[j] = act(a + b);
    }
    __syncthreads();
    double* t = cur;
    cur = nxt;
    nxt = t;
  }
  __shared__ double red[kGcThreads];
  double e = 0.0;
  for (int k = tid; k < g.fo[g.L - 1]; k += blockDim.x) {
    const double d = cur[k] - (k == digit ? 1.0 : -1.0);
    e += d * d;
  }
  red[tid] = e;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (tid < s) red[tid] += red[tid + s];
    __syncthreads();
  }
  return 0.5 * red[0];
}

__global__ void __launch_bounds__(kGcThreads)
    k_gc_analytic(const GcNet g, const double* __restrict__ w, const double* __restrict__ x,
                  int digit, double* pre, double* out, double* delta, double* grad) {
  const int tid = threadIdx.x;
  for (int l = 0; l < g.L; l++) {  // forward, every layer kept (kernels.py:313-326)
    const int fi = g.fi[l], fo = g.fo[l];
    const double* in = l == 0 ? x : out + g.aoff[l - 1];
    const double* W = w + g.woff[l];
    for (int j = tid; j < fo; j += blockDim.x) {
      double a = 0.0;
      for (int i = 0; i < fi; i++) a += W[(long long)j * (fi + 1) + i] * in[i];
      a += W[(long long)j * (fi + 1) + fi];
      pre[g.aoff[l] + j] = a;
      out[g.aoff[l] + j] = act(a);
    }
    __syncthreads();
  }
  {  // output deltas (kernels.py:229-236) in float64
    const int l = g.L - 1;
    for (int k = tid; k < g.fo[l]; k += blockDim.x) {
      const double th = tanh(kBd * pre[g.aoff[l] + k]);
      const double t = k == digit ? 1.0 : -1.0;
      delta[g.aoff[l] + k] = (t - out[g.aoff[l] + k]) * (kAd * kBd * (1.0 - th * th));
    }
    __syncthreads();
  }
  for (int l = g.L - 1; l >= 1; l--) {  // hidden deltas (kernels.py:239-252)
    const int fi = g.fi[l], fo = g.fo[l];
    const double* W = w + g.woff[l];
    for (int i = tid; i < fi; i += blockDim.x) {
      double acc = 0.0;
      for (int j = 0; j < fo; j++) acc += W[(long long)j * (fi + 1) + i] * delta[g.aoff[l] + j];
      const double th = tanh(kBd * pre[g.aoff[l - 1] + i]);
      delta[g.aoff[l - 1] + i] = acc * (kAd * kBd * (1.0 - th * th));
    }
    __syncthreads();
  }
  for (int l = 0; l < g.L; l++) {  // gradients (kernels.py:382-389)
    const int fi = g.fi[l], fo = g.fo[l];
    const double* in = l == 0 ? x : out + g.aoff[l - 1];
    for (long long e = tid; e < (long long)fo * (fi + 1); e += blockDim.x) {
      const int j = (int)(e / (fi + 1)), i = (int)(e % (fi + 1));
      const double d = delta[g.aoff[l] + j];
      grad[g.woff[l] + e] = i < fi ? -d * in[i] : -d;
    }
  }
}

__global__ void __launch_bounds__(kGcThreads)
    k_gc_fd(const GcNet g, const double* __restrict__ w, const double* __restrict__ x,
            const double* __restrict__ out, int digit, double step, double* loss) {
  __shared__ double bufa[kGcMaxWidth], bufb[kGcMaxWidth];
  const long long p = blockIdx.x;
  const long long wi = p >> 1;
  const double dw = (p & 1) ? -step : step;
  int l = 0;
  while (wi >= g.woff[l + 1]) l++;
  const double* xin = l == 0 ? x : out + g.aoff[l - 1];
  const double e = fwd_loss(g, w, xin, l, wi, dw, digit, bufa, bufb);
  if (threadIdx.x == 0) loss[p] = e;
}

}  // namespace dmlp

using namespace dmlp;

extern "C" int dmlp_gradient_check(const int32_t* sizes, int32_t n_sizes, const double* w_host,
                                   const double* x_host, int32_t digit, double step,
                                   double* grad_bp, double* grad_fd, double* worst) {
  if (!sizes || !w_host || !x_host || !worst) return set_error(DMLP_EINVAL, "null argument");
  if (n_sizes < 2 || n_sizes - 1 > kMaxLayers)
    return set_error(DMLP_EINVAL, "need 1..%d weight layers", kMaxLayers);
  if (!(step > 0.0)) return set_error(DMLP_EINVAL, "step must be positive");
  GcNet g{};
  g.L = n_sizes - 1;
  long long W = 0, A = 0;
  for (int l = 0; l < g.L; l++) {
    g.fi[l] = sizes[l];
    g.fo[l] = sizes[l + 1];
    if (g.fi[l] < 1 || g.fo[l] < 1 || g.fi[l] > kGcMaxWidth || g.fo[l] > kGcMaxWidth)
      return set_error(DMLP_EINVAL, "gradient check supports layers of 1..%d units",
                       kGcMaxWidth);
    g.woff[l] = W;
    g.aoff[l] = A;
    W += (long long)g.fo[l] * (g.fi[l] + 1);
    A += g.fo[l];
  }
  g.woff[g.L] = W;
  g.aoff[g.L] = A;
  if (digit < 0 || digit >= g.fo[g.L - 1]) return set_error(DMLP_EINVAL, "digit out of range");
  double *dw = nullptr, *dx = nullptr, *pre = nullptr, *out = nullptr, *del = nullptr,
         *grad = nullptr, *loss = nullptr;
  auto cleanup = [&]() {
    cudaFree(dw); cudaFree(dx); cudaFree(pre); cudaFree(out); cudaFree(del); cudaFree(grad);
    cudaFree(loss);
  };
  auto fail = [&](cudaError_t e, const char* what) {
    cleanup();
    return cuda_check(e, what);
  };
  cudaError_t e;
  if ((e = cudaMalloc(&dw, W * 8)) || (e = cudaMalloc(&dx, g.fi[0] * 8)) ||
      (e = cudaMalloc(&pre, A * 8)) || (e = cudaMalloc(&out, A * 8)) ||
      (e = cudaMalloc(&del, A * 8)) || (e = cudaMalloc(&grad, W * 8)) ||
      (e = cudaMalloc(&loss, 2 * W * 8)))
    return fail(e, "cudaMalloc");
  if ((e = cudaMemcpy(dw, w_host, W * 8, cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(dx, x_host, g.fi[0] * 8, cudaMemcpyHostToDevice)))
    return fail(e, "cudaMemcpy");
  k_gc_analytic<<<1, kGcThreads>>>(g, dw, dx, digit, pre, out, del, grad);
  if ((e = cudaGetLastError())) return fail(e, "k_gc_analytic");
  k_gc_fd<<<(unsigned)(2 * W), kGcThreads>>>(g, dw, dx, out, digit, step, loss);
  if ((e = cudaGetLastError())) return fail(e, "k_gc_fd");
  std::vector<double> gb(W), lo(2 * W);
  if ((e = cudaMemcpy(gb.data(), grad, W * 8, cudaMemcpyDeviceToHost)) ||
      (e = cudaMemcpy(lo.data(), loss, 2 * W * 8, cudaMemcpyDeviceToHost)))
    return fail(e, "cudaMemcpy");
  cleanup();
  // kernels.py:409-418: max relative error, denominator max(|g_bp|, |g_fd|, 1e-8)
  double wmax = 0.0;
  for (long long k = 0; k < W; k++) {
    const double fd = (lo[2 * k] - lo[2 * k + 1]) / (2.0 * step);
    if (grad_bp) grad_bp[k] = gb[k];
    if (grad_fd) grad_fd[k] = fd;
    double den = fabs(fd) > fabs(gb[k]) ? fabs(fd) : fabs(gb[k]);
    if (den < 1e-8) den = 1e-8;
    const double r = fabs(gb[k] - fd) / den;
    if (r > wmax) wmax = r;
  }
  *worst = wmax;
  return DMLP_OK;
}
