// deform_kernel.cu -- per-image elastic + affine deformation on sm_100a.
//
// Replaces deform.deform_epoch / deform_image (deform.py:203-247), the
// numpy Philox substreams (rng.py:19-38) and upscale_dataset (deform.py:
// 250-257).  One CTA deforms one image at a time (grid-stride over images):
//   1. key = splitmix chain over (seed, 2, epoch, index); the 423 Philox4x64-10
//      blocks the image consumes are generated in parallel (one block per
//      thread) and decoded straight into the draw map of SURVEY App. A.1;
//   2. 28->29 re-centring upscale in float32 (deform.py:87-99);
//   3. 21-tap Gaussian (numpy pairwise-sum normalisation) and two separable
//      zero-padded passes per field in fp64, scipy's symmetric tap order;
//   4. rotation-or-shear with anisotropic scale about the centre pixel,
//      plus the elastic field, then the bilinear warp with -1 background.
// This translation unit is compiled with -fmad=false: the reference never
// fuses multiply-adds, and the fp64 geometry is evaluated in numpy's order.
#include <cuda_runtime.h>

#include "dmlp_internal.h"

namespace dmlp {

constexpr int kGrid = 29;
constexpr int kPix = kGrid * kGrid;          // 841
constexpr int kWords = 2 + 2 * kPix + 5;     // 1689 Philox words per image
constexpr int kBlocks = (kWords + 3) / 4;    // 423
constexpr int kDefThreads = 256;

struct DefP {
  double sig_lo, sig_hi, al_lo, al_hi, beta_def, beta_red, ga_lo, ga_hi;
  int ks;
};

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x = x + 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

__device__ __forceinline__ void philox4x64_10(uint64_t k0, uint64_t k1, uint64_t ctr,
                                              uint64_t out[4]) {
  uint64_t c0 = ctr, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; r++) {
    const uint64_t hi0 = __umul64hi(0xD2E7470EE14C6C93ULL, c0), lo0 = 0xD2E7470EE14C6C93ULL * c0;
    const uint64_t hi1 = __umul64hi(0xCA5A826395121157ULL, c2), lo1 = 0xCA5A826395121157ULL * c2;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

__device__ __forceinline__ double u53(uint64_t w) {
  return (double)(w >> 11) * (1.0 / 9007199254740992.0);
}
__device__ __forceinline__ double uniform(double lo, double hi, double u) {
  return lo + (hi - lo) * u;
}

struct DefSmem {
  double nx[kPix], ny[kPix], tmp[kPix];
  float up[kPix];
  double g[64];
  double u[8];  // sigma-u, alpha-u, mode, angle-u, gamma-u, sx-u, sy-u
  double scal[6];
  uint64_t key[2];
};

// scipy.ndimage.convolve1d, constant mode, symmetric kernel (deform.py:130-131):
// out = x[c]*g(0) + sum_{k=h..1} (x[c-k] + x[c+k]) * g(k).
__device__ __forceinline__ void conv_pass(const double* in, double* out, const double* g, int h,
                                          int axis, double scale) {
  for (int p = threadIdx.x; p < kPix; p += blockDim.x) {
    const int r = p / kGrid, c = p % kGrid;
    const int pos = axis == 0 ? r : c;
    double acc = in[p] * g[h];
    for (int k = h; k >= 1; k--) {
      const int lo = pos - k, hi = pos + k;
      double xl = 0.0, xh = 0.0;
      if (lo >= 0) xl = axis == 0 ? in[lo * kGrid + c] : in[r * kGrid + lo];
      if (hi < kGrid) xh = axis == 0 ? in[hi * kGrid + c] : in[r * kGrid + hi];
      acc = acc + (xl + xh) * g[h + k];
    }
    out[p] = scale == 0.0 ? acc : scale * acc;
  }
}

__device__ __forceinline__ void upscale_img(const uint8_t* img, float* up) {
  for (int p = threadIdx.x; p < kPix; p += blockDim.x) {
    const int r = p / kGrid, c = p % kGrid;
    const int r0 = max(r - 1, 0), r1 = min(r, 27), c0 = max(c - 1, 0), c1 = min(c, 27);
    const float n00 = (float)img[r0 * 28 + c0] / 127.5f - 1.0f;
    const float n01 = (float)img[r0 * 28 + c1] / 127.5f - 1.0f;
    const float n10 = (float)img[r1 * 28 + c0] / 127.5f - 1.0f;
    const float n11 = (float)img[r1 * 28 + c1] / 127.5f - 1.0f;
    up[p] = 0.25f * (((n00 + n01) + n10) + n11);
  }
}

// Full pipeline for one image given the draws in S (noise in nx/ny, scalars in scal).
__device__ void deform_from_draws(DefSmem& S, int ks, float* out) {
  const int tid = threadIdx.x;
  const double sigma = S.scal[0], alpha = S.scal[1];
  const int h = ks / 2;
  if (tid < ks) {
    const double off = (double)tid - (double)h;
    S.g[tid] = exp(-(off * off) / (2.0 * sigma * sigma));
  }
  __syncthreads();
  if (tid == 0) {  // numpy pairwise sum of the taps (n < 128 branch)
    double s;
    if (ks < 8) {
      s = 0.0;
      for (int i = 0; i < ks; i++) s += S.g[i];
    } else {
      double r[8];
      for (int k = 0; k < 8; k++) r[k] = S.g[k];
      int i;
      for (i = 8; i < ks - (ks % 8); i += 8)
        for (int k = 0; k < 8; k++) r[k] += S.g[i + k];
      s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
      for (; i < ks; i++) s += S.g[i];
    }
    S.u[7] = s;
  }
  __syncthreads();
  if (tid < ks) S.g[tid] = S.g[tid] / S.u[7];
  __syncthreads();
  conv_pass(S.nx, S.tmp, S.g, h, 0, 0.0);
  __syncthreads();
  conv_pass(S.tmp, S.nx, S.g, h, 1, 0.0);
  __syncthreads();
  conv_pass(S.ny, S.tmp, S.g, h, 0, 0.0);
  __syncthreads();
  conv_pass(S.tmp, S.ny, S.g, h, 1, 0.0);
  __syncthreads();

  const int mode = (int)S.scal[2];
  const double angle = S.scal[3], sx = S.scal[4], sy = S.scal[5];
  const double rad = angle * (3.141592653589793 / 180.0);  // np.deg2rad
  const double cs = cos(rad), sn = sin(rad), tn = tan(rad);
  const double center = (kGrid - 1) / 2.0;
  for (int p = tid; p < kPix; p += blockDim.x) {
    const int r = p / kGrid, c = p % kGrid;
    const double y = (double)r - center, x = (double)c - center;
    const double xs = sx * x, ys = sy * y;
    double xr, yr;
    if (mode == 0) {
      xr = cs * xs - sn * ys;
      yr = sn * xs + cs * ys;
    } else {
      xr = xs + tn * ys;
      yr = ys;
    }
    const double dx = (xr - x) + alpha * S.nx[p];
    const double dy = (yr - y) + alpha * S.ny[p];
    const double sr = (double)r + dy, sc = (double)c + dx;
    const double flr = floor(sr), flc = floor(sc);
    const long long i0 = (long long)flr, j0 = (long long)flc;
    const double fr = sr - (double)i0, fc = sc - (double)j0;
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const long long ii = i0 + (q >> 1), jj = j0 + (q & 1);
      const bool valid = ii >= 0 && ii < kGrid && jj >= 0 && jj < kGrid;
      v[q] = valid ? (double)S.up[ii * kGrid + jj] : -1.0;
    }
    double o = (1.0 - fr) * (1.0 - fc) * v[0];
    o = o + (1.0 - fr) * fc * v[1];
    o = o + fr * (1.0 - fc) * v[2];
    o = o + fr * fc * v[3];
    o = o < -1.0 ? -1.0 : (o > 1.0 ? 1.0 : o);
    out[p] = (float)o;
  }
}

__global__ void __launch_bounds__(kDefThreads, 4)
    k_deform(const uint8_t* __restrict__ raw, const uint8_t* __restrict__ labels, long long first,
             long long n, unsigned long long seed, unsigned long long epoch, DefP P,
             float* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smraw[];
  DefSmem& S = *reinterpret_cast<DefSmem*>(smraw);
  const int tid = threadIdx.x;
  const int N = kPix;
  for (long long img = blockIdx.x; img < n; img += gridDim.x) {
    if (tid == 0) {
      uint64_t hh = splitmix64(seed);
      hh = splitmix64(hh ^ 2ULL);
      hh = splitmix64(hh ^ epoch);
      hh = splitmix64(hh ^ (uint64_t)(first + img));
      S.key[0] = hh;
      S.key[1] = splitmix64(hh);
    }
    upscale_img(raw + img * 784, S.up);
    __syncthreads();
    const uint64_t k0 = S.key[0], k1 = S.key[1];
    for (int b = tid; b < kBlocks; b += blockDim.x) {
      uint64_t w[4];
      philox4x64_10(k0, k1, (uint64_t)b + 1, w);
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const int wi = 4 * b + e;
        if (wi >= kWords) break;
        if (wi >= 2 && wi < 2 + N) {
          S.nx[wi - 2] = uniform(-1.0, 1.0, u53(w[e]));
        } else if (wi >= 2 + N && wi < 2 + 2 * N) {
          S.ny[wi - 2 - N] = uniform(-1.0, 1.0, u53(w[e]));
        } else if (wi == 2 + 2 * N) {  // integers(0, 2): bit 31 of the low half
          S.u[2] = (double)(((w[e] & 0xFFFFFFFFULL) * 2ULL) >> 32);
        } else {
          const int slot = wi < 2 ? wi : wi - 2 * N;  // 0,1 | 3..6
          S.u[slot] = u53(w[e]);
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      const int digit = labels[img];
      const double beta = (digit == 1 || digit == 7) ? P.beta_red : P.beta_def;
      S.scal[0] = uniform(P.sig_lo, P.sig_hi, S.u[0]);
      S.scal[1] = uniform(P.al_lo, P.al_hi, S.u[1]);
      S.scal[2] = S.u[2];
      S.scal[3] = uniform(-beta, beta, S.u[3]);
      const double gamma = uniform(P.ga_lo, P.ga_hi, S.u[4]);
      S.scal[4] = uniform(1.0 - gamma / 100.0, 1.0 + gamma / 100.0, S.u[5]);
      S.scal[5] = uniform(1.0 - gamma / 100.0, 1.0 + gamma / 100.0, S.u[6]);
    }
    __syncthreads();
    deform_from_draws(S, P.ks, out + img * kPix);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kDefThreads, 4)
    k_deform_injected(const uint8_t* __restrict__ raw, long long n, const double* __restrict__ ndx,
                      const double* __restrict__ ndy, const double* __restrict__ scal, int ks,
                      float* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smraw[];
  DefSmem& S = *reinterpret_cast<DefSmem*>(smraw);
  const int tid = threadIdx.x;
  for (long long img = blockIdx.x; img < n; img += gridDim.x) {
    upscale_img(raw + img * 784, S.up);
    for (int p = tid; p < kPix; p += blockDim.x) {
      S.nx[p] = ndx[img * kPix + p];
      S.ny[p] = ndy[img * kPix + p];
    }
    if (tid < 6) S.scal[tid] = scal[img * 6 + tid];
    __syncthreads();
    deform_from_draws(S, ks, out + img * kPix);
    __syncthreads();
  }
}

__global__ void k_upscale(const uint8_t* __restrict__ raw, long long n, float* __restrict__ out) {
  __shared__ float up[kPix];
  for (long long img = blockIdx.x; img < n; img += gridDim.x) {
    upscale_img(raw + img * 784, up);
    __syncthreads();
    for (int p = threadIdx.x; p < kPix; p += blockDim.x) out[img * kPix + p] = up[p];
    __syncthreads();
  }
}

static int grid_for(long long n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long g = (long long)sms * 8;
  return (int)(n < g ? n : g);
}

static int check_params(const dmlp_deform_params* p) {
  auto bad = [](double lo, double hi) { return !(isfinite(lo) && isfinite(hi)) || lo > hi; };
  if (bad(p->sigma_lo, p->sigma_hi) || bad(p->alpha_lo, p->alpha_hi) ||
      bad(p->gamma_lo, p->gamma_hi))
    return set_error(DMLP_EINVAL, "ranges must be finite (lo, hi) with lo <= hi");
  if (p->sigma_lo <= 0) return set_error(DMLP_EINVAL, "InvalidSigma: sigma must be positive");
  if (p->alpha_lo < 0 || p->gamma_lo < 0)
    return set_error(DMLP_EINVAL, "alpha and gamma ranges must be non-negative");
  if (p->beta_default < 0 || p->beta_reduced < 0)
    return set_error(DMLP_EINVAL, "beta angles must be non-negative");
  if (p->kernel_size < 3 || p->kernel_size % 2 == 0 || p->kernel_size > 63)
    return set_error(DMLP_EINVAL, "EvenSize: kernel_size must be odd, >= 3 and <= 63");
  return DMLP_OK;
}

}  // namespace dmlp

using namespace dmlp;

extern "C" {

int dmlp_deform(const uint8_t* raw_dev, const uint8_t* labels_dev, int64_t first, int64_t n,
                uint64_t seed, uint64_t epoch, const dmlp_deform_params* params, float* out_dev,
                void* stream) {
  if (!params) return set_error(DMLP_EINVAL, "null params");
  int rc = check_params(params);
  if (rc) return rc;
  if (n <= 0) return DMLP_OK;
  if (!raw_dev || !labels_dev || !out_dev) return set_error(DMLP_EINVAL, "null argument");
  DefP P{params->sigma_lo,     params->sigma_hi,     params->alpha_lo, params->alpha_hi,
         params->beta_default, params->beta_reduced, params->gamma_lo, params->gamma_hi,
         params->kernel_size};
  const int smem = (int)sizeof(DefSmem);
  rc = cuda_check(cudaFuncSetAttribute(k_deform, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                  "cudaFuncSetAttribute");
  if (rc) return rc;
  k_deform<<<grid_for(n), kDefThreads, smem, (cudaStream_t)stream>>>(
      raw_dev, labels_dev, first, n, seed, epoch, P, out_dev);
  return cuda_check(cudaGetLastError(), "k_deform");
}

int dmlp_deform_injected(const uint8_t* raw_dev, int64_t n, const double* noise_dx_dev,
                         const double* noise_dy_dev, const double* scalars_dev,
                         int32_t kernel_size, float* out_dev, void* stream) {
  if (kernel_size < 3 || kernel_size % 2 == 0 || kernel_size > 63)
    return set_error(DMLP_EINVAL, "EvenSize: kernel_size must be odd, >= 3 and <= 63");
  if (n <= 0) return DMLP_OK;
  if (!raw_dev || !noise_dx_dev || !noise_dy_dev || !scalars_dev || !out_dev)
    return set_error(DMLP_EINVAL, "null argument");
  const int smem = (int)sizeof(DefSmem);
  int rc = cuda_check(
      cudaFuncSetAttribute(k_deform_injected, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
      "cudaFuncSetAttribute");
  if (rc) return rc;
  k_deform_injected<<<grid_for(n), kDefThreads, smem, (cudaStream_t)stream>>>(
      raw_dev, n, noise_dx_dev, noise_dy_dev, scalars_dev, kernel_size, out_dev);
  return cuda_check(cudaGetLastError(), "k_deform_injected");
}

int dmlp_upscale(const uint8_t* raw_dev, int64_t n, float* out_dev, void* stream) {
  if (n <= 0) return DMLP_OK;
  if (!raw_dev || !out_dev) return set_error(DMLP_EINVAL, "null argument");
  k_upscale<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(raw_dev, n, out_dev);
  return cuda_check(cudaGetLastError(), "k_upscale");
}

}  // extern "C"
