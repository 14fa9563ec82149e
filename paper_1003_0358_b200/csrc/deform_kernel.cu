// deform_kernel.cu -- per-image elastic + affine deformation on sm_100a.
//
// Replaces deform.deform_epoch / deform_image (deform.py:203-247), the
// numpy Philox substreams (rng.py:19-38) and upscale_dataset (deform.py:
// 250-257).  One CTA deforms one image at a time (grid-stride over images):
//   0. a CTA of 256 threads takes kImgs = 4 images at a time, every phase
//      spread over all of them (one barrier per phase for four images);
//   1. key = splitmix chain over (seed, 2, epoch, index); the 423 Philox4x64-10
//      blocks each image consumes are generated in parallel (one block per
//      thread) and decoded straight into the draw map of SURVEY App. A.1;
//   2. 28->29 re-centring upscale in float32 (deform.py:87-99);
//   3. 21-tap Gaussian (numpy pairwise-sum normalisation) and two separable
//      zero-padded passes per field in fp64, scipy's symmetric tap order: one
//      thread per (image, field, line), the 29-sample line in registers and
//      the 21-tap case fully unrolled, smoothed in place;
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

// Several images per CTA (kImgs): every phase below runs over all of them at
// once, so each barrier is shared by kImgs images and the per-image phases
// with little parallelism (the 21 taps, the scalars) fill the CTA.
constexpr int kImgs = 4;

struct ImgSmem {
  double nx[kPix], ny[kPix];  // noise fields, smoothed in place
  float up[kPix];
  __align__(16) uint8_t raw[784];
  double g[64];    // Gaussian taps
  double u[8];     // sigma-u, alpha-u, mode, angle-u, gamma-u, sx-u, sy-u | tap sum
  double scal[9];  // sigma, alpha, mode, angle, sx, sy | cos, sin, tan of the angle
  uint64_t key[2];
};

// deform.py:87-99: v / 127.5 - 1 per byte (float32, the IEEE division done
// once per byte value into a 256-entry table), then the 2x2 mean of the
// re-centred 29x29 grid.  img: the 784 bytes, staged in shared memory.
__device__ __forceinline__ void byte_table(float* lut) {
  for (int v = threadIdx.x; v < 256; v += blockDim.x) lut[v] = (float)v / 127.5f - 1.0f;
}
__device__ __forceinline__ void upscale_px(const uint8_t* img, const float* lut, int p, float* up) {
  const int r = p / kGrid, c = p % kGrid;
  const int r0 = max(r - 1, 0), r1 = min(r, 27), c0 = max(c - 1, 0), c1 = min(c, 27);
  const float n00 = lut[img[r0 * 28 + c0]];
  const float n01 = lut[img[r0 * 28 + c1]];
  const float n10 = lut[img[r1 * 28 + c0]];
  const float n11 = lut[img[r1 * 28 + c1]];
  up[p] = 0.25f * (((n00 + n01) + n10) + n11);
}

// scipy.ndimage.convolve1d, constant mode (zero padding), symmetric kernel
// (deform.py:130-131), along one 29-sample line held in registers:
// out[c] = x[c]*g(0) + sum_{k=h..1} (x[c-k] + x[c+k]) * g(k), with the
// out-of-range samples as explicit zeros (the same additions as scipy).
// H = the half width at compile time (fully unrolled, taps in registers);
// H < 0: the half width h at run time (any odd kernel size).
template <int H>
__device__ __forceinline__ void conv_line(double* base, int stride, bool act, const double* gs,
                                          int h) {
  double x[kGrid];
#pragma unroll
  for (int i = 0; i < kGrid; i++) x[i] = act ? base[i * stride] : 0.0;
  __syncthreads();  // every line of the pass is read before any is overwritten
  if (!act) return;
  if constexpr (H >= 0) {
    double g[H + 1];  // g[k] = tap at distance k
#pragma unroll
    for (int k = 0; k <= H; k++) g[k] = gs[H + k];
#pragma unroll
    for (int c = 0; c < kGrid; c++) {
      double acc = x[c] * g[0];
#pragma unroll
      for (int k = H; k >= 1; k--) {
        const double xl = c - k >= 0 ? x[c - k >= 0 ? c - k : 0] : 0.0;
        const double xh = c + k < kGrid ? x[c + k < kGrid ? c + k : 0] : 0.0;
        acc = acc + (xl + xh) * g[k];
      }
      base[c * stride] = acc;
    }
  } else {
    for (int c = 0; c < kGrid; c++) {
      double acc = x[c] * gs[h];
      for (int k = h; k >= 1; k--) {
        const double xl = c - k >= 0 ? x[c - k] : 0.0;
        const double xh = c + k < kGrid ? x[c + k] : 0.0;
        acc = acc + (xl + xh) * gs[h + k];
      }
      base[c * stride] = acc;
    }
  }
}

// The smoothing and the warp of up to kImgs images whose draws are in S[]
// (noise in nx/ny, scalars in scal[0..5]); out rows of kPix floats.
template <int H>
__device__ __forceinline__ void deform_batch(ImgSmem* S, int nimg, int ks, float* out) {
  const int tid = threadIdx.x;
  const int h = ks / 2;
  // taps (64 threads per image) and the rotation's trig (one thread per image)
  {
    const int i = tid >> 6, j = tid & 63;
    if (i < nimg) {
      const double sigma = S[i].scal[0];
      if (j < ks) {
        const double off = (double)j - (double)h;
        S[i].g[j] = exp(-(off * off) / (2.0 * sigma * sigma));
      }
      if (j == 63) {
        const double rad = S[i].scal[3] * (3.141592653589793 / 180.0);  // np.deg2rad
        S[i].scal[6] = cos(rad);
        S[i].scal[7] = sin(rad);
        S[i].scal[8] = tan(rad);
      }
    }
  }
  __syncthreads();
  if ((tid & 63) == 0 && (tid >> 6) < nimg) {  // numpy pairwise sum of the taps (n < 128)
    const double* g = S[tid >> 6].g;
    double sum;
    if (ks < 8) {
      sum = 0.0;
      for (int i = 0; i < ks; i++) sum += g[i];
    } else {
      double r[8];
      for (int k = 0; k < 8; k++) r[k] = g[k];
      int i;
      for (i = 8; i < ks - (ks % 8); i += 8)
        for (int k = 0; k < 8; k++) r[k] += g[i + k];
      sum = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
      for (; i < ks; i++) sum += g[i];
    }
    S[tid >> 6].u[7] = sum;
  }
  __syncthreads();
  {
    const int i = tid >> 6, j = tid & 63;
    if (i < nimg && j < ks) S[i].g[j] = S[i].g[j] / S[i].u[7];
  }
  __syncthreads();
  // separable passes: axis 0 (down the columns) then axis 1 (along the rows),
  // one thread per (image, field, line), the line in registers
  const int nl = nimg * 2 * kGrid;
  const bool act = tid < nl;
  const int i = act ? tid / (2 * kGrid) : 0, f = (tid / kGrid) & 1, line = tid % kGrid;
  double* fld = f ? S[i].ny : S[i].nx;
  conv_line<H>(fld + line, kGrid, act, S[i].g, h);  // column `line`
  __syncthreads();
  conv_line<H>(fld + line * kGrid, 1, act, S[i].g, h);  // row `line`
  __syncthreads();
  // rotation-or-shear + scale about the centre, plus the elastic field, then
  // the bilinear warp with -1 background and clip (deform.py:170-200)
  const double center = (kGrid - 1) / 2.0;
  for (int t = tid; t < nimg * kPix; t += blockDim.x) {
    const int im = t / kPix, p = t - im * kPix;
    const ImgSmem& Si = S[im];
    const double alpha = Si.scal[1];
    const int mode = (int)Si.scal[2];
    const double sx = Si.scal[4], sy = Si.scal[5];
    const double cs = Si.scal[6], sn = Si.scal[7], tn = Si.scal[8];
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
    const double dx = (xr - x) + alpha * Si.nx[p];
    const double dy = (yr - y) + alpha * Si.ny[p];
    const double sr = (double)r + dy, sc = (double)c + dx;
    const double flr = floor(sr), flc = floor(sc);
    const long long i0 = (long long)flr, j0 = (long long)flc;
    const double fr = sr - (double)i0, fc = sc - (double)j0;
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const long long ii = i0 + (q >> 1), jj = j0 + (q & 1);
      const bool valid = ii >= 0 && ii < kGrid && jj >= 0 && jj < kGrid;
      v[q] = valid ? (double)Si.up[ii * kGrid + jj] : -1.0;
    }
    double o = (1.0 - fr) * (1.0 - fc) * v[0];
    o = o + (1.0 - fr) * fc * v[1];
    o = o + fr * (1.0 - fc) * v[2];
    o = o + fr * fc * v[3];
    o = o < -1.0 ? -1.0 : (o > 1.0 ? 1.0 : o);
    out[(size_t)im * kPix + p] = (float)o;
  }
}

template <int H>
__global__ void __launch_bounds__(kDefThreads, 2)
    k_deform(const uint8_t* __restrict__ raw, const uint8_t* __restrict__ labels, long long first,
             long long n, unsigned long long seed, unsigned long long epoch, DefP P,
             float* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smraw[];
  ImgSmem* S = reinterpret_cast<ImgSmem*>(smraw);
  float* lut = reinterpret_cast<float*>(S + kImgs);
  const int tid = threadIdx.x;
  const int N = kPix;
  byte_table(lut);
  for (long long b0 = (long long)blockIdx.x * kImgs; b0 < n; b0 += (long long)gridDim.x * kImgs) {
    const int nimg = (int)min((long long)kImgs, n - b0);
    if (tid < nimg) {  // substream key (seed, 2, epoch, index), rng.py:27-38
      uint64_t hh = splitmix64(seed);
      hh = splitmix64(hh ^ 2ULL);
      hh = splitmix64(hh ^ epoch);
      hh = splitmix64(hh ^ (uint64_t)(first + b0 + tid));
      S[tid].key[0] = hh;
      S[tid].key[1] = splitmix64(hh);
    }
    if ((reinterpret_cast<uintptr_t>(raw) & 15) == 0) {  // raw bytes as 16-byte vectors (784 = 49*16)
      for (int t = tid; t < nimg * 49; t += blockDim.x) {
        const int im = t / 49;
        reinterpret_cast<uint4*>(S[im].raw)[t - im * 49] =
            reinterpret_cast<const uint4*>(raw + (b0 + im) * 784)[t - im * 49];
      }
    } else {
      for (int t = tid; t < nimg * 784; t += blockDim.x) S[t / 784].raw[t % 784] = raw[b0 * 784 + t];
    }
    __syncthreads();
    for (int t = tid; t < nimg * kPix; t += blockDim.x) {
      const int im = t / kPix;
      upscale_px(S[im].raw, lut, t - im * kPix, S[im].up);
    }
    // the 423 Philox4x64-10 blocks of every image, decoded into the draw map
    // (two blocks per thread interleaved measured slower: 47.0 -> 45.1M imgs/s)
    for (int t = tid; t < nimg * kBlocks; t += blockDim.x) {
      const int im = t / kBlocks, b = t - im * kBlocks;
      ImgSmem& Si = S[im];
      uint64_t w[4];
      philox4x64_10(Si.key[0], Si.key[1], (uint64_t)b + 1, w);
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const int wi = 4 * b + e;
        if (wi >= kWords) break;
        if (wi >= 2 && wi < 2 + N) {
          Si.nx[wi - 2] = uniform(-1.0, 1.0, u53(w[e]));
        } else if (wi >= 2 + N && wi < 2 + 2 * N) {
          Si.ny[wi - 2 - N] = uniform(-1.0, 1.0, u53(w[e]));
        } else if (wi == 2 + 2 * N) {  // integers(0, 2): bit 31 of the low half
          Si.u[2] = (double)(((w[e] & 0xFFFFFFFFULL) * 2ULL) >> 32);
        } else {
          const int slot = wi < 2 ? wi : wi - 2 * N;  // 0,1 | 3..6
          Si.u[slot] = u53(w[e]);
        }
      }
    }
    __syncthreads();
    if (tid < nimg) {
      ImgSmem& Si = S[tid];
      const int digit = labels[b0 + tid];
      const double beta = (digit == 1 || digit == 7) ? P.beta_red : P.beta_def;
      Si.scal[0] = uniform(P.sig_lo, P.sig_hi, Si.u[0]);
      Si.scal[1] = uniform(P.al_lo, P.al_hi, Si.u[1]);
      Si.scal[2] = Si.u[2];
      Si.scal[3] = uniform(-beta, beta, Si.u[3]);
      const double gamma = uniform(P.ga_lo, P.ga_hi, Si.u[4]);
      Si.scal[4] = uniform(1.0 - gamma / 100.0, 1.0 + gamma / 100.0, Si.u[5]);
      Si.scal[5] = uniform(1.0 - gamma / 100.0, 1.0 + gamma / 100.0, Si.u[6]);
    }
    __syncthreads();
    deform_batch<H>(S, nimg, P.ks, out + b0 * kPix);
    __syncthreads();
  }
}

template <int H>
__global__ void __launch_bounds__(kDefThreads, 2)
    k_deform_injected(const uint8_t* __restrict__ raw, long long n, const double* __restrict__ ndx,
                      const double* __restrict__ ndy, const double* __restrict__ scal, int ks,
                      float* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smraw[];
  ImgSmem* S = reinterpret_cast<ImgSmem*>(smraw);
  float* lut = reinterpret_cast<float*>(S + kImgs);
  const int tid = threadIdx.x;
  byte_table(lut);
  for (long long b0 = (long long)blockIdx.x * kImgs; b0 < n; b0 += (long long)gridDim.x * kImgs) {
    const int nimg = (int)min((long long)kImgs, n - b0);
    for (int t = tid; t < nimg * 784; t += blockDim.x) S[t / 784].raw[t % 784] = raw[b0 * 784 + t];
    __syncthreads();
    for (int t = tid; t < nimg * kPix; t += blockDim.x) {
      const int im = t / kPix, p = t - im * kPix;
      upscale_px(S[im].raw, lut, p, S[im].up);
      S[im].nx[p] = ndx[(b0 + im) * kPix + p];
      S[im].ny[p] = ndy[(b0 + im) * kPix + p];
    }
    if (tid < 6 * nimg) S[tid / 6].scal[tid % 6] = scal[b0 * 6 + tid];
    __syncthreads();
    deform_batch<H>(S, nimg, ks, out + b0 * kPix);
    __syncthreads();
  }
}

__global__ void k_upscale(const uint8_t* __restrict__ raw, long long n, float* __restrict__ out) {
  __shared__ float lut[256];
  __shared__ __align__(16) uint8_t img[784];
  byte_table(lut);
  for (long long i = blockIdx.x; i < n; i += gridDim.x) {
    for (int t = threadIdx.x; t < 784; t += blockDim.x) img[t] = raw[i * 784 + t];
    __syncthreads();
    for (int p = threadIdx.x; p < kPix; p += blockDim.x) {
      const int r = p / kGrid, c = p % kGrid;
      const int r0 = max(r - 1, 0), r1 = min(r, 27), c0 = max(c - 1, 0), c1 = min(c, 27);
      out[i * kPix + p] = 0.25f * (((lut[img[r0 * 28 + c0]] + lut[img[r0 * 28 + c1]]) +
                                    lut[img[r1 * 28 + c0]]) + lut[img[r1 * 28 + c1]]);
    }
    __syncthreads();
  }
}

static int grid_for(long long n, int per_cta = 1, int per_sm = 8) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long units = (n + per_cta - 1) / per_cta;
  const long long g = (long long)sms * per_sm;
  return (int)(units < g ? units : g);
}

// The compiled half width of the fully unrolled smoothing (kernel_size 21,
// deform.py's default); other sizes run the run-time-width instance.
constexpr int kUnrolledH = 10;

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
  const int smem = (int)sizeof(ImgSmem) * kImgs + 256 * (int)sizeof(float);
  auto fn = params->kernel_size == 2 * kUnrolledH + 1 ? k_deform<kUnrolledH> : k_deform<-1>;
  rc = cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                  "cudaFuncSetAttribute");
  if (rc) return rc;
  fn<<<grid_for(n, kImgs, 2), kDefThreads, smem, (cudaStream_t)stream>>>(
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
  const int smem = (int)sizeof(ImgSmem) * kImgs + 256 * (int)sizeof(float);
  auto fn = kernel_size == 2 * kUnrolledH + 1 ? k_deform_injected<kUnrolledH>
                                              : k_deform_injected<-1>;
  int rc = cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                      "cudaFuncSetAttribute");
  if (rc) return rc;
  fn<<<grid_for(n, kImgs, 2), kDefThreads, smem, (cudaStream_t)stream>>>(
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
