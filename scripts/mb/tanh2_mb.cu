// tanh2_mb.cu -- candidate fast tanh forms for the training kernel against the
// glibc restatement (dev_tanhf): dependent-chain latency, and an exhaustive
// comparison over every float (ulp histogram vs glibc and vs correctly
// rounded, the latter from CUDA's double tanh rounded to float).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I paper_1003_0358_b200/csrc \
//        scripts/mb/tanh2_mb.cu -o /tmp/tanh2_mb && /tmp/tanh2_mb
#include <cstdio>
#include "dmlp_math.cuh"
using namespace dmlp;

// fp64 core: tanh = em1 / (em1 + 2), em1 = expm1(2|x|) = 2^k (expm1(r) + 1) - 1.
template <int DEG>
__device__ __forceinline__ float tanh_f64(float x) {
  const double ax = fabs((double)x);
  const double t = fmin(2.0 * ax, 40.0);
  const double L2E = 1.4426950408889634, LN2_HI = 6.93147180369123816490e-01,
               LN2_LO = 1.90821492927058770002e-10, MAGIC = 6755399441055744.0;  // 1.5 * 2^52
  const double km = __fma_rn(t, L2E, MAGIC);
  const double k = __dsub_rn(km, MAGIC);
  const int ki = __double2loint(km);
  double r = __fma_rn(-k, LN2_HI, t);
  r = __fma_rn(-k, LN2_LO, r);
  // Taylor coefficients 1/n!, n = DEG .. 2
  const double c[10] = {1.0, 1.0, 0.5, 1.0 / 6, 1.0 / 24, 1.0 / 120, 1.0 / 720, 1.0 / 5040,
                        1.0 / 40320, 1.0 / 362880};
  double p = c[DEG];
#pragma unroll
  for (int n = DEG - 1; n >= 2; n--) p = __fma_rn(p, r, c[n]);
  const double em1r = __fma_rn(__dmul_rn(p, r), r, r);
  const double tk = __hiloint2double((ki + 1023) << 20, 0);
  const double em1 = __fma_rn(tk, em1r, __dsub_rn(tk, 1.0));
  const double d = __dadd_rn(em1, 2.0);
  double rc;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rc) : "d"(d));
  double e = __fma_rn(-d, rc, 1.0);
  rc = __fma_rn(rc, e, rc);
  e = __fma_rn(-d, rc, 1.0);
  rc = __fma_rn(rc, e, rc);
  const float f = __double2float_rn(__dmul_rn(em1, rc));
  const float s = copysignf(f, x);
  return x != x ? x : s;
}

// fp32 core, same structure.
template <int DEG>
__device__ __forceinline__ float tanh_f32(float x) {
  const float ax = fabsf(x);
  const float t = fminf(2.0f * ax, 20.0f);
  const float L2E = 1.44269504f, LN2_HI = 0.693145751953125f, LN2_LO = 1.428606765330187e-06f,
              MAGIC = 12582912.0f;  // 1.5 * 2^23
  const float km = __fmaf_rn(t, L2E, MAGIC);
  const float k = __fsub_rn(km, MAGIC);
  const int ki = __float_as_int(km) & 0x3fffff;
  float r = __fmaf_rn(-k, LN2_HI, t);
  r = __fmaf_rn(-k, LN2_LO, r);
  const float c[10] = {1.0f, 1.0f, 0.5f, 1.0f / 6, 1.0f / 24, 1.0f / 120, 1.0f / 720, 1.0f / 5040,
                       1.0f / 40320, 1.0f / 362880};
  float p = c[DEG];
#pragma unroll
  for (int n = DEG - 1; n >= 2; n--) p = __fmaf_rn(p, r, c[n]);
  const float em1r = __fmaf_rn(__fmul_rn(p, r), r, r);
  const float tk = __int_as_float((ki + 127) << 23);
  const float em1 = __fmaf_rn(tk, em1r, __fsub_rn(tk, 1.0f));
  const float q = fdiv_fast(em1, __fadd_rn(em1, 2.0f));
  const float s = copysignf(q, x);
  return x != x ? x : s;
}

// hybrid: odd polynomial below 0.55 (x + x s Q(s), s = x^2, Q fitted for
// relative error 2^-29 on [0, 0.55]), the exp form above; both evaluated,
// one selected (no divergence).  FORM 0: em1 / (em1 + 2); 1: 1 - 2 / (em1 + 2).
template <int DEG, int FORM>
__device__ __forceinline__ float tanh_hyb(float x) {
  const float ax = fabsf(x);
  const float s = __fmul_rn(x, x);
  float Q = -0.006324879825115204f;
  Q = __fmaf_rn(Q, s, 0.021108314394950867f);
  Q = __fmaf_rn(Q, s, -0.05386148393154144f);
  Q = __fmaf_rn(Q, s, 0.13332676887512207f);
  Q = __fmaf_rn(Q, s, -0.33333319425582886f);
  const float ysmall = __fmaf_rn(__fmul_rn(ax, s), Q, ax);
  const float t = fminf(2.0f * ax, 20.0f);
  const float L2E = 1.44269504f, LN2_HI = 0.693145751953125f, LN2_LO = 1.428606765330187e-06f,
              MAGIC = 12582912.0f;
  const float km = __fmaf_rn(t, L2E, MAGIC);
  const float k = __fsub_rn(km, MAGIC);
  const int ki = __float_as_int(km) & 0x3fffff;
  float r = __fmaf_rn(-k, LN2_HI, t);
  r = __fmaf_rn(-k, LN2_LO, r);
  const float c[10] = {1.0f, 1.0f, 0.5f, 1.0f / 6, 1.0f / 24, 1.0f / 120, 1.0f / 720, 1.0f / 5040,
                       1.0f / 40320, 1.0f / 362880};
  float p = c[DEG];
#pragma unroll
  for (int n = DEG - 1; n >= 2; n--) p = __fmaf_rn(p, r, c[n]);
  const float em1r = __fmaf_rn(__fmul_rn(p, r), r, r);
  const float tk = __int_as_float((ki + 127) << 23);
  const float em1 = __fmaf_rn(tk, em1r, __fsub_rn(tk, 1.0f));
  const float ylarge = FORM == 0 ? fdiv_fast(em1, __fadd_rn(em1, 2.0f))
                                 : __fsub_rn(1.0f, fdiv_fast(2.0f, __fadd_rn(em1, 2.0f)));
  const float y = fsel(ax < 0.55f, ysmall, ylarge);
  const float sg = copysignf(y, x);
  return x != x ? x : sg;
}

template <int V>
__device__ __forceinline__ float tv(float x) {
  if (V == 6) return tanh_hyb<8, 0>(x);
  if (V == 7) return tanh_hyb<8, 1>(x);
  if (V == 8) return tanh_hyb<7, 1>(x);
  if (V == 9) return tanh_hyb<6, 1>(x);
  if (V == 0) return dev_tanhf(x);
  if (V == 1) return tanh_f64<9>(x);
  if (V == 2) return tanh_f64<8>(x);
  if (V == 3) return tanh_f32<8>(x);
  if (V == 4) return tanh_f32<7>(x);
  float r;
  asm("tanh.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

template <int V>
__global__ void k_lat(float x0, int n, float* out, long long* cyc) {
  float x = x0 + threadIdx.x * 1e-3f;
  const long long t0 = clock64();
  for (int i = 0; i < n; i++) x = tv<V>(x) * 1.3f;
  const long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[V & 7] = (t1 - t0) / n;
}

// per variant: [0] differ from glibc, [1] max ulp vs glibc, [2] differ from
// correctly rounded, [3] max ulp vs correctly rounded
template <int V>
__global__ void k_cmp(unsigned long long* st) {
  unsigned long long dg = 0, dc = 0, mg = 0, mc = 0;
  for (unsigned long long u = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
       u < 0x100000000ull; u += (unsigned long long)gridDim.x * blockDim.x) {
    const float x = __uint_as_float((uint32_t)u);
    if (x != x) continue;
    const int a = __float_as_int(tv<V>(x)), g = __float_as_int(dev_tanhf(x));
    const int c = __float_as_int(__double2float_rn(tanh((double)x)));
    const unsigned long long eg = (unsigned long long)llabs((long long)a - g);
    const unsigned long long ec = (unsigned long long)llabs((long long)a - c);
    dg += eg != 0; dc += ec != 0;
    mg = eg > mg ? eg : mg; mc = ec > mc ? ec : mc;
  }
  atomicAdd(st + 0, dg); atomicMax(st + 1, mg); atomicAdd(st + 2, dc); atomicMax(st + 3, mc);
}

template <int V>
void run(const char* name, float* o, long long* c, unsigned long long* st) {
  long long h[8];
  for (int th : {1, 32}) {
    k_lat<V><<<1, th>>>(0.3f, 2000, o, c);
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-22s threads=%2d  %lld cycles/call\n", name, th, h[V & 7]);
  }
  cudaMemset(st, 0, 32);
  k_cmp<V><<<148 * 4, 512>>>(st);
  unsigned long long s[4];
  cudaMemcpy(s, st, 32, cudaMemcpyDeviceToHost);
  printf("%-22s vs glibc: %llu differ (max %llu ulp); vs correctly rounded: %llu differ (max %llu ulp)\n",
         name, s[0], s[1], s[2], s[3]);
}

int main() {
  float* o; long long* c; unsigned long long* st;
  cudaMalloc(&o, 4096); cudaMalloc(&c, 64); cudaMalloc(&st, 32);
  run<0>("glibc restatement", o, c, st);
  run<1>("fp64 core, deg 9", o, c, st);
  run<2>("fp64 core, deg 8", o, c, st);
  run<3>("fp32 core, deg 8", o, c, st);
  run<4>("fp32 core, deg 7", o, c, st);
  run<5>("tanh.approx.f32", o, c, st);
  run<6>("hybrid deg8 em1/(em1+2)", o, c, st);
  run<7>("hybrid deg8 1-2/(em1+2)", o, c, st);
  run<8>("hybrid deg7 1-2/(em1+2)", o, c, st);
  run<9>("hybrid deg6 1-2/(em1+2)", o, c, st);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
