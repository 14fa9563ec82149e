// dmlp_internal.h -- shared host/device declarations of libdmlp.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/dmlp.h"

namespace dmlp {

constexpr int kThreads = 512;  // threads per CTA of the persistent kernel
constexpr int kWarps = kThreads / 32;
constexpr int kMaxLayers = 16;
constexpr int kMaxOut = 32;  // output layer: at most 32 classes
constexpr int kProfPhases = 16;  // per-phase profile slots per CTA
constexpr int kProfKinds = 5;    // per-layer slots: fwd, fwd gather, bwd partials, bwd update, bwd gather
constexpr int kProfWords = kProfPhases + kProfKinds * 16;  // (kMaxLayers = 16)
constexpr int kMaxRegLayers = 4;  // register-resident row blocks per CTA
enum { kResL2 = 0, kResSmem = 1, kResReg = 2 };

// One weight layer as the persistent kernel sees it.
//
// Hidden layer l: CTA c owns the row block [c*R, min(c*R+R, fo)).  Inside a
// CTA the 512 threads form G = 2^gs row groups of TG = 512/G threads; thread
// (g, u) handles rows g, g+G, ... and the float4 column quads u, u+TG, ...,
// so every phase (forward dot, column partials, update) keeps all threads
// busy and walks a row with consecutive lanes on consecutive quads.
// Output layer: CTA c owns the COLUMNS of W_out that match its rows of the
// last hidden layer (CTA 0 also the bias column); its [fo][R+1] tile lives
// in shared memory for the whole launch.
struct LayerDev {
  int fi, fo, pitch;     // fan-in, fan-out, floats per device row (>= fi+1, %4 == 0)
  int in_off;            // hidden l >= 1: smem offset of the gathered input vector (pitch long)
  int t_off;             // hidden: smem offset of the owned rows' tanh(B*a) cache
  int res;               // hidden: where the CTA's rows live: kResL2 / kResSmem / kResReg
  int wsm_off;           // smem offset: resident hidden rows / register-block tail / output tile
  int R;                 // hidden: rows per CTA block; output: owned input columns per CTA
  int P;                 // CTAs owning at least one row (output: producing a partial)
  int gs, CH;            // hidden: log2 of the row groups G, rows per reduction chunk
  int ylog;              // log2 words per producer slot of yll (>= 16 words, line aligned)
  int yflat;             // hidden: y words stored flat (word of row i at i) instead of per
                         // producer slot, so every float4 quad is 4 consecutive words
  int pstride;           // hidden l>=1: per-CTA row stride of pll (multiple of 16 words)
  float* w;              // [fo][pitch], reference order, bias in column fi
  // Exchange buffers: every CTA's slice starts on its own 128-byte line, so a
  // polled line has exactly one writer.
  unsigned long long* yll;  // hidden l < L-2: [2][P][1<<ylog] activations;
                            // output: [2][P][1<<ylog] partial pre-activations
  unsigned long long* pll;  // hidden l>=1: [2][P][pstride] column partials
};

struct NetDev {
  int L;    // weight layers
  int nct;  // CTAs (row owners)
  int in0_off[2];
  int delta_off[2];
  int dsc_off[2];
  int yown_off;  // [R] y of the owned rows of the last hidden layer
  int red_off;   // [kWarps][32] reduction scratch
  int pbuf_off;  // [Gmax][pitch] per-row-group column partials (G > 1 layers)
  int out_off;   // output layer scratch: a | y | delta | eta*delta (kMaxOut each)
  int reg_layer[kMaxRegLayers];  // register slot -> hidden layer (-1: unused)
  int* err;
  unsigned long long* prof;  // optional [nct][kProfWords] phase cycles (0 loop, 1 exchange)
  unsigned long long* trace;  // optional [nct][64] %globaltimer marks of one sample
  long long trace_sample;     // which sample of the launch is traced
  LayerDev ly[kMaxLayers];
};

struct HostLayer {
  int fi, fo, pitch;
  size_t w_off;  // float offset into the weights allocation
};

}  // namespace dmlp

struct dmlp_net {
  int device;
  int feat;       // feature set of the launched training instance (kFeat*)
  int residency;
  int n_sizes;
  int32_t sizes[dmlp::kMaxLayers + 1];
  dmlp::HostLayer hl[dmlp::kMaxLayers];
  dmlp::NetDev dev;
  float* d_w = nullptr;
  size_t w_floats = 0;
  unsigned long long* d_ll = nullptr;
  size_t ll_words = 0;
  int* d_err = nullptr;
  int smem_bytes = 0;
  unsigned resident_mask = 0;
  unsigned reg_mask = 0;
  int reg_tail = 0;  // floats of shared-memory tail per register row block
  int variant = 0;                      // selected TrainVariant
  const void* train_fn = nullptr;       // its instance for the net's feature set
  const void* train_fn_prof = nullptr;  // its profiling instance
  uint32_t seq = 1;  // next sample sequence number (flag value)
  cudaStream_t stream = nullptr;
  cudaEvent_t done = nullptr;  // recorded after every operation on the net, whatever the stream
  float* d_stage = nullptr;  // train_step staging: x, y
  uint8_t* d_stage_lab = nullptr;
  long long* d_stage_wrong = nullptr;
  // evaluation scratch
  float* d_act[3] = {nullptr, nullptr, nullptr};  // layer outputs (ping-pong) | padded inputs
  size_t act_rows = 0;
  int act_ld = 0;
};

namespace dmlp {
// Makes `device` current for the scope of an entry point and restores the
// caller's device on exit (torch's current device is never changed behind
// its back).
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int device) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != device) err = cudaSetDevice(device);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
int set_error(int code, const char* fmt, ...);
int cuda_check(cudaError_t e, const char* what);
int net_begin(dmlp_net* net, cudaStream_t st);
int net_end(dmlp_net* net, cudaStream_t st);
cudaError_t launch_train(const dmlp_net* net, const float* x, long long ldx,
                         const uint8_t* labels, const int32_t* order, long long n, float eta,
                         uint32_t seq0, long long* wrong, float* y_last, uint8_t* pred,
                         cudaStream_t st);
// Compiled instantiations of the training kernel: n_reg register row blocks
// of at most rr rows x rc columns per thread (0 = none), plus rs column
// slots per thread in shared memory.
// residency paths compiled into an instance; kFeatL1: the streamed layer's
// first kL1Rows rows per thread through L1 (train_phases.cuh: ldw4)
enum { kFeatSmem = 1, kFeatL2 = 2, kFeatL1 = 4 };
constexpr int kL1Rows = 5;            // 5 x 1504 floats: C4's layer 3, 30 KB of L1
constexpr int kL1Budget = 30 * 1024;  // bytes per SM (the 228 KB carve-out leaves 28 KB)
struct TrainVariant {
  int n_reg, rr, rc, rs;  // rs: column slots of each block kept in a shared-memory tail
  const void* fn[8];      // by feature set (kFeatSmem | kFeatL2 | kFeatL1), no profile hooks; may be null
  const void* fn_prof;    // every feature plus the profile / trace hooks
};
int train_variants(const TrainVariant** out);
// The instance of plan tv compiled with the fewest features covering `feat`.
const void* train_instance(const TrainVariant& tv, int feat);
cudaError_t set_train_attributes(const void* fn, int smem_bytes);
cudaError_t train_occupancy(const void* fn, int smem_bytes, int* blocks_per_sm);
}  // namespace dmlp
