/*
 * dmlp.h -- C-ABI of libdmlp.so, the sm_100a implementation of the on-line
 * back-propagation / deformation / evaluation hot path of the reference
 * package deepmlp (/root/reference/pkg/src/deepmlp).
 *
 * Plain pointers and sizes only.  Device pointers are CUDA device addresses
 * (e.g. torch.Tensor.data_ptr()); "host or device" pointers are resolved by
 * UVA (cudaMemcpyDefault).  Every call returns a status code; on failure
 * dmlp_last_error() returns a thread-local message.
 *
 * Status codes map to the reference's Python exceptions:
 *   DMLP_ESIZE  -> network.SizeMismatch      (network.py:20-21)
 *   DMLP_EINVAL -> ValueError / deform.InvalidSigma / deform.EvenSize
 *                  (kernels.py:289-290, deform.py:26-31, 51-62)
 *   DMLP_ECUDA  -> RuntimeError (CUDA failure)
 */
#ifndef DMLP_H
#define DMLP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DMLP_OK 0
#define DMLP_ESIZE 1
#define DMLP_EINVAL 2
#define DMLP_ECUDA 3
#define DMLP_ENCCL 4

/* Weight residency of the persistent training kernel. */
#define DMLP_RES_AUTO 0   /* keep the largest set of layers that fits in smem, stream the rest */
#define DMLP_RES_L2 1     /* every hidden layer streamed through L2 (.cg) every sample */
#define DMLP_RES_SMEM 2   /* every CTA keeps its owned rows in shared memory */
#define DMLP_RES_HYBRID 3 /* (reported only) some layers resident, the rest streamed */
#define DMLP_RES_MASK 0x10000 /* DMLP_RES_MASK | m: exactly the layers in bitmask m resident */
#define DMLP_RES_NOREG 0x20000 /* with AUTO: shared memory / L2 only, no register row blocks */
#define DMLP_RES_ALLPATHS 0x40000 /* run the kernel instance with every residency path compiled in
                                     (same plan; for compute-sanitizer coverage) */

typedef struct dmlp_net dmlp_net;

/* deform.DeformParams (deform.py:40-62). */
typedef struct {
  double sigma_lo, sigma_hi;
  double alpha_lo, alpha_hi;
  double beta_default, beta_reduced;
  double gamma_lo, gamma_hi;
  int32_t kernel_size;
} dmlp_deform_params;

/* Thread-local description of the last failure ("" when none). */
const char *dmlp_last_error(void);

/* Library / device facts: SM count, max opt-in smem per block, L2 bytes. */
int dmlp_device_info(int device, int32_t *n_sms, int32_t *smem_per_block,
                     int64_t *l2_bytes, int64_t *persisting_l2_max);

/* ---- network state (replaces network.Mlp / Architecture, network.py:40-106) ---- */

/* sizes = Architecture.layer_sizes (input first).  n_ctas <= 0 selects one
 * CTA per SM.  Weights are zero until dmlp_net_set_layer. */
int dmlp_net_create(int device, const int32_t *sizes, int32_t n_sizes, int32_t residency,
                    int32_t n_ctas, dmlp_net **out);
int dmlp_net_destroy(dmlp_net *net);
/* Residency actually selected, CTA count, threads per CTA, dynamic smem bytes. */
int dmlp_net_info(dmlp_net *net, int32_t *residency, int32_t *n_ctas, int32_t *threads,
                  int32_t *smem_bytes);

/* Where each weight layer's owned rows live in the training kernel:
 * where[l] = 0 streamed from L2 every sample, 1 shared memory, 2 registers
 * (n_layers entries; the output layer's column tile is always in smem). */
int dmlp_net_layer_residency(dmlp_net *net, int32_t *where);

/* Per weight layer, how many of the `fi+1` columns of every owned row sit in
 * registers (reg_cols) and in the register plan's shared-memory tail
 * (tail_cols); both 0 for smem / L2 layers.  For the hybrid roofline
 * (bench.py: bytes per level / that level's peak). */
int dmlp_net_layer_regcols(dmlp_net *net, int32_t *reg_cols, int32_t *tail_cols);
/* Per weight layer: rows per CTA of an L2-streamed layer whose weights the
 * training kernel serves from L1 (the streamed layer's first rows per thread,
 * kernel instances with the L1 feature; 0 elsewhere). */
int dmlp_net_layer_l1rows(dmlp_net *net, int32_t *rows);

/* Pack one layer from the reference layout (fo, fi+1) row-major, bias last
 * (network.py:61-64), host or device pointer, n = fo*(fi+1) floats. */
int dmlp_net_set_layer(dmlp_net *net, int32_t layer, const float *w, int64_t n);
/* Unpack one layer back into the reference layout (host or device pointer). */
int dmlp_net_get_layer(dmlp_net *net, int32_t layer, float *w, int64_t n);

/* In-kernel profile of the persistent training kernel: when enabled, thread
 * 0 of every CTA accumulates per-phase cycle counts.  read fills slots[16]
 * with the sums over CTAs and resets them: slot 0 = sample-loop cycles,
 * 1 = cycles waiting in inter-CTA exchanges, 2.. = phases. */
int dmlp_net_profile(dmlp_net *net, int32_t enable);
int dmlp_net_read_profile(dmlp_net *net, int64_t *slots);
/* The same plus the per-layer split: slots[16 + 5*l + k] for weight layer l,
 * k = 0 forward, 1 gather of its input, 2 column partials, 3 update,
 * 4 gather of the partials by the layer below.  Fills n_slots (<= 96). */
int dmlp_net_read_profile_all(dmlp_net *net, int64_t *slots, int32_t n_slots);
/* The same per CTA, unsummed: slots[c * 96 + k] (96 words per CTA: the 16
 * phase slots -- slot 12 = the CTA's SM id + 1, per launch -- then 5 per
 * layer), and reset. */
int dmlp_net_read_profile_cta(dmlp_net *net, int64_t *slots);
/* One-sample timeline of the next launches: every CTA records %globaltimer
 * at 64 marks of sample `sample` (mark 0 start; for exchange e, 1+2e = its
 * contribution published, 2+2e = its gather done; 63 end).  marks (optional,
 * [n_ctas][64]) receives the previous recording; sample < 0 disables. */
int dmlp_net_trace(dmlp_net *net, int64_t sample, uint64_t *marks);

/* ---- on-line training (kernels.train_step / trainer.train_epoch) ---- */

/* kernels.train_step (kernels.py:329-361): one on-line update on input x
 * (n_inputs floats, host or device), target class digit, rate eta >= 0.
 * y_out (10 floats, host or device) receives the output activations
 * computed before the update.  Synchronous. */
int dmlp_train_step(dmlp_net *net, const float *x, int32_t digit, float eta, float *y_out);

/* trainer.train_epoch (trainer.py:104-123): sequential on-line pass over
 * samples order[0..n) (order NULL = identity) of x_dev (rows of n_inputs
 * floats, row stride ldx floats) with labels_dev (u8).  Adds the number of
 * argmax errors to *wrong_dev (device int64).  y_last_dev (optional, 10
 * floats) receives the output of the last sample.  pred_dev (optional, n
 * bytes) receives the argmax of every sample's output in training order
 * (np.argmax, first maximum: trainer.py:121).  Asynchronous on stream. */
int dmlp_train_epoch(dmlp_net *net, const float *x_dev, int64_t ldx, const uint8_t *labels_dev,
                     const int32_t *order_dev, int64_t n, float eta, int64_t *wrong_dev,
                     float *y_last_dev, uint8_t *pred_dev, void *stream);

/* ---- evaluation (network.forward_batch / eval_report.evaluate) ---- */

/* network.forward_batch (network.py:118-130): out_dev (n,10) = outputs. */
int dmlp_forward_batch(dmlp_net *net, const float *x_dev, int64_t n, float *out_dev,
                       void *stream);

/* trainer.error_percent + eval_report.evaluate counting (trainer.py:90-96,
 * eval_report.py:36-67): counts_dev (int64[102]) += {wrong, confusion[10][10]
 * (rows = true digit), second_guess_correct}; guess_dev (optional, int32
 * (n,2)) = top-2 ranked digits (stable: ties go to the smaller digit). */
int dmlp_eval_counts(dmlp_net *net, const float *x_dev, const uint8_t *labels_dev, int64_t n,
                     int64_t *counts_dev, int32_t *guess_dev, void *stream);

/* ---- deformation (deform.py / rng.py) ---- */

/* deform.deform_epoch (deform.py:217-247) for images [first, first+n) of a
 * split: raw_dev (n,28,28) u8, labels_dev (n) u8 -> out_dev (n,29,29) f32.
 * Image i uses substream(seed, 2, epoch, first+i) (rng.py:27-38). */
int dmlp_deform(const uint8_t *raw_dev, const uint8_t *labels_dev, int64_t first, int64_t n,
                uint64_t seed, uint64_t epoch, const dmlp_deform_params *params,
                float *out_dev, void *stream);

/* Injected-field parity mode: the random draws are supplied.
 * noise_dx_dev / noise_dy_dev: (n,29,29) f64; scalars_dev: (n,6) f64 =
 * sigma, alpha, mode (0 rotation, 1 shear), angle (deg), sx, sy. */
int dmlp_deform_injected(const uint8_t *raw_dev, int64_t n, const double *noise_dx_dev,
                         const double *noise_dy_dev, const double *scalars_dev,
                         int32_t kernel_size, float *out_dev, void *stream);

/* deform.upscale_dataset (deform.py:250-257): (n,28,28) u8 -> (n,841) f32. */
int dmlp_upscale(const uint8_t *raw_dev, int64_t n, float *out_dev, void *stream);

/* ---- K6 microbenchmarks (roofline denominators, exchange floor) ----
 * kind 0: streaming read of `bytes` (float4, .cg), `iters` passes;
 * kind 1: streaming read+write; kind 2: shared-memory read+write, 128 KB
 * per CTA, `iters` passes; kind 3: exchange ping, `iters` rounds.
 * One 512-thread CTA per SM unless n_ctas > 0.  Returns wall seconds
 * (CUDA events) and the slowest CTA's clock64 cycles. */
int dmlp_bench(int32_t kind, int64_t bytes, int32_t iters, int32_t n_ctas, double *seconds,
               double *cycles);
/* Cycles per op of the sample loop's primitives: [0] __syncthreads (512
 * threads), [1] exact scaled tanh, [2] IEEE fp32 divide, [3] warp shuffle
 * reduction, [4] dependent L2 load, [5] dependent ld.relaxed.gpu, [6] smem load. */
int dmlp_bench_prims(double *out);

/* ---- fp64 gradient-check oracle (kernels.backprop_gradients / gradient_check,
 * kernels.py:374-418), a debug aid for small nets (every layer <= 1024 units).
 * sizes: layer sizes (input first); w_host: float64 weights of every layer in
 * the reference layout (fo, fi+1), bias last, concatenated; x_host: float64
 * input.  grad_bp / grad_fd (optional, host, one float64 per weight): the
 * analytic gradient of E = 0.5*sum((y - t)^2) and the central finite
 * difference with `step`; *worst = max |g_bp - g_fd| / max(|g_bp|, |g_fd|,
 * 1e-8).  Synchronous. */
int dmlp_gradient_check(const int32_t *sizes, int32_t n_sizes, const double *w_host,
                        const double *x_host, int32_t digit, double step, double *grad_bp,
                        double *grad_fd, double *worst);

/* Device tanhf checks: the select-form kernel tanhf against its branchy
 * glibc restatement on all 2^32 inputs (NaN payloads aside), and evaluation
 * on given inputs (device pointers) for comparison with the host libm. */
int dmlp_tanhf_check(uint64_t *mismatches, uint32_t *first_bad);
int dmlp_tanhf_eval(const float *x_dev, float *y_dev, int64_t n);

/* The training kernel's faithfully rounded tanhf (dev_tanhf_fast) over all
 * non-NaN floats: stats[0] inputs where it differs from the glibc
 * restatement, stats[1] the largest difference in ulp; stats[2], stats[3]
 * the same against the correctly rounded tanh.  And evaluation on given
 * inputs (device pointers). */
int dmlp_tanhf_fast_check(uint64_t *stats);
int dmlp_tanhf_fast_eval(const float *x_dev, float *y_dev, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
