/* unet.h -- C ABI of the temporally conditioned U-Net inference path.
 *
 * The surrogate operator G of Eq. (1), section 4.3:
 *   c(t + dt) = G([c(t-lb+1), ..., c(t)])(dt)
 * encoder  z^{L1} = conv_block(history), z^{Lp} = conv_block(down(z^{Lp-1})), p = 2..4
 * condition z^{Lp}_{t+dt} = z^{Lp}_t (.) w^{Lp} f(dt), f = the sin MLP of P:367-372
 * decoder  d^{L3} = up(conv_block(z^{L4})), d^{Lp} = up(conv_block(z^{Lp+1} (+) d^{Lp+1}))
 * output   GN(conv(conv_block(z^{L1} (+) d^{L1})))
 * conv_block = GELU(GN(conv3x3)); readings R-29..R-35 of DESIGN.md 14.
 *
 * Every step runs in this library's kernels on the GPU: the 3x3 convolutions are implicit GEMMs on
 * the 5th-generation tensor cores (tcgen05.mma, bf16 operands, fp32 accumulators in TMEM); GroupNorm
 * statistics, GELU, conditioning, pooling, up-sampling, concatenation and the time MLP are CUDA
 * kernels.  Activations are stored as bf16 (NHWC) between layers; GroupNorm statistics are fp64.
 * There is no CPU fallback: without a CUDA device every call fails with PF_ERR_CUDA.
 *
 * Status codes are pf_status (pf.h).  Functions never throw; the ctx owns every device buffer and
 * its stream; callers own host buffers.  un_last_error(ctx) describes the last failure.
 */
#ifndef UNET_H_
#define UNET_H_

#include <stddef.h>
#include <stdint.h>

#include "pf.h"

#ifdef __cplusplus
extern "C" {
#endif

#define UN_ABI_VERSION 1u

typedef struct un_ctx un_ctx;

typedef struct {
    uint32_t abi_version;   /* UN_ABI_VERSION                                                  */
    int32_t lb;             /* look-back channels, 1..16 (paper: 3, Appendix D)                  */
    int32_t widths[4];      /* channels C1..C4 of levels L1..L4; multiples of 16, <= 128 (R-33) */
    int32_t height, width;  /* input grid H x W; multiples of 8 (three 2x2 poolings)             */
    int32_t max_batch;      /* largest batch a forward call may pass                             */
    int32_t device;         /* CUDA device ordinal                                               */
} un_params;

/* Defaults: lb = 3, widths (16, 32, 64, 128), 256 x 256 (the paper's grid), batch 64. */
pf_status un_default_params(un_params *out);

/* Number of floats of the weight blob for these params.  Blob layout (row-major, in order):
 * for each conv layer L of enc1 enc2 enc3 enc4 dec4 dec3 dec2 head1 head2 (cin -> cout):
 *   w_L [cout][3][3][cin] (cross-correlation taps), g_L [cout], b_L [cout] (GN gamma, beta);
 * then wl1..wl4 [C_p][128] (w^{Lp}); up3, up2, up1 [2][2] (w^{tconv} of d^{L3}, d^{L2}, d^{L1});
 * then the MLP m_w0 [128], m_b0 [128], m_w1 [128][128], m_b1 [128], m_w2 [128][128], m_b2 [128].
 * Channel counts: enc1 lb->C1, enc2 C1->C2, enc3 C2->C3, enc4 C3->C4, dec4 C4->C3, dec3 2C3->C2,
 * dec2 2C2->C1, head1 2C1->C1, head2 C1->1.  Conv weights are rounded to bf16 on upload. */
int64_t un_blob_size(const un_params *p);

pf_status un_create(const un_params *p, un_ctx **out);

/* Upload a weight blob (host, n = un_blob_size floats). Synchronous. */
pf_status un_set_weights(un_ctx *ctx, const float *blob, int64_t n);

/* Forward pass, device pointers, asynchronous on the ctx stream (un_stream):
 *   hist [batch][lb][H][W] fp32 (values are rounded to bf16 on entry), dt [batch] fp32,
 *   out [batch][H][W] fp32.  1 <= batch <= max_batch.  The 29 launches are captured into a CUDA
 *   graph on the first call with a given (batch, hist, dt, out) and replayed by later calls with
 *   the same arguments (buffer contents and weights may change in between; up to 8 such graphs
 *   are kept, least recently used replaced). */
pf_status un_forward_device(un_ctx *ctx, int32_t batch, const float *hist, const float *dt, float *out);

/* Same with host buffers: H2D copy, forward, D2H copy; returns after the result is on the host.
 * Batches of >= 16 samples are pipelined over 4 sample chunks (the H2D copy of chunk k+1 and the D2H
 * copy of chunk k-1 overlap the forward of chunk k; one cached CUDA graph per chunk); the copies
 * overlap only when hist / dt / out are page-locked host memory.  Same results as one forward of
 * the whole batch (samples are independent). */
pf_status un_forward(un_ctx *ctx, int32_t batch, const float *hist, const float *dt, float *out);

/* Autoregressive rollout (SPEC-style window bookkeeping, "roll out the remaining part"):
 * starting from hist [batch][lb][H][W] (host), n_leaps times predict dt = 1..lf (one forward per dt
 * on the same window), write the lf predictions to out[batch][leap*lf + q][H][W] (host), then
 * take the last lb predictions (lb <= lf) as the next window.  Synchronous. */
pf_status un_rollout(un_ctx *ctx, int32_t batch, const float *hist, int32_t lf, int32_t n_leaps, float *out);

/* Hybrid schedule DNS -> surrogate (section 2.2, the "DNS until t1, then U-Net" runs of
 * P:240-241): n_dns composite-c snapshots of the DNS ctx `dns` (pf_trajectory, steps_between steps
 * apart), then the U-Net rollout (un_rollout) from the last lb of them for n_leaps x lf
 * snapshots.  The DNS ctx must hold a single domain of H x W (= the U-Net grid) with members <=
 * max_batch; n_dns >= lb; lf >= lb.  out [members][n_dns + n_leaps*lf][H][W] (host, fp32);
 * seconds[0] = DNS wall time, seconds[1] = surrogate wall time (host clock around each segment,
 * both synchronised).  The composite (c where phi > 1/2, else 0) is the surrogate's state;
 * no reconstruction of phi and rho follows the last leap (the paper does not describe one). */
pf_status un_hybrid(un_ctx *ctx, pf_ctx *dns, int32_t n_dns, int64_t steps_between, int32_t lf, int32_t n_leaps,
                    float *out, double seconds[2]);

/* One bf16 3x3 'same' convolution on the tensor cores, for parity tests of the GEMM kernel alone:
 * in [npix = batch*H*W][cin] bf16 bits (NHWC), w [cout][9][cin] bf16 bits, out [npix][cout] fp32.
 * cin a multiple of 16, cout in {16, 32, 64, 128}; device pointers; runs on stream (or 0) and
 * synchronises it.  The input is repacked on the device into the kernels' row-chunk activation
 * layout ([b][y][chunk][x][8], unet.cu) before the convolution. */
pf_status un_conv3x3(const uint16_t *in, int32_t batch, int32_t H, int32_t W, int32_t cin, const uint16_t *w,
                     int32_t cout, float *out, void *stream);

/* Diagnostic of a UN_TRACE build (PF_NVCC_EXTRA=-DUN_TRACE=1): per CTA (160 slots) cycle sums of the
 * row-tile convolution's roles since the last reset, out[160][8] = {MMA warp: full wait, acce wait,
 * issue; producer: empty wait, copy issue; epilogue warp 0: accf wait, drain; iterations}.  Zeros
 * in a normal build; then out[160 * 8 + 4 c + k] = CTA c's clock64 at entry, MMA loop start, MMA loop
 * end and exit of the last launch (out holds 160 * 12 values).  reset != 0 zeroes the sums after
 * reading.  Returns a cudaError_t value. */
int un_debug_trace(unsigned long long *out, int reset);

pf_status un_stream(un_ctx *ctx, void **stream);
/* Kernel launches issued by this ctx so far. */
pf_status un_launch_count(un_ctx *ctx, int64_t *launches);
/* Per-forward time of the convolution kernels and of the whole forward (CUDA events, ms), summed
 * since the last reset; enable = 1 turns event recording on (and resets), 0 off.
 * out[0] conv ms, out[1] forward ms, out[2] forwards, out[3] conv flops per forward. */
pf_status un_profile(un_ctx *ctx, int32_t enable);
pf_status un_profile_read(un_ctx *ctx, double out[4]);
const char *un_last_error(const un_ctx *ctx);
void un_free(un_ctx *ctx);

#ifdef __cplusplus
}
#endif

#endif /* UNET_H_ */
