/*
 * libptyger — C ABI of the B200-native PtyGer ML-CG iteration (arXiv 2106.07575).
 *
 * The library computes, entirely on the GPU, the conjugate-gradient iteration of the
 * Poisson maximum-likelihood ptychographic reconstruction of the complex object psi:
 *
 *   forward model      |G psi|^2 = |F Q psi|^2 = d                  (Eq.1)
 *   objective          F(psi) = sum_j |G psi|_j^2 - 2 d_j log|G psi|_j   (Eq.2)
 *   gradient           grad F = G^H (G psi - d / (G psi)^*)             (Eq.3)
 *   direction          eta_m = -grad F_m + alpha_m eta_{m-1},
 *                      alpha_m = ||grad F_m||^2 / <eta_{m-1}, grad F_m - grad F_{m-1}>
 *                                                                    (Eq.6, 533-538 Eq.8)
 *   line search        first gamma = gamma0 tau^k with F(psi+gamma eta) <= F(psi) + gamma t
 *                                                                    (Eq.7, Alg.1 659-668)
 *   update             psi_{m+1} = psi_m + gamma_m eta_m                (Eq.5)
 *
 * Conventions (R#k):
 *   - F is the UNITARY 2-D DFT, e^{-2 pi i k.n/N}, DC at [0,0], no fftshift (R#1, R#2).
 *   - Scan positions are integer TOP-LEFT window corners (row, col) (R#3).
 *   - log|u| and d/u^* are guarded with eps (config.eps, default 1e-16) (R#4).
 *   - the gradient is the Wirtinger derivative dF/dpsi^* (R#5).
 *   - complex numbers are interleaved (re, im) float32 pairs ("complex64", Alg.1);
 *     images are row-major; all scalar accumulation is float64 (R#16).
 *
 * Threading / ownership: one context per host thread, not re-entrant.  Input arrays are
 * COPIED during ptyger_init (host or device pointers, detected with
 * cudaPointerGetAttributes); the caller keeps ownership.  Outputs go to caller-allocated
 * HOST buffers unless stated otherwise.  The context owns all device memory, streams,
 * CUDA graphs and the NCCL communicator; ptyger_destroy frees them.
 *
 * Errors: every call returns a ptyger_status; ptyger_last_error(ctx) (or
 * ptyger_last_error(NULL) after a failed ptyger_init / host helper) gives a message
 * naming the stage, frame index and iteration where applicable.  There is no CPU
 * fallback: without a CUDA device every device call returns PTYGER_E_CUDA.
 */
#ifndef PTYGER_H
#define PTYGER_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ptyger_ctx ptyger_ctx;

typedef enum {
    PTYGER_OK = 0,
    PTYGER_E_ARG = 2,      /* bad configuration / argument / infeasible partition  */
    PTYGER_E_DATA = 3,     /* out-of-bounds window, negative or non-finite d, shape */
    PTYGER_E_NUMERIC = 4,  /* non-finite F, alpha or gamma; last good iterate kept  */
    PTYGER_E_CUDA = 5,     /* CUDA runtime / driver failure or no device            */
    PTYGER_E_NCCL = 6,     /* NCCL failure (world > 1)                              */
    PTYGER_E_OOM = 7,      /* device allocation failed                              */
    PTYGER_E_STATE = 8     /* call not valid in the current context state           */
} ptyger_status;

/* Direction variants (R#6). */
enum { PTYGER_DIR_DY = 0,      /* complex alpha exactly as printed (Eq.6 / Eq.8)   */
       PTYGER_DIR_DY_REAL = 1, /* Re(alpha)                                        */
       PTYGER_DIR_FR = 2,      /* Fletcher-Reeves ||g||^2 / ||g_prev||^2            */
       PTYGER_DIR_PR = 3,      /* Polak-Ribiere+ max(0, Re<g, g - g_prev>) / ||g_prev||^2 */
       PTYGER_DIR_GD = 4 };    /* gradient descent, Eq.4: eta = -g, gamma = gamma0
                                  taken without line search (constant step)         */

/* Estimators (R#19): the Poisson maximum likelihood of Eq.2 or the least squares (Gaussian)
 * estimator F = sum (|G psi| - sqrt d)^2 the paper says the techniques also apply to. */
enum { PTYGER_EST_ML = 0, PTYGER_EST_LS = 1 };

typedef struct {
    double gamma0;        /* first LS trial, 1.0 (Alg.1)                            */
    double tau;           /* shrink factor, 0.5 (Alg.1)                             */
    double t;             /* Armijo-like constant, 0.0                            */
    double eps;           /* modulus guard, 1e-16 (R#4)                                   */
    int32_t max_shrinks;  /* trials per iteration before a stall (gamma = 0), 32 (R#9)    */
    int32_t direction;    /* PTYGER_DIR_*                                                 */
    int32_t ls_batch;     /* K in [4, 16] (default 16): cap of the adaptive pass-0 trial count (k*_prev + 3)
                             and trials per extra LS pass over the frames (the first extra pass takes
                             min(K, 8): a k* past pass 0 is usually a jump of a few) */
    int32_t estimator;    /* PTYGER_EST_ML (default) or PTYGER_EST_LS                          */
    int32_t device;       /* CUDA device ordinal                                          */
    int32_t rank;         /* this process's rank, 0..world-1                              */
    int32_t world;        /* number of ranks (one GPU each)                               */
    const void* nccl_id;  /* 128-byte ncclUniqueId from ptyger_nccl_unique_id (world > 1, NCCL transport) */
    int32_t transport;    /* world > 1: PTYGER_TRANSPORT_P2P (default) or PTYGER_TRANSPORT_NCCL        */
} ptyger_config;

/* Transports of the per-iteration exchanges when world > 1 (band partial gradients, fp64 scalar
 * allreduces, object gather).  NCCL: ncclSend/Recv/AllReduce captured in the iteration graph.
 * P2P: the producing kernels store straight into the other ranks' CUDA-IPC-mapped exchange windows
 * and signal with system-scope release/acquire epoch flags (kernels_p2p.cu); the scalar sums are
 * taken in rank order, so every rank gets bitwise identical values.  P2P contexts are created in two
 * steps: ptyger_init (everything local), then ptyger_ipc_handle on every rank, an out-of-band exchange
 * of the 64-byte handles (e.g. torch.distributed), and ptyger_ipc_connect with all of them.  Ranks may
 * share one GPU (CUDA IPC within a device) or use peer GPUs (NVLink). */
enum { PTYGER_TRANSPORT_NCCL = 0, PTYGER_TRANSPORT_P2P = 1 };

/* Per-iteration trace (SPEC trace fields S:226-229; step_norm = ||psi_{m+1}-psi_m||_2). */
typedef struct {
    int32_t iter;         /* m                                                            */
    int32_t shrinks;      /* accepted trial index k (gamma = gamma0 tau^k); max_shrinks if stalled */
    int32_t restarted;    /* 1 if eta = -grad (m = 0 excluded) because |den| < 1e-30 or alpha non-finite */
    int32_t stalled;      /* 1 if no trial accepted (gamma = 0)                           */
    double F;             /* F(psi_{m+1}) = F(psi_m) + DeltaF_k (cached, R#11)             */
    double gamma;         /* accepted step                                                */
    double alpha_re;      /* alpha_m (0 at m = 0 / restart)                               */
    double alpha_im;
    double grad_norm;     /* ||grad F(psi_m)||_2                                          */
    double step_norm;     /* gamma ||eta_m||_2                                            */
    /* device time of this iteration's stages (ms, GPU global timer stamps between the stages of the
     * graph-launched iteration; SURVEY 8(b), P:284-287 time breakdown): GRAD (frame kernel + adjoint,
     * incl. the band exchange when world > 1), DIR (DY sums, alpha, eta), LS (all passes and
     * decisions), Update; ms_comm = the band-exchange part of ms_grad (0 when world = 1; the fp64
     * scalar sums over ranks ride inside the DIR / LS reductions). */
    float ms_grad, ms_dir, ms_ls, ms_update, ms_comm;
    int32_t ls_passes;        /* line-search passes over the cached far fields this iteration: the
                                 screened pass 0 (fused into the LS frame kernel) plus every further
                                 K-trial pass (no trial of the earlier passes accepted)             */
    int32_t ls_exact_passes;  /* exact re-evaluations of a pass the screening left undecided        */
} ptyger_trace;

/* Fill cfg with the paper's defaults (gamma0 1, tau 0.5, t 0, eps 1e-16, max_shrinks 32,
 * direction DY, ls_batch 16, device 0, rank 0, world 1, nccl_id NULL, transport P2P). */
void ptyger_config_default(ptyger_config* cfg);

/*
 * Create a context and upload one problem (Alg.1).
 *   object       psi_0: H*W complex64 (2*H*W floats), row-major, host or device.
 *   probe        p: N*N complex64, host or device; N in {16, 32, 64, 128, 256}.
 *   scan         n*(row, col) int32 top-left corners, 0<=row<=H-N, 0<=col<=W-N, host.
 *   intensities  d: n*N*N float32 >= 0 and finite, frame j at offset j*N*N, detector pixel
 *                (k1, k2) at k1*N + k2 in DFT order (DC at [0,0]); host or device.
 * When cfg->world > 1 every rank passes the SAME full arrays; the library partitions the
 * frames into row stripes (ptyger_partition) and uploads only its shard.
 * Computes u = G psi_0 and F(psi_0) on the device.
 * Errors: E_ARG (config, N unsupported, infeasible P), E_DATA (window out of bounds,
 * d negative / non-finite: message names the frame), E_CUDA, E_OOM, E_NCCL.
 */
ptyger_status ptyger_init(ptyger_ctx** out, const ptyger_config* cfg,
                          const float* object, int64_t H, int64_t W,
                          const float* probe, int32_t N,
                          const int32_t* scan, int64_t n,
                          const float* intensities);

/*
 * ptyger_init with FRACTIONAL scan positions (Alg.1 input 'float32 h_s').
 * The paper does not say how a non-integer position samples the object; reading R#22: frame j's
 * window is the BILINEAR interpolation of psi at (y_j + i, x_j + k), i.e. with r0 = floor(y_j),
 * fy = y_j - r0 (same for x):
 *     Q_j psi[i, k] = p[i, k] sum_{a, b in {0,1}} wy_a wx_b psi[r0 + i + a, c0 + k + b],
 *     wy_0 = 1 - fy, wy_1 = fy, wx_0 = 1 - fx, wx_1 = fx,
 * and the adjoint Q_j^H scatters with the same real weights.  Integral positions reproduce
 * ptyger_init exactly (the all-integer case runs the integer kernels).
 *   scan  n*(row, col) float32 top-left positions, host; 0 <= row, floor(row) + N + (fy > 0) <= H,
 *         likewise for col / W.
 * Every other argument, the ownership rules and the errors are those of ptyger_init; with
 * world > 1 the partition uses the integer corners floor(x) and an N + 1 row footprint
 * (ptyger_partition_subpixel).  E_DATA: a negative, non-finite or out-of-bounds position.
 */
ptyger_status ptyger_init_subpixel(ptyger_ctx** out, const ptyger_config* cfg,
                                   const float* object, int64_t H, int64_t W,
                                   const float* probe, int32_t N,
                                   const float* scan, int64_t n,
                                   const float* intensities);

/*
 * Run n_iter CG iterations (Alg.1) as CUDA-graph launches with no host
 * synchronisation inside; traces (nullable) receives n_iter entries.  Collective when
 * world > 1.  Errors: E_NUMERIC (non-finite F/alpha/gamma: message names iteration
 * and stage; psi keeps the last good iterate), E_CUDA, E_NCCL.
 */
ptyger_status ptyger_cg_iterate(ptyger_ctx* ctx, int32_t n_iter, ptyger_trace* traces);

/* Split form of ptyger_cg_iterate: cg_launch enqueues n_iter graph launches on the context's stream
 * and returns at once; cg_wait synchronises, fills traces (nullable, n_iter entries) and reports
 * E_NUMERIC like cg_iterate.  Independent contexts (e.g. the views of a 3-D batch) launched before
 * waiting run concurrently on their own streams.  E_STATE: cg_launch twice without cg_wait. */
ptyger_status ptyger_cg_launch(ptyger_ctx* ctx, int32_t n_iter);
ptyger_status ptyger_cg_wait(ptyger_ctx* ctx, ptyger_trace* traces);

/* The context's CUDA stream (cudaStream_t) -- for timing with events / ordering other work. */
void* ptyger_stream(const ptyger_ctx* ctx);

/* Current psi_m, H*W complex64 into a host buffer (Alg.1).  Collective when
 * world > 1 (every rank receives the full united object). */
ptyger_status ptyger_get_object(ptyger_ctx* ctx, float* out);

/* Last computed gradient grad F(psi_{m-1}) (H*W complex64, zero before the first
 * iteration).  Collective when world > 1. */
ptyger_status ptyger_get_gradient(ptyger_ctx* ctx, float* out);

/* Cached far field u = G psi_m (n*N*N complex64, frames in input order) of the frames this
 * rank owns (all frames when world = 1), for parity tests.  The cache lags psi by the last
 * accepted gamma v (R#11); this call first folds that update in on the device (the same
 * fp32 fma the next GRAD stage would apply, which then skips it), so the result is G psi_m
 * of ptyger_get_object's psi_m and the iteration sequence is unchanged. */
ptyger_status ptyger_get_farfield(ptyger_ctx* ctx, float* out);

/* Teacher-forcing state: psi_m, grad F(psi_{m-1}), eta_{m-1} (H*W complex64 each), the
 * cached F(psi_m) and m.  get_state: any pointer may be NULL.  set_state uploads
 * (psi, g_prev, eta_prev, m), recomputes u = G psi and F(psi) by definition on the
 * device; g_prev / eta_prev are ignored when m == 0.  World == 1 only (E_STATE otherwise). */
ptyger_status ptyger_get_state(ptyger_ctx* ctx, float* psi, float* g_prev, float* eta_prev,
                               double* F, int32_t* m);
ptyger_status ptyger_set_state(ptyger_ctx* ctx, const float* psi, const float* g_prev,
                               const float* eta_prev, int32_t m);

/* DeltaF_k = F(psi + gamma_k eta) - F(psi) for the trials k = 0..K-1 the last iteration's
 * line search evaluated (difference form), and (bound, nullable) the error bound
 * of each value: > 0 for a screened value (MUFU log2, decision certified outside the bound),
 * 0 for an exact re-evaluation (accurate log1p).  Entries beyond the evaluated trials are NaN.
 * Returns the number evaluated in *n_eval (nullable). */
ptyger_status ptyger_get_ls_partials(ptyger_ctx* ctx, double* dF, double* bound, int32_t K, int32_t* n_eval);

/* Device-measured durations of the two frame kernels, summed over every launch since the last
 * reset: ms[0] / count[0] the GRAD-stage frame kernel (k_grad), ms[1] / count[1] the LS pass-0
 * frame kernel (k_ls).  One launch = max CTA end - min CTA start on the GPU's global nanosecond
 * timer, recorded by the kernels themselves, so the numbers cover graph-launched iterations
 * (ptyger_cg_iterate) exactly as they ran.  reset != 0 zeroes the sums after reading. */
ptyger_status ptyger_kernel_times(ptyger_ctx* ctx, double* ms, int32_t* count, int32_t reset);

/* Host-only helpers (no GPU needed) --------------------------------------------------- */

/* Integer stripe partition (R#18; PAPER.md:493-503 workload distribution).
 *   frame_rank  n int32: rank owning each frame (by centre row r_j + N/2).
 *   rows        P*6 int64: own_lo, own_hi, ext_lo, ext_hi, store_lo, store_hi per rank.
 * Returns E_ARG if a stripe's centre-row height is < N (message states the largest
 * feasible P), E_DATA for a window out of bounds. */
ptyger_status ptyger_partition(const int32_t* scan, int64_t n, int64_t H, int32_t N, int32_t P,
                               int32_t* frame_rank, int64_t* rows);

/* ptyger_partition for fractional positions (R#22): rows by the integer corners floor(x) and,
 * when any fraction is nonzero, ext_hi = min(max owned floor(row) + N + 1, H) (the bilinear
 * window's footprint).  scan: n*(row, col) float32.  Errors as ptyger_partition. */
ptyger_status ptyger_partition_subpixel(const float* scan, int64_t n, int64_t H, int32_t N, int32_t P,
                                        int32_t* frame_rank, int64_t* rows);

/* Float scan positions (Alg.1 'float32 h_s') -> int32 corners, round half-up
 * in double: floor((double)x + 0.5) (R#3).  raw and out hold 2*n values. */
ptyger_status ptyger_round_positions(const float* raw, int64_t n, int32_t* out);

/* Device helpers ------------------------------------------------------------------------ */

/* The library's batched unitary 2-D FFT on DEVICE buffers (cross-check against cuFFT):
 * batch frames of N*N complex64, forward (inverse = 0, e^{-i}) or inverse (e^{+i}), 1/N scale.
 * stream is a cudaStream_t (NULL = default stream).  N in {16, 32, 64, 128, 256}. */
ptyger_status ptyger_fft2(const float* in, float* out, int32_t N, int64_t batch, int32_t inverse,
                          void* stream);

/* 128-byte NCCL unique id for world > 1 (rank 0 creates, all ranks pass it in config). */
ptyger_status ptyger_nccl_unique_id(void* out128);

/* Context-owned message for the last error (valid until the next call on ctx); with
 * ctx == NULL the calling thread's last init / helper error. */
const char* ptyger_last_error(const ptyger_ctx* ctx);

/* Device time (ms, CUDA events on the context's stream) of the last ptyger_cg_iterate call,
 * from before its first graph launch to after its last. */
float ptyger_last_iterate_ms(const ptyger_ctx* ctx);

/* Measured FP32 FMA-pipe peak of `device` in TFLOP/s (the FP32 roofline of the lower
 * bound t_min): a microbenchmark kernel of independent fma chains on every SM, 2 flop per FMA lane-op,
 * best of three timed launches.  paired != 0: Blackwell's paired FFMA2 (fma.rn.f32x2, the form the
 * frame kernels use), else scalar FFMA.  Runs on the legacy default stream of `device` and makes it
 * current.  Errors: E_ARG (null), E_CUDA (no such device / launch failure). */
ptyger_status ptyger_fp32_peak(int32_t device, int32_t paired, double* tflops);

/* Number of kernel launches the last ptyger_cg_iterate call issued (graph nodes counted). */
int64_t ptyger_kernel_launches(const ptyger_ctx* ctx);

void ptyger_destroy(ptyger_ctx* ctx);

const char* ptyger_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PTYGER_H */
