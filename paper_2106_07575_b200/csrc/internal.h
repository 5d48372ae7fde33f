// Internal declarations shared by the kernels (kernels.cu) and the host runtime (ctx.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ptyger.h"

namespace pty {

constexpr int KC = 16;       // LS trial capacity of one pass over the frames
constexpr int KMIN = 4;      // smallest adaptive pass-0 trial count
constexpr int SMAX = 64;     // max trials per iteration (max_shrinks bound)
constexpr int NDY = 7;       // DY partial sums per tile (+ Re<g, g_prev> for Polak-Ribiere)
constexpr int LSP = KC + 4;  // screening partials: [S_0..S_{KC-1} | A, D, sum|a|, sum b]
constexpr int LSW = LSP + 4; // reduced LS vector in DevState: + ||eta||^2 and the object-grid moments
constexpr int LS_ETA = LSP;  // ||eta||^2 over owned rows
constexpr int LS_QA = LSP + 1, LS_QB = LSP + 2, LS_QC = LSP + 3;   // sum I 2Re(psi* eta), I|eta|^2, I|psi|^2

// Device-resident scalar state of the iteration (all decisions are taken on the device).
struct DevState {
    double F;                // F(psi_m) (cached accepted value, R#11)
    double gamma;            // gamma of the last accepted step (u <- u + gamma v in k_grad)
    double alpha_re, alpha_im;
    double dy[NDY];          // reduced: |g|^2, Re/Im <eta,g-g_prev>, |g_prev|^2, Re/Im <eta,g>
    double ls_pass[LSW];     // reduced LS partials of the current pass (+ ||eta||^2 at LS_ETA)
    double ls_hist[SMAX];    // DeltaF_k of every trial evaluated this iteration
    double ls_bnd[SMAX];     // error bound of ls_hist (0 = exact evaluation)
    double eta2;             // ||eta_m||^2 over owned rows (global after reduction)
    // object-grid moments of this iteration's line (SolverCfg::qg): qa = sum_px a = sum_rho I 2 Re(psi* eta),
    // qb = sum_px |v|^2 = sum_rho I |eta|^2, qc = sum_px |u|^2 = sum_rho I |psi|^2 (G^H G = diag I)
    double qa, qb, qc;
    double F_init_part;      // scratch for k_fwd reductions
    int m;                   // iteration counter
    int accepted;            // 1 once a trial was accepted in this iteration
    int kstar;               // accepted trial index
    int n_eval;              // trials evaluated this iteration
    int restarted;
    int stalled;
    int numeric_error;       // 0 = ok; else stage code (1 DIR, 2 LS, 3 F)
    int err_iter;
    int keff;                // trials of LS pass 0 this iteration (adaptive: k*_prev + 3 in [KMIN, K])
    int need_exact;          // pass + 1 when the screening pick left that pass undecided
    int k_unc;               // first undecided trial
    int n_exact;             // exact re-evaluations so far (diagnostic)
    int n_pass, n_xpass;     // LS passes over the frames this iteration: screening, exact
    // device-side kernel timers (globaltimer ns) of the two frame kernels, [0] GRAD, [1] LS pass 0:
    // first CTA start / last CTA end of the current launch, folded into sums by k_begin_iter
    unsigned long long tk_start[2], tk_end[2];
    // peer-memory transport (world > 1, PTYGER_TRANSPORT_P2P): per-channel epochs (start at 1, the
    // windows' flags at 0) and grid-completion counters of the put kernels
    unsigned long long p2p_epoch[4];
    unsigned int p2p_done[4];
    double tk_sum_ms[2];
    int tk_cnt[2];
    // per-stage device timestamps of the current iteration (globaltimer ns): [0] begin, [1] GRAD frame
    // kernels + adjoint done, [2] DIR done, [3] LS done, [4] update done, [5] adjoint done before the
    // band exchange (world > 1); the final stamp folds them into the iteration's trace entry
    unsigned long long stamp[6];
    int trace_written;       // pick_body wrote this iteration's trace entry (slot trace_idx - 1)
    int trace_idx;           // slot of the current iteration in the trace buffer
    int trace_cap;           // capacity of trace_ptr
    ptyger_trace* trace_ptr; // device trace buffer of the current ptyger_cg_iterate call
};

struct Geometry {
    int N;
    int64_t W;               // object width (all ranks store full-width rows)
    int64_t SH;              // storage rows on this rank
    int64_t own_lo, own_hi;  // owned rows, storage-local coordinates (for reductions)
    int64_t band_lo0, band_hi0, band_lo1, band_hi1;  // storage-local band rows excluded from k_adj partials
    int64_t n_local;         // frames stored on this rank
    int est;                 // estimator (PTYGER_EST_ML / PTYGER_EST_LS) for the residual and F terms
    const float2* frac;      // per storage frame (row, col) fractional offsets of a bilinear window
                             // (R#22, ptyger_init_subpixel); nullptr = integer positions
};

struct SolverCfg {
    double gamma0, tau, t, eps;
    int max_shrinks, direction, K;   // K = trials per extra pass and cap of the adaptive pass 0 (<= KC)
    int est;                         // PTYGER_EST_ML / PTYGER_EST_LS
    // 1: the non-log part q_k = gamma_k a + gamma_k^2 b of the LS trial sums comes from the object grid
    // (qa, qb of DevState; Parseval + G^H G = diag(I), exact for integer positions) instead of per frame
    // pixel moments.  Set for the Poisson ML estimator with integer positions.
    int qg;
    int kadd;                        // adaptive pass-0 trials: keff = k*_prev + kadd (clamped to [KMIN, K])
    int side;                        // N = 256: per mille of the frames for the LS side kernel (0 = off)
};

// Trials [base, base + count) evaluated by LS pass p (host and device agree on this rule): pass 0
// the adaptive keff = k*_prev + 3; pass 1 (k* jumped past keff, usually by a few) the next
// K1 = min(K, 8) trials; later passes K each.  A pass over (u, v, d) costs a full read of the far
// fields plus, per d > 0 pixel, a MUFU log per trial: 16 trials made the large view's pass 1
// compute-bound (28.7 ms, ALU 53 %, MUFU 39 %, DRAM 56 %).
__host__ __device__ inline int ls_k1(const SolverCfg& c) { return c.K < 8 ? c.K : 8; }
__host__ __device__ inline void ls_pass_range(int pass, int keff, const SolverCfg& c, int& base, int& count) {
    const int k1 = ls_k1(c);
    base = pass == 0 ? 0 : pass == 1 ? keff : keff + k1 + (pass - 2) * c.K;
    count = pass == 0 ? keff : pass == 1 ? k1 : c.K;
    if (base + count > c.max_shrinks) count = c.max_shrinks - base;
    if (count < 0) count = 0;
}

// -------- kernel launchers (kernels.cu) ------------------------------------------------
int launch_fft2(const float2* in, float2* out, int N, int64_t batch, bool inverse, cudaStream_t s);
int launch_fwd(const Geometry& g, const float2* psi, const float2* probe, const int2* pos,
               const int* order, const float* d, float2* u, double* part, int grid, float eps,
               cudaStream_t s);
// probe_s = probe / N (power-of-two scale, exact): the unitary 1/N of the FFTs rides on the probe
int launch_grad(const Geometry& g, float2* u, float2* v, const float* d, const float2* probe,
                const float2* probe_s, const DevState* st, float eps, int grid, cudaStream_t s);
int launch_grad256(const Geometry& g, float2* u, float2* v, const float* d, const float2* probe, const DevState* st,
                   float eps, int grid, cudaStream_t s);
int launch_fwd256(const Geometry& g, const float2* psi, const float2* probe, const int2* pos, const int* order,
                  const float* d, float2* u, double* part, int grid, float eps, cudaStream_t s);
int launch_fft2_256(const float2* in, float2* out, int64_t batch, bool inv, cudaStream_t s);
struct P2PView;
// pv (peer-memory transport): band rows are also stored into the neighbours' windows and the band
// flags raised by the kernel's last tile (fused compute + exchange); nullptr otherwise
int launch_adj(const Geometry& g, const float2* y, const int* tile_ptr, const int* tile_frames,
               int ntx, int nty, float2* gcur, const float2* gprev, const float2* eta, double* part,
               const DevState* st, cudaStream_t s, const P2PView* pv = nullptr);
int launch_ls(const Geometry& g, const float2* eta, const float2* probe, const float2* probe_s, const int2* pos,
              const int* order, const float2* u, float2* v, const float* d, const SolverCfg& c,
              double* part, int grid, const DevState* st, cudaStream_t s);
int launch_lsx(const Geometry& g, const float2* u, const float2* v, const float* d,
               const SolverCfg& c, int pass, bool exact, double* part, int grid, const DevState* st,
               cudaStream_t s);
struct P2PView;
// step to run at the end of a reduction kernel: on = 1 the LS decision (k_pick), 2 the DIR step (k_dir)
struct PickArgs {
    int on, pass, exact, last;
    SolverCfg c;
};
// mode 0: always; 1: only while no LS trial is accepted; 2: only when pass `pass` needs its exact pass.
// pv (peer-memory transport, st required): the rank-ordered sum over ranks follows in the same kernel.
// pick: the LS decision of the pass follows in the same kernel (it also runs when the reduction is skipped).
int launch_reduce(const double* part, int nblocks, int width, double* dst, cudaStream_t s,
                  const DevState* st = nullptr, int mode = 0, int pass = 0, const P2PView* pv = nullptr,
                  const PickArgs* pick = nullptr);
int launch_dir(DevState* st, const SolverCfg& c, cudaStream_t s);
// illum = I(rho) = sum_j |p(rho - s_j)|^2 over this rank's frames (tile CSR, canonical order)
int launch_illum(const Geometry& g, const float2* probe, const int* tile_ptr, const int* tile_frames, int ntx, int nty,
                 float* illum, cudaStream_t s);
// psi, illum non-null (SolverCfg::qg): also the object-grid moments qa, qb, qc (partials [eta2, qa, qb, qc])
int launch_eta(const Geometry& g, const float2* gcur, float2* eta, const float2* psi, const float* illum,
               const DevState* st,
               double* part, int grid, cudaStream_t s);
int launch_pick(DevState* st, const SolverCfg& c, int pass, int exact_mode, int last_pass, cudaStream_t s);
int launch_upd(const Geometry& g, float2* psi, const float2* eta, const DevState* st, int grid,
               cudaStream_t s);
int launch_begin_iter(DevState* st, cudaStream_t s);
// stage timestamp `slot` (see DevState::stamp); slot 4 also writes the stage ms into the trace entry
int launch_stamp(DevState* st, int slot, cudaStream_t s);
int launch_timers(DevState* st, double* out, int reset, cudaStream_t s);
int launch_fold(const Geometry& g, float2* u, const float2* v, DevState* st, int grid, cudaStream_t s);
int launch_validate_d(const float* d, int64_t count, int64_t frame_elems, unsigned long long* bad,
                      cudaStream_t s);
// init: d >= 0 / finite check fused with the F(psi_0) partials over u_0 (part[grid])
int launch_f0_validate(const float2* u, const float* d, int64_t count, int64_t frame_elems, unsigned long long* bad,
                       double* part, int grid, float eps, int est, cudaStream_t s);
int launch_set_F(DevState* st, const double* src, int keff0, cudaStream_t s);
// FP32 FMA-pipe peak of `device` in TFLOP/s (kernels_peak.cu), paired FFMA2 or scalar FFMA; < 0 on error
double measure_fp32_peak(int device, bool paired);
// warp-specialised LS pass 0 for N = 128 (kernels_ls128.cu): FFT group + epilogue group, TMEM hand-off
int launch_ls_ws(const Geometry& g, const float2* eta, const float2* probe_s, const int2* pos, const int* order,
                 const float2* u, float2* v, const float* d, const SolverCfg& c, double* part, int grid,
                 const DevState* st, cudaStream_t s);
// cluster-of-four frame kernels for N = 256 (kernels_c256.cu); probe_s = probe / N
int c256_ls_parts(int64_t nfr, int side);
int c256_ls_side(int64_t nfr, int side);   // CTAs of the concurrent side kernel (0: none)
int launch_ls_c256(const Geometry& g, const float2* eta, const float2* probe_s, const int2* pos, const int* order,
                   const float2* u, float2* v, const float* d, const SolverCfg& c, double* part, const DevState* st,
                   cudaStream_t s);
// LS pass 0 for N = 256 on the SMs the clusters leave idle, frames [i0, n_local) of the canonical order,
// concurrent with k_ls_c256ws (programmatic dependent launch); part: its first partial row (kernels_n256.cu)
int launch_ls256_side(const Geometry& g, const float2* eta, const float2* probe_s, const int2* pos, const int* order,
                      const float2* u, float2* v, const float* d, const SolverCfg& c, double* part, const DevState* st,
                      int64_t i0, int grid, cudaStream_t s);
int launch_scale_c(const float2* in, float2* out, int64_t n, float s, cudaStream_t st);
int launch_band_add(float2* gcur, const float2* recv, int64_t row_lo, int64_t rows, int64_t W,
                    const float2* gprev, const float2* eta, int64_t own_lo, int64_t own_hi,
                    double* part, int grid, cudaStream_t s);

}  // namespace pty
