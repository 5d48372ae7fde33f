// Device helpers shared by the libptyger kernels: reductions, the Poisson residual and the
// line-search (LS) pixel terms.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fft.cuh"
#include "internal.h"

namespace pty {

#define FULLMASK 0xffffffffu

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(FULLMASK, v, m);
    return v;
}

// Block sum in fixed order (deterministic).  All threads must call; result valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sred) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) sred[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NT / 32; ++i) s += sred[i];
    }
    return s;
}

template <int K>
struct Log2 {
    static constexpr int value = (K <= 1) ? 0 : 1 + Log2<K / 2>::value;
};
template <>
struct Log2<1> {
    static constexpr int value = 0;
};

// Warp reduce-scatter of K (power of two <= 32) per-lane values: afterwards every lane holds
// the warp total of entry  lane >> (5 - log2 K).
template <int K>
__device__ __forceinline__ double warp_reduce_scatter(double (&v)[K], int lane) {
    constexpr int P = Log2<K>::value;
#pragma unroll
    for (int s = 0; s < P; ++s) {
        const int h = K >> (s + 1);
        const int m = 16 >> s;
        const bool upper = (lane & m) != 0;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const double send = upper ? v[i] : v[i + h];
            const double keep = upper ? v[i + h] : v[i];
            v[i] = keep + __shfl_xor_sync(FULLMASK, send, m);
        }
    }
    double r = v[0];
#pragma unroll
    for (int m = (32 >> P) >> 1; m >= 1; m >>= 1) r += __shfl_xor_sync(FULLMASK, r, m);
    return r;
}

__device__ __forceinline__ float2 ldg2(const float2* p) { return __ldg(p); }
// streamed reads that should not displace the frame-invariant probe / window data from L1
__device__ __forceinline__ float2 ldg2_na(const float2* p) {
    float2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ float ldg1_na(const float* p) {
    float r;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
    return r;
}

// L2 cache-policy hints (createpolicy + .L2::cache_hint): keep short-lived intermediates (the N = 256
// slot transpose) resident, stream data that is read or written once per pass.
__device__ __forceinline__ uint64_t l2_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st2_hint(float2* a, float2 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(a), "f"(v.x), "f"(v.y), "l"(pol) : "memory");
}
__device__ __forceinline__ float2 ld2_hint(const float2* a, uint64_t pol) {
    float2 v;
    asm volatile("ld.global.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(v.x), "=f"(v.y) : "l"(a), "l"(pol));
    return v;
}
// streamed (read-once, fully coalesced) loads: L2 policy + no L1 allocation
__device__ __forceinline__ float2 ld2_hint_na(const float2* a, uint64_t pol) {
    float2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;"
                 : "=f"(v.x), "=f"(v.y) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld1_hint_na(const float* a, uint64_t pol) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld1_hint(const float* a, uint64_t pol) {
    float v;
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
    return v;
}

// Frame-kernel timers (DevState::tk_*): thread 0 of every CTA marks its start / end with the
// global nanosecond timer, so one launch's duration is max(end) - min(start) over its CTAs.
// The timer words are the only DevState fields these kernels write (hence the const_cast).
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void ktime_start(const DevState* st, int i) {
    if (threadIdx.x == 0) atomicMin(const_cast<unsigned long long*>(&st->tk_start[i]), gtimer());
}
__device__ __forceinline__ void ktime_end(const DevState* st, int i) {
    if (threadIdx.x == 0) atomicMax(const_cast<unsigned long long*>(&st->tk_end[i]), gtimer());
}

// Row-pass input of a window: x[n1] = p[row, T n1 + t] * psi~(s + (row, T n1 + t)).
// Integer positions (R#3): psi~ = psi.  Fractional positions (R#22, g.frac set): psi~ is the bilinear
// interpolation at (s.x + fy + row, s.y + fx + col):
//     (1 - fy) [(1 - fx) psi[r, c] + fx psi[r, c + 1]] + fy [(1 - fx) psi[r + 1, c] + fx psi[r + 1, c + 1]].
// A +1 tap past the last stored row / column only occurs with weight 0 (init validation and the
// partition's N + 1 footprint) and is clamped in bounds.
template <int R, int T>
__device__ __forceinline__ void window_row(const float2* __restrict__ obj, const Geometry& g, int2 s, int64_t j,
                                           int row, int t, const float2* __restrict__ pp, float2 (&x)[R]) {
    const float2* src = obj + (int64_t)(s.x + row) * g.W + s.y + t;
    if (!g.frac) {
#pragma unroll
        for (int n1 = 0; n1 < R; ++n1) x[n1] = cmul(ldg2(pp + T * n1), ldg2(src + T * n1));
        return;
    }
    const float2 fr = g.frac[j];
    const float wy0 = 1.0f - fr.x, wy1 = fr.x, wx0 = 1.0f - fr.y, wx1 = fr.y;
    const int64_t dn = ((int64_t)s.x + row + 1 < g.SH) ? g.W : 0;
#pragma unroll
    for (int n1 = 0; n1 < R; ++n1) {
        const int dc = ((int64_t)s.y + t + T * n1 + 1 < g.W) ? 1 : 0;
        const float2* q = src + T * n1;
        const float2 a = ldg2(q), b = ldg2(q + dc), c = ldg2(q + dn), e = ldg2(q + dn + dc);
        const float2 top = make_float2(fmaf(wx1, b.x, wx0 * a.x), fmaf(wx1, b.y, wx0 * a.y));
        const float2 bot = make_float2(fmaf(wx1, e.x, wx0 * c.x), fmaf(wx1, e.y, wx0 * c.y));
        x[n1] = cmul(ldg2(pp + T * n1), make_float2(fmaf(wy1, bot.x, wy0 * top.x), fmaf(wy1, bot.y, wy0 * top.y)));
    }
}

// gamma_k = gamma0 tau^k by repeated multiplication in double: exactly the trial sequence of
// Eq.7's backtracking (gamma <- gamma tau, Alg.1 662) and of the oracle's line_search.
__device__ __forceinline__ double trial_gamma(double gamma0, double tau, int k) {
    double g = gamma0;
    for (int i = 0; i < k; ++i) g *= tau;
    return g;
}

// Residual of Eq.3: u - d/u^* = u - d u / |u|^2, quotient dropped where |u| < eps (R#4).
// Least-squares estimator (R#19): u - sqrt(d) u / |u|.
__device__ __forceinline__ float2 residual(float2 u, float dd, float eps2, int est = PTYGER_EST_ML) {
    const float c = u.x * u.x + u.y * u.y;
    if (c >= eps2) {
        // d / c to <= 1 ulp (MUFU reciprocal + one Newton correction of the quotient): where |u| is
        // small and d > 0 the residual is ill-conditioned and a 2-ulp approximate
        // quotient measurably inflated the gradient error; __fdiv_rn's slow-path call cost the
        // GRAD kernel 18 %.  c >= eps^2 = 1e-32 is a normal float, so the FTZ reciprocal is exact
        // to 1 ulp over the whole guarded range.
        float r;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(c));
        float s = dd * r;
        s = fmaf(fmaf(-c, s, dd), r, s);
        if (est == PTYGER_EST_LS) s = __fsqrt_rn(s);
        return make_float2(u.x - s * u.x, u.y - s * u.y);
    }
    return u;
}

// Per-pixel objective term: Eq.2 c - d log c (Poisson ML) or (|u| - sqrt d)^2 (LS estimator).
__device__ __forceinline__ float objective_term(float c, float dd, float eps2, int est) {
    if (est == PTYGER_EST_LS) {
        const float r = __fsqrt_rn(c) - __fsqrt_rn(dd);
        return r * r;
    }
    return c - dd * logf(fmaxf(c, eps2));
}

// ---------------------------------------------------------------------------------------------
// Line search pixel terms.  With u = G psi, v = G eta (Eq.1 linearity) the change of the Eq.2
// objective along eta at trial gamma is, per detector pixel,
//     t(gamma) = |u + gamma v|^2 - |u|^2 - d log(|u + gamma v|^2 / |u|^2)
//              = q - d log w,   q = gamma (a + gamma b),  w = |u + gamma v|^2 / |u|^2,
// a = 2 Re(u^* v), b = |v|^2, c = |u|^2 (oracle ls_delta).  Logs are guarded (R#4).
// ---------------------------------------------------------------------------------------------

// Accurate, branch-free float log1p for z > -1 (max rel err 1.7e-7 measured in fp32):
// w = 1 + z = m 2^e with m in [sqrt(1/2), sqrt(2)); the polynomial runs on z itself when e = 0
// (so the rounding of 1 + z is never used there), otherwise on m - 1.  log1p(x) = x + x^2 P(x),
// P a degree-8 Chebyshev fit on [sqrt(1/2)-1, sqrt(2)-1].  No MUFU, no branch.
__device__ __forceinline__ float log1p_poly(float z) {
    const float w = 1.0f + z;
    const int iw = __float_as_int(w);
    const int e = (iw - 0x3f3504f3) >> 23;
    const float m = __int_as_float(iw - (e << 23));
    const float x = (e == 0) ? z : (m - 1.0f);
    float P = -0.07764425f;
    P = fmaf(P, x, 0.12656558f);
    P = fmaf(P, x, -0.13065042f);
    P = fmaf(P, x, 0.14209557f);
    P = fmaf(P, x, -0.1663307f);
    P = fmaf(P, x, 0.20001242f);
    P = fmaf(P, x, -0.25000605f);
    P = fmaf(P, x, 0.33333328f);
    P = fmaf(P, x, -0.49999997f);
    const float ef = __int_as_float(e + 0x4B400000) - 12582912.0f;  // (float)e on the FMA pipe
    return fmaf(ef, 0.693147182464599609375f, fmaf(x * x, P, x));
}

// Guarded exact definition, used where |u| < eps or |u + gamma v| < eps or 1 + z underflows.
// qg: the log part only (the non-log part q comes from the object grid, SolverCfg::qg).
static __device__ __noinline__ float ls_term_slow(float a, float b, float c, float dd, float gam, float eps2,
                                                  bool qg) {
    const float q = gam * fmaf(gam, b, a);
    const float cn = c + q;
    if (c >= eps2 && cn >= eps2) {
        const float z = q / c;
        if (z > -0.999f) return qg ? -dd * log1p_poly(z) : fmaf(-dd, log1p_poly(z), q);
    }
    const float lg = -dd * (logf(fmaxf(cn, eps2)) - logf(fmaxf(c, eps2)));
    return qg ? lg : (cn - c) + lg;
}

// Least-squares estimator terms t = q (1 - 2 sqrt(d) / (|u + g v| + |u|)), q = |u + g v|^2 - |u|^2
// with correctly rounded sqrt / reciprocal (a few ulp per term, no transcendental approximation).
template <int KT, int K, typename G>
__device__ __forceinline__ void ls_screen_lse(float2 uu, float2 vv, float dd, const G& sgam, float (&S)[K]) {
    const float c = fmaf(uu.x, uu.x, uu.y * uu.y);
    const float sc = __fsqrt_rn(c), sd2 = 2.0f * __fsqrt_rn(dd);
#pragma unroll
    for (int k = 0; k < KT; ++k) {
        const float gam = sgam[k];
        const float ex = fmaf(gam, vv.x, uu.x), ey = fmaf(gam, vv.y, uu.y);
        const float cn = fmaf(ex, ex, ey * ey);
        const float q = cn - c;
        const float den = __fsqrt_rn(cn) + sc;
        S[k] += (den > 0.f) ? fmaf(-q, sd2 * __frcp_rn(den), q) : q;
    }
}

// EXACT terms (accurate log1p, ~1.7e-7 relative): t_k = q_k - d log1p(q_k / c).  Branch-free
// fast path; a lane needing the guarded definition sends its warp through ls_term_slow.
// KT trials (compile time) accumulate into acc[0..KT).
template <int KT, bool LSE, bool QG, int K>
__device__ __forceinline__ void ls_exact(float2 uu, float2 vv, float dd, const float* sgam, float eps2,
                                         float (&acc)[K]) {
    static_assert(KT <= K, "trial count above capacity");
    if constexpr (LSE) {   // least-squares estimator: the screening formula is already exact
        ls_screen_lse<KT>(uu, vv, dd, sgam, acc);
        return;
    }
    const float a = 2.0f * fmaf(uu.x, vv.x, uu.y * vv.y);
    const float b = fmaf(vv.x, vv.x, vv.y * vv.y);
    const float c = fmaf(uu.x, uu.x, uu.y * uu.y);
    bool bad = !(c >= eps2);
    const float rc = bad ? 0.0f : 1.0f / c;
    float t[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) {
        const float gam = sgam[k];
        const float q = gam * fmaf(gam, b, a);
        const float z = q * rc;
        bad |= (c + q < eps2) | (z <= -0.999f);
        t[k] = QG ? -dd * log1p_poly(fmaxf(z, -0.999f)) : fmaf(-dd, log1p_poly(fmaxf(z, -0.999f)), q);
    }
    if (__any_sync(__activemask(), bad)) {
        if (bad) {
#pragma unroll
            for (int k = 0; k < KT; ++k) t[k] = ls_term_slow(a, b, c, dd, sgam[k], eps2, QG);
        }
    }
#pragma unroll
    for (int k = 0; k < KT; ++k) acc[k] += t[k];
}

// SCREENING terms.  cn = |u + gamma v|^2 is formed from the components of u + gamma v (each an
// fma of exact inputs, correctly rounded), so w = cn / c keeps a few-ulp RELATIVE accuracy even
// when u + gamma v nearly cancels; log2 w on the MUFU without denormal fix-up (lg2.approx.ftz:
// |abs err| <= 2^-22 on [0.5, 2], 2 ulp relative elsewhere).  The non-log part q_k = gamma_k a +
// gamma_k^2 b (a = 2 Re(u* v), b = |v|^2) enters through per-pixel moments (LsQState).  Per
// trial: 7 FMA-pipe ops, 1 ALU op, 1 MUFU.  The caller also accumulates A = sum d max_k |ln w_k|,
// D = sum (d + 0.12 c), sum |a|, sum b, which bound the error of every trial of the pass:
//     |S_k - t_exact| <= LS_EPS_D D + LS_EPS_R (A + gamma_k sum|a| + gamma_k^2 sum b)
// (the 0.12 c part of D covers the rounding of the q moments: 2e-6 * 0.12 = 2.4e-7 >= 2 * 2^-23).
// |u| < eps makes w = 0 -> S non-finite -> the exact pass decides (guarded definition, R#4).
constexpr double LS_EPS_D = 2e-6;
constexpr double LS_EPS_R = 2e-6;

__device__ __forceinline__ float lg2_ftz(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Per-thread moments of the screening bound.  sa2 = sum |a| / 2 (a / 2 = Re(u* v) is what the
// pixel loop forms; ls_run_out doubles it).
struct LsMom {
    float A = 0.f, D = 0.f, sa2 = 0.f, sb = 0.f;
};

// ---------------------------------------------------------------------------------------------
// Sparse-data screening.  Poisson counts are 0 on most detector pixels (59 % at the bench
// workload), and where d = 0 the log term vanishes EXACTLY: t_k = q_k = gamma_k a + gamma_k^2 b,
// so those pixels only add to two moments (za, zb) folded into S_k at the end.  The d > 0 pixels
// are compacted per warp into a shared-memory queue (ballot + popc; u, v as one 16-B entry, d as a
// second word) and screened in full 32-lane batches, so the per-trial MUFU/FMA work scales with
// the nonzero fraction.  The queue is linear: a lane's NP pixels of one push land at
// pending + prefix, full batches are screened from the front and the (< 32) remainder moves
// to the front, so no wrap arithmetic is needed; capacity 31 + 32 NP entries.
// All 32 lanes must call ls_push / ls_flush together (inactive lanes push zeros).
// ---------------------------------------------------------------------------------------------
template <int NP>
struct LsWarpQ {
    static constexpr int CAP = 31 + 32 * NP;
    float4 uv[CAP];
    float d[CAP];
};

// LSE = false: Poisson ML terms (screened, MUFU log2).  LSE = true: least-squares estimator terms
// t = q (1 - 2 sqrt(d) / (|u + g v| + |u|)) with correctly rounded sqrt / reciprocal: a few ulp per
// term, no transcendental approximation, so A stays 0 and the bound reduces to its rounding part.
//
// ML: cn = |u + gamma v|^2 is formed from the components of u + gamma v (each an fma of exact
// inputs, correctly rounded), so w = cn / c keeps a few-ulp RELATIVE accuracy even when u + gamma v
// nearly cancels (a pre-scaled u / |u| would lose it).
template <int KT, bool LSE, bool QG, int K, typename G>
__device__ __forceinline__ void ls_screen_nz(float4 uv, float dd, const G& sgam, float eps2, float (&S)[K],
                                             LsMom& m) {
    const float2 uu = make_float2(uv.x, uv.y), vv = make_float2(uv.z, uv.w);
    if constexpr (LSE) {
        ls_screen_lse<KT>(uu, vv, dd, sgam, S);
    } else {
        const float c = fmaf(uu.x, uu.x, uu.y * uu.y);
        // |u| < eps: rc = 0, w = 0, log2 = -inf, a non-finite S and therefore the exact pass, which
        // applies the guarded definition R#4 (as does an FTZ underflow of w)
        const float rc = (c >= eps2) ? __fdividef(1.0f, c) : 0.0f;
        const float dl = dd * 0.693147182464599609375f;
        if (QG) m.D += dd;   // the bound's D = sum d (no q-moment rounding to cover)
        float amax = 0.f;
        // Trials run in pairs on the paired FP32 pipe (FFMA2 / FMUL2: per lane the same fp32
        // operations as the scalar form).
#pragma unroll
        for (int k = 0; k + 1 < KT; k += 2) {
            const float2 g2 = make_float2(sgam[k], sgam[k + 1]);
            const float2 ex = fma2(g2, bc2(vv.x), bc2(uu.x));
            const float2 ey = fma2(g2, bc2(vv.y), bc2(uu.y));
            const float2 w = mul2(fma2(ex, ex, mul2(ey, ey)), bc2(rc));
            const float L0 = lg2_ftz(w.x), L1 = lg2_ftz(w.y);
            const float2 s2 = fma2(bc2(-dl), make_float2(L0, L1), make_float2(S[k], S[k + 1]));
            S[k] = s2.x;
            S[k + 1] = s2.y;
            amax = fmaxf(amax, fmaxf(fabsf(L0), fabsf(L1)));
        }
        if constexpr (KT & 1) {
            constexpr int k = KT - 1;
            const float gam = sgam[k];
            const float ex = fmaf(gam, vv.x, uu.x), ey = fmaf(gam, vv.y, uu.y);
            const float L2 = lg2_ftz(fmaf(ex, ex, ey * ey) * rc);
            S[k] = fmaf(-dl, L2, S[k]);
            amax = fmaxf(amax, fabsf(L2));
        }
        m.A = fmaf(dl, amax, m.A);
    }
}

// za2, zb: per lane sums of a / 2, b.  Poisson ML: over ALL pixels (q_k = gamma_k a + gamma_k^2 b is
// the whole non-log part of t_k, so the d > 0 screening only adds -d ln w_k).  Its rounding is
// inside the screening bound: gamma |err a| <= 2^-23 (c + gamma^2 b) (AM-GM on 2|u||v|), covered
// by the 0.12 c part of D and the gamma^2 sum b term.  LS estimator: over the d = 0 pixels only
// (its d > 0 term is not separable).
struct LsQState {
    int pending = 0;   // warp-uniform queue fill
    float za2 = 0.f, zb = 0.f;
};

// Elements [O, O + M) of a register array as an array reference (for fixed-width pushes).
template <int O, int M, typename E, int N>
__device__ __forceinline__ E (&slice(E (&a)[N]))[M] {
    static_assert(O + M <= N, "slice out of range");
    return *reinterpret_cast<E(*)[M]>(a + O);
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

// Screen every full batch of 32 queued pixels; move the remainder to the front of the queue.
template <int KT, bool LSE, bool QG, int QN, int K, typename G>
__device__ __forceinline__ void ls_drain_full(LsWarpQ<QN>& q, LsQState& qs, const G& sgam, float eps2,
                                              float (&S)[K], LsMom& m, int lane) {
    __syncwarp();
    int b = 0;
#pragma unroll 1
    for (; b + 32 <= qs.pending; b += 32) ls_screen_nz<KT, LSE, QG>(q.uv[b + lane], q.d[b + lane], sgam, eps2, S, m);
    const int rem = qs.pending - b;
    float4 tu = make_float4(0.f, 0.f, 0.f, 0.f);
    float td = 0.f;
    if (lane < rem) {
        tu = q.uv[b + lane];
        td = q.d[b + lane];
    }
    __syncwarp();
    if (lane < rem) {
        q.uv[lane] = tu;
        q.d[lane] = td;
    }
    __syncwarp();
    qs.pending = rem;
}

// Push NP pixels per lane (all lanes together) into a queue sized for QN >= NP.
// QG (SolverCfg::qg): no per-pixel moments at all (the non-log part and the bound's q terms come from the
// object grid); only the d > 0 compaction remains.
template <int KT, bool LSE, bool QG, int QN, int NP, int K, typename G>
__device__ __forceinline__ void ls_push(LsWarpQ<QN>& q, LsQState& qs, const float2 (&uu)[NP],
                                        const float2 (&vv)[NP], const float (&dd)[NP], const G& sgam, float eps2,
                                        float (&S)[K], LsMom& m, int lane) {
    static_assert(NP <= QN, "queue too small for the push width");
    const unsigned lt = lanemask_lt();
    int off = qs.pending;
#pragma unroll
    for (int e = 0; e < NP; ++e) {
        const float2 u = uu[e], v = vv[e];
        const bool nz = dd[e] != 0.0f;
        if constexpr (!QG) {
            const float a2 = fmaf(u.x, v.x, u.y * v.y);   // a / 2
            const float b = fmaf(v.x, v.x, v.y * v.y);
            const float c = fmaf(u.x, u.x, u.y * u.y);
            m.D += fmaf(0.12f, c, dd[e]);
            m.sa2 += fabsf(a2);
            if (LSE) m.sb += b;   // Poisson ML: sum b is zb (all pixels), folded in at ls_flush
            if (!LSE || !nz) {
                qs.za2 += a2;
                qs.zb += b;
            }
        }
        const unsigned mask = __ballot_sync(FULLMASK, nz);
        if (nz) {
            const int slot = off + __popc(mask & lt);
            q.uv[slot] = make_float4(u.x, u.y, v.x, v.y);
            q.d[slot] = dd[e];
        }
        off += __popc(mask);
    }
    qs.pending = off;
    if (off >= 32) ls_drain_full<KT, LSE, QG>(q, qs, sgam, eps2, S, m, lane);
}

// Drain the queue and fold the (za, zb) moments into S (call once per accumulation run).
template <int KT, bool LSE, bool QG, int QN, int K, typename G>
__device__ __forceinline__ void ls_flush(LsWarpQ<QN>& q, LsQState& qs, const G& sgam, float eps2, float (&S)[K],
                                         LsMom& m, int lane) {
    if (qs.pending > 0) {
        __syncwarp();
        if (lane < qs.pending) ls_screen_nz<KT, LSE, QG>(q.uv[lane], q.d[lane], sgam, eps2, S, m);
        qs.pending = 0;
        __syncwarp();
    }
    if constexpr (!QG) {
        const float za = 2.0f * qs.za2;
#pragma unroll
        for (int k = 0; k < KT; ++k) S[k] += sgam[k] * fmaf(sgam[k], qs.zb, za);
        if (!LSE) m.sb += qs.zb;
        qs.za2 = qs.zb = 0.f;
    }
}

// Warp reduce-scatter of the K per-lane fp32 trial sums in fp32 (5 rounding levels of 2^-24 relative
// to the sum of |partials|, inside the LS_EPS_R part of the bound); returns, as fp64, the warp total
// of entry lane >> (5 - log2 K).
template <int K>
__device__ __forceinline__ double warp_reduce_scatter_f(float (&v)[K], int lane) {
    constexpr int P = Log2<K>::value;
#pragma unroll
    for (int s = 0; s < P; ++s) {
        const int h = K >> (s + 1);
        const int msk = 16 >> s;
        const bool upper = (lane & msk) != 0;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const float send = upper ? v[i] : v[i + h];
            const float keep = upper ? v[i + h] : v[i];
            v[i] = keep + __shfl_xor_sync(FULLMASK, send, msk);
        }
    }
    float r = v[0];
#pragma unroll
    for (int msk = (32 >> P) >> 1; msk >= 1; msk >>= 1) r += __shfl_xor_sync(FULLMASK, r, msk);
    return (double)r;
}

// Fold one accumulation run (per-lane S, moments) into the thread's fp64 running totals.
template <int K>
__device__ __forceinline__ void ls_run_out(float (&S)[K], const LsMom& m, double& tot, double (&mom)[4], int lane) {
    tot += warp_reduce_scatter_f<K>(S, lane);
    mom[0] += (double)m.A;
    mom[1] += (double)m.D;
    mom[2] += 2.0 * (double)m.sa2;
    mom[3] += (double)m.sb;
}

// Run body.template operator()<KT, LSE, QG>() with KT = cnt (4..10) or cnt rounded up to an even count
// (<= 16): the trial count of a pass is uniform for the whole launch, so one branch at the top selects a
// fully unrolled variant and only its code is executed (instruction-cache footprint of one).
// Exact variants cover the adaptive pass-0 counts k*_prev + 3 around the typical k* = 4..7.
template <bool LSE, bool QG, typename F>
__device__ __forceinline__ void trial_dispatch_k(int cnt, F& body) {
    if (cnt <= 4)
        body.template operator()<4, LSE, QG>();
    else if (cnt == 5)
        body.template operator()<5, LSE, QG>();
    else if (cnt == 6)
        body.template operator()<6, LSE, QG>();
    else if (cnt == 7)
        body.template operator()<7, LSE, QG>();
    else if (cnt == 8)
        body.template operator()<8, LSE, QG>();
    else if (cnt == 9)
        body.template operator()<9, LSE, QG>();
    else if (cnt == 10)
        body.template operator()<10, LSE, QG>();
    else if (cnt <= 12)
        body.template operator()<12, LSE, QG>();
    else if (cnt <= 14)
        body.template operator()<14, LSE, QG>();
    else
        body.template operator()<16, LSE, QG>();
}

// ... and on the estimator and the moment source (uniform for the whole run): body<KT, LSE, QG>.
// The least-squares estimator keeps the per-pixel moments (its d > 0 term is not separable).
template <typename F>
__device__ __forceinline__ void trial_dispatch(int cnt, const SolverCfg& c, F&& body) {
    if (c.est == PTYGER_EST_LS)
        trial_dispatch_k<true, false>(cnt, body);
    else if (c.qg)
        trial_dispatch_k<false, true>(cnt, body);
    else
        trial_dispatch_k<false, false>(cnt, body);
}

// ls_run_out over the first KR entries only (KR >= the pass's trial count; the others are 0): an 8-entry
// reduce-scatter costs half the shuffles of the 16-entry one when a pass holds <= 8 trials (the usual
// pass 0); lane l then holds the warp total of entry l >> 2.
template <int KR, int K>
__device__ __forceinline__ void ls_run_out_r(float (&S)[K], const LsMom& m, double& tot, double (&mom)[4], int lane) {
    static_assert(KR <= K, "reduce width above the array");
    tot += warp_reduce_scatter_f<KR>(slice<0, KR>(S), lane);
    mom[0] += (double)m.A;
    mom[1] += (double)m.D;
    mom[2] += 2.0 * (double)m.sa2;
    mom[3] += (double)m.sb;
}

// Block-level output of the screening partials: per-lane fp64 running total `tot` of entry
// lane >> (5 - log2 K) of S (after warp_reduce_scatter<K>), per-thread fp64 moments.  Writes
// [S_0..S_{K-1} | A, D, sum|a|, sum b] for this CTA.  sred: [NW][K], smom: [NW][4].
// ... from per-lane totals of a KR-entry reduce-scatter, written in the KC-entry row layout (entries
// [KR, KC) zero) that k_reduce reads.
template <int KR, int NW>
__device__ __forceinline__ void ls_block_out_r(double tot, const double (&mom)[4], double (*sred)[KC],
                                               double (*smom)[4], double* __restrict__ part) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int P = Log2<KR>::value;
    constexpr int G = 32 >> P;
    if ((lane & (G - 1)) == 0) sred[warp][lane >> (5 - P)] = tot;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double w = warp_sum(mom[i]);
        if (lane == 0) smom[warp][i] = w;
    }
    __syncthreads();
    if (tid < KC) {
        double s = 0.0;
        if (tid < KR)
            for (int w = 0; w < NW; ++w) s += sred[w][tid];
        part[(int64_t)blockIdx.x * (KC + 4) + tid] = s;
    } else if (tid < KC + 4) {
        double s = 0.0;
        for (int w = 0; w < NW; ++w) s += smom[w][tid - KC];
        part[(int64_t)blockIdx.x * (KC + 4) + tid] = s;
    }
}

template <int K, int NW>
__device__ __forceinline__ void ls_block_out(double tot, const double (&mom)[4], double (*sred)[K],
                                             double (*smom)[4], double* __restrict__ part) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int P = Log2<K>::value;
    constexpr int G = 32 >> P;
    if ((lane & (G - 1)) == 0) sred[warp][lane >> (5 - P)] = tot;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double w = warp_sum(mom[i]);
        if (lane == 0) smom[warp][i] = w;
    }
    __syncthreads();
    if (tid < K) {
        double s = 0.0;
        for (int w = 0; w < NW; ++w) s += sred[w][tid];
        part[(int64_t)blockIdx.x * (K + 4) + tid] = s;
    } else if (tid < K + 4) {
        double s = 0.0;
        for (int w = 0; w < NW; ++w) s += smom[w][tid - K];
        part[(int64_t)blockIdx.x * (K + 4) + tid] = s;
    }
}

}  // namespace pty
