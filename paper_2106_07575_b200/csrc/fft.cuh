// Shared-memory batched unitary 2-D FFT for detector-sized frames (N = 16..128), sm_100a.
//
// F in Eq.1 and F^H in Eq.3, read as the UNITARY DFT
// (R#1, R#2): X[k] = (1/N) sum_n x[n] exp(-/+ 2 pi i (k.n)/N), DC at [0,0].
//
// Decomposition of one length-N line (N = R*T, R = min(N,16)):
//   x[n], n = T*n1 + n2 (n1 < R, n2 < T);  X[k], k = k1 + R*k2 (k1 < R, k2 < T)
//   X[k1 + R k2] = sum_{n2} W_T^{n2 k2} [ W_N^{n2 k1} sum_{n1} x[T n1 + n2] W_R^{n1 k1} ]
// phase 1: thread n2 holds its R strided inputs in registers -> radix-R DFT (radix-4
//          stages, compile-time twiddles) -> W_N^{n2 k1} twiddle (table in smem, fp64-built)
// phase 2: exchange through shared memory, each thread takes R/T values of k1 and runs
//          T-point DFTs over n2.
// A 2-D transform = a ROW pass (lines = rows; the T threads of a row sit in one warp and
// exchange in place with an XOR swizzle, __syncwarp only) followed by a COLUMN pass (warp
// lanes = 32 consecutive columns of one row, so every smem access is conflict-free; the
// T sub-threads of a column sit in T different warps and exchange through __syncthreads).
// Frame rows live in smem with stride LD = N + 8 complex so the two rows a half-warp
// touches in the row pass fall in disjoint bank halves.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pty {

// Complex arithmetic on Blackwell's paired FP32 instructions (PTX add/sub/mul/fma .rn.f32x2 ->
// SASS FADD2 / FMUL2 / FFMA2, one issue slot for both components; a float2 is a 64-bit register
// pair, so packing is free).  Each lane is an IEEE fp32 operation (round to nearest), so accuracy
// is that of the scalar forms; the products of a complex multiply round in a different order.
__device__ __forceinline__ uint64_t f2u(float2 a) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
    return r;
}
__device__ __forceinline__ float2 u2f(uint64_t r) {
    float2 a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
    return a;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(r);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(r);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(r);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
    return u2f(r);
}
__device__ __forceinline__ float2 bc2(float a) { return make_float2(a, a); }

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return add2(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return sub2(a, b); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return mul2(a, bc2(s)); }
// a * b = a.x (b.x, b.y) + a.y (-b.y, b.x)
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return fma2(bc2(a.y), make_float2(-b.y, b.x), mul2(bc2(a.x), b));
}
// a * conj(b) = a.x (b.x, -b.y) + a.y (b.y, b.x)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
    return fma2(bc2(a.y), make_float2(b.y, b.x), mul2(bc2(a.x), make_float2(b.x, -b.y)));
}
// conj(a) * b = a.x (b.x, b.y) + a.y (b.y, -b.x)
__device__ __forceinline__ float2 cconjmul(float2 a, float2 b) {
    return fma2(bc2(a.y), make_float2(b.y, -b.x), mul2(bc2(a.x), b));
}

// cos / sin of 2 pi q / 16 for q in [0, 16) (compile-time after unrolling)
__host__ __device__ constexpr float cos16_0_8(int q) {
    return q == 0 ? 1.0f : q == 1 ? 0.92387953251128674f : q == 2 ? 0.70710678118654752f
         : q == 3 ? 0.38268343236508977f : q == 4 ? 0.0f : q == 5 ? -0.38268343236508977f
         : q == 6 ? -0.70710678118654752f : q == 7 ? -0.92387953251128674f : -1.0f;
}
__host__ __device__ constexpr float sin16_0_8(int q) {
    return q == 0 ? 0.0f : q == 1 ? 0.38268343236508977f : q == 2 ? 0.70710678118654752f
         : q == 3 ? 0.92387953251128674f : q == 4 ? 1.0f : q == 5 ? 0.92387953251128674f
         : q == 6 ? 0.70710678118654752f : q == 7 ? 0.38268343236508977f : 0.0f;
}
__host__ __device__ constexpr float cos16(int q) { return q <= 8 ? cos16_0_8(q) : cos16_0_8(16 - q); }
__host__ __device__ constexpr float sin16(int q) { return q <= 8 ? sin16_0_8(q) : -sin16_0_8(16 - q); }

// x * W_R^m, W_R = exp(-2 pi i / R) (forward) or exp(+2 pi i / R) (INV); R divides 16.
template <int R, bool INV>
__device__ __forceinline__ float2 twr(float2 x, int m) {
    const int q = (m % R) * (16 / R);
    if (q == 0) return x;
    if (q == 8) return make_float2(-x.x, -x.y);
    if (q == 4) return INV ? make_float2(-x.y, x.x) : make_float2(x.y, -x.x);
    if (q == 12) return INV ? make_float2(x.y, -x.x) : make_float2(-x.y, x.x);
    const float c = cos16(q);
    const float s = INV ? sin16(q) : -sin16(q);
    return cmul(x, make_float2(c, s));
}

template <int R, bool INV> struct DFT;

template <bool INV> struct DFT<1, INV> {
    __device__ __forceinline__ static void run(float2 (&)[1]) {}
};
template <bool INV> struct DFT<2, INV> {
    __device__ __forceinline__ static void run(float2 (&x)[2]) {
        const float2 t = x[0];
        x[0] = cadd(t, x[1]);
        x[1] = csub(t, x[1]);
    }
};
template <bool INV> struct DFT<4, INV> {
    __device__ __forceinline__ static void run(float2 (&x)[4]) {
        const float2 t0 = cadd(x[0], x[2]), t1 = csub(x[0], x[2]);
        const float2 t2 = cadd(x[1], x[3]), t3 = twr<4, INV>(csub(x[1], x[3]), 1);
        x[0] = cadd(t0, t2);
        x[2] = csub(t0, t2);
        x[1] = cadd(t1, t3);
        x[3] = csub(t1, t3);
    }
};

// R = R1*R2 with n = R2*n1 + n2, k = k1 + R1*k2 (same split as the line decomposition).
template <int R1, int R2, bool INV>
__device__ __forceinline__ void dft_2level(float2 (&x)[R1 * R2]) {
    constexpr int R = R1 * R2;
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) {
        float2 a[R1];
#pragma unroll
        for (int n1 = 0; n1 < R1; ++n1) a[n1] = x[R2 * n1 + n2];
        DFT<R1, INV>::run(a);
#pragma unroll
        for (int k1 = 0; k1 < R1; ++k1) x[R2 * k1 + n2] = twr<R, INV>(a[k1], n2 * k1);
    }
    float2 y[R];
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) {
        float2 b[R2];
#pragma unroll
        for (int n2 = 0; n2 < R2; ++n2) b[n2] = x[R2 * k1 + n2];
        DFT<R2, INV>::run(b);
#pragma unroll
        for (int k2 = 0; k2 < R2; ++k2) y[k1 + R1 * k2] = b[k2];
    }
#pragma unroll
    for (int i = 0; i < R; ++i) x[i] = y[i];
}

template <bool INV> struct DFT<8, INV> {
    __device__ __forceinline__ static void run(float2 (&x)[8]) { dft_2level<4, 2, INV>(x); }
};
template <bool INV> struct DFT<16, INV> {
    __device__ __forceinline__ static void run(float2 (&x)[16]) { dft_2level<4, 4, INV>(x); }
};

// ------------------------------------------------------------------------------------
// Line FFTs over a frame held in shared memory.
// ------------------------------------------------------------------------------------
template <int N>
struct FFTCfg {
    static constexpr int R = N < 16 ? N : 16;    // radix of phase 1 (registers)
    static constexpr int T = N / R;              // threads per line / radix of phase 2
    static constexpr int LD = N + 8;             // smem row stride (complex), LD % 16 == 8
    static constexpr int NT = 512;               // threads per CTA
    static constexpr int FPB = (NT / (N * T)) > 0 ? (NT / (N * T)) : 1;  // frames per CTA step
    static constexpr int LINES = FPB * N;        // lines per pass
    static constexpr int LPR = NT / T;           // lines per round
    static constexpr int ROUNDS = LINES / LPR;   // rounds per pass
    static constexpr int FRAME_ELEMS = N * LD;
    // + N: twiddle table tw[m] = W_N^m; + R*T: the row-pass copy twr[k1*T + t] = W_N^{t k1}
    static constexpr size_t SMEM_BYTES = (size_t)(FPB * FRAME_ELEMS + N + R * T) * sizeof(float2);
    // with the pre-swapped float4 tables (build_twiddles4)
    static constexpr size_t SMEM_BYTES4 = (size_t)FPB * FRAME_ELEMS * sizeof(float2) + (size_t)(N + R * T) * 16;
    static_assert(N * T * FPB % NT == 0 || FPB == 1, "bad config");
    static_assert(LINES % LPR == 0, "bad rounds");
};

// Twiddle table tw[m] = exp(-2 pi i m / N), built in double precision.
template <int N>
__device__ __forceinline__ void build_twiddles(float2* tw) {
    for (int m = threadIdx.x; m < N; m += blockDim.x) {
        double s, c;
        sincospi(2.0 * (double)m / (double)N, &s, &c);
        tw[m] = make_float2((float)c, (float)(-s));
    }
}

template <bool INV>
__device__ __forceinline__ float2 twmul(float2 x, float2 w) { return INV ? cmulc(x, w) : cmul(x, w); }

// Pre-swapped twiddle entries w4 = (c, s, -s, c) for w = c + i s (the direction's sign already in s):
// x w = x.x (c, s) + x.y (-s, c) is one FMUL2 + one FFMA2 straight from the 16-B table entry (the
// float2 table needs a negation to form (-s, c) for every multiply).
__device__ __forceinline__ float2 twmul4(float2 x, float4 w) {
    return fma2(bc2(x.y), make_float2(w.z, w.w), mul2(bc2(x.x), make_float2(w.x, w.y)));
}
template <bool INV>
__device__ __forceinline__ float2 twm(float2 x, const float2* tw, int i) { return twmul<INV>(x, tw[i]); }
template <bool INV>
__device__ __forceinline__ float2 twm(float2 x, const float4* tw, int i) { return twmul4(x, tw[i]); }

// float4 tables: tw4[m] = W^m and the row-pass copy tw4[N + k1*T + t] = W^{t k1}, W = exp(-/+ 2 pi i / N)
// (INV: +), built in double precision (same values as build_twiddles / build_row_twiddles).
template <int N, bool INV>
__device__ __forceinline__ void build_twiddles4(float4* tw4) {
    constexpr int R = N < 16 ? N : 16, T = N / R;
    for (int i = threadIdx.x; i < N + R * T; i += blockDim.x) {
        const int m = i < N ? i : ((i - N) % T) * ((i - N) / T);
        double sn, cs;
        sincospi(2.0 * (double)m / (double)N, &sn, &cs);
        const float c = (float)cs, sg = INV ? (float)sn : (float)(-sn);
        tw4[i] = make_float4(c, sg, -sg, c);
    }
}

// Row-pass twiddles laid out [k1][t]: the T sub-threads of a row read T consecutive entries (the
// tw[t k1] layout made those reads 2..8-way bank conflicted).  Same fp64-built values as tw.
template <int N>
__device__ __forceinline__ void build_row_twiddles(float2* twr) {
    constexpr int R = N < 16 ? N : 16, T = N / R;
    for (int i = threadIdx.x; i < R * T; i += blockDim.x) {
        const int k1 = i / T, t = i % T;
        double sn, cs;
        sincospi(2.0 * (double)(t * k1) / (double)N, &sn, &cs);
        twr[i] = make_float2((float)cs, (float)(-sn));
    }
}

// ROW pass in two halves (row_fft = row_fft_a then row_fft_b): a = radix-R DFT + twiddles in
// registers (no shared memory), b = the exchange through srow + the T-point DFTs.  Lets a caller
// place a barrier between them (before its first write of the row buffer).
template <int N, bool INV, bool TWR = false, typename TW = float2>
__device__ __forceinline__ void row_fft_a(float2 (&x)[FFTCfg<N>::R], int t, const TW* tw, const TW* twr = nullptr) {
    constexpr int R = FFTCfg<N>::R, T = FFTCfg<N>::T;
    static_assert(T > 1, "row_fft_a needs T > 1");
    DFT<R, INV>::run(x);
#pragma unroll
    for (int k1 = 1; k1 < R; ++k1) {
        if constexpr (TWR)
            x[k1] = twm<INV>(x[k1], twr, k1 * T + t);
        else
            x[k1] = twm<INV>(x[k1], tw, t * k1);
    }
}
template <int N, bool INV>
__device__ __forceinline__ void row_fft_b(float2 (&x)[FFTCfg<N>::R], float2* srow, int t) {
    constexpr int R = FFTCfg<N>::R, T = FFTCfg<N>::T;
#pragma unroll
    for (int k1 = 0; k1 < R; ++k1) srow[T * k1 + (t ^ (k1 & (T - 1)))] = x[k1];
    __syncwarp();
    float2 y[R];
#pragma unroll
    for (int j = 0; j < R / T; ++j) {
        const int k1 = j * T + t;
#pragma unroll
        for (int n2 = 0; n2 < T; ++n2) y[j * T + n2] = srow[T * k1 + (n2 ^ t)];
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < R / T; ++j) {
        float2 b[T];
#pragma unroll
        for (int n2 = 0; n2 < T; ++n2) b[n2] = y[j * T + n2];
        DFT<T, INV>::run(b);
        const int k1 = j * T + t;
#pragma unroll
        for (int k2 = 0; k2 < T; ++k2) srow[k1 + R * k2] = b[k2];
    }
}

// ROW pass for one row: x[n1] = input element at column T*n1 + t.  Leaves the row's DFT
// (unnormalised) in srow[0..N) in natural order.  The T threads of the row must be
// consecutive lanes of one warp and all 32 lanes must call this together.
template <int N, bool INV, bool TWR = false, typename TW = float2>
__device__ __forceinline__ void row_fft(float2 (&x)[FFTCfg<N>::R], float2* srow, int t, const TW* tw,
                                        const TW* twr = nullptr) {
    constexpr int R = FFTCfg<N>::R, T = FFTCfg<N>::T;
    DFT<R, INV>::run(x);
    if constexpr (T == 1) {
#pragma unroll
        for (int k = 0; k < R; ++k) srow[k] = x[k];
    } else {
#pragma unroll
        for (int k1 = 1; k1 < R; ++k1) {
            if constexpr (TWR)
                x[k1] = twm<INV>(x[k1], twr, k1 * T + t);
            else
                x[k1] = twm<INV>(x[k1], tw, t * k1);
        }
#pragma unroll
        for (int k1 = 0; k1 < R; ++k1) srow[T * k1 + (t ^ (k1 & (T - 1)))] = x[k1];
        __syncwarp();
        float2 y[R];
#pragma unroll
        for (int j = 0; j < R / T; ++j) {
            const int k1 = j * T + t;
#pragma unroll
            for (int n2 = 0; n2 < T; ++n2) y[j * T + n2] = srow[T * k1 + (n2 ^ t)];
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < R / T; ++j) {
            float2 b[T];
#pragma unroll
            for (int n2 = 0; n2 < T; ++n2) b[n2] = y[j * T + n2];
            DFT<T, INV>::run(b);
            const int k1 = j * T + t;
#pragma unroll
            for (int k2 = 0; k2 < T; ++k2) srow[k1 + R * k2] = b[k2];
        }
    }
}

// ROW pass whose results stay in registers: X[j*T + k2] is column (j*T + t) + R*k2 of the row
// (same arithmetic as row_fft; srow is used only for the exchange and is clobbered).
template <int N, bool INV, bool TWR = false, typename TW = float2>
__device__ __forceinline__ void row_fft_regs(float2 (&x)[FFTCfg<N>::R], float2* srow, int t, const TW* tw,
                                             const TW* twr = nullptr) {
    constexpr int R = FFTCfg<N>::R, T = FFTCfg<N>::T;
    static_assert(T > 1, "row_fft_regs needs T > 1");
    DFT<R, INV>::run(x);
#pragma unroll
    for (int k1 = 1; k1 < R; ++k1) {
        if constexpr (TWR)
            x[k1] = twm<INV>(x[k1], twr, k1 * T + t);
        else
            x[k1] = twm<INV>(x[k1], tw, t * k1);
    }
    __syncwarp();
#pragma unroll
    for (int k1 = 0; k1 < R; ++k1) srow[T * k1 + (t ^ (k1 & (T - 1)))] = x[k1];
    __syncwarp();
#pragma unroll
    for (int j = 0; j < R / T; ++j) {
        const int k1 = j * T + t;
        float2 b[T];
#pragma unroll
        for (int n2 = 0; n2 < T; ++n2) b[n2] = srow[T * k1 + (n2 ^ t)];
        DFT<T, INV>::run(b);
#pragma unroll
        for (int k2 = 0; k2 < T; ++k2) x[j * T + k2] = b[k2];
    }
}

// COLUMN pass phase 1 for column scol (pointer to element [0][c]); sub-thread t.
// Reads rows T*n1 + t, writes the twiddled radix-R outputs back to rows T*k1 + t.
template <int N, bool INV, typename TW = float2>
__device__ __forceinline__ void col_fft_phase1(float2* scol, int t, const TW* tw) {
    constexpr int R = FFTCfg<N>::R, T = FFTCfg<N>::T, LD = FFTCfg<N>::LD;
    float2 x[R];
#pragma unroll
    for (int n1 = 0; n1 < R; ++n1) x[n1] = scol[(T * n1 + t) * LD];
    DFT<R, INV>::run(x);
    if constexpr (T > 1) {
#pragma unroll
        for (int k1 = 1; k1 < R; ++k1) x[k1] = twm<INV>(x[k1], tw, t * k1);
    }
#pragma unroll
    for (int k1 = 0; k1 < R; ++k1) scol[(T * k1 + t) * LD] = x[k1];
}

// COLUMN pass phase 2 (after a block barrier): X[j*T + k2] is output row k1 + R*k2 with
// k1 = j*T + t.  Results stay in registers (the caller's epilogue consumes them).
template <int N, bool INV>
__device__ __forceinline__ void col_fft_phase2(const float2* scol, int t, float2 (&X)[FFTCfg<N>::R]) {
    constexpr int R = FFTCfg<N>::R, T = FFTCfg<N>::T, LD = FFTCfg<N>::LD;
#pragma unroll
    for (int j = 0; j < R / T; ++j) {
        const int k1 = j * T + t;
        float2 b[T];
#pragma unroll
        for (int n2 = 0; n2 < T; ++n2) b[n2] = scol[(T * k1 + n2) * LD];
        DFT<T, INV>::run(b);
#pragma unroll
        for (int k2 = 0; k2 < T; ++k2) X[j * T + k2] = b[k2];
    }
}

template <int N>
__device__ __forceinline__ int col_out_row(int idx, int t) {
    constexpr int R = FFTCfg<N>::R, T = FFTCfg<N>::T;
    const int j = idx / T, k2 = idx % T;
    return (j * T + t) + R * k2;
}

}  // namespace pty
