// demod_kernel.cuh — sm_100a windowed root-MUSIC demodulation kernel (thread per pixel).
//
// Window sizes M ≤ 20 (the warp kernel, demod_wide.cuh, takes 21…32).  One CTA = 4 warps on
// a 32-column strip walking (frame, 4-row block) work items; each warp stages the clamped
// M×(32+M−1) halo rows of its image row in shared memory (cp.async-prefetched one item ahead
// for M ≤ 15; the M² windows of neighbouring pixels overlap in SMEM, HBM is read about once),
// then each thread runs the whole per-pixel chain of Algorithm 1 in registers
// (R_y's triangle in per-thread shared-memory slices for M = 17…20), fused with the
// reference-phase difference and the flag store:
//
//   a2  R_y = Γ_w Γ_w^H (lower triangle, FP32)                            Eq.(4)
//   a3  u_1: power iteration on R_y from the lag-1 tone estimate; v_1 ∝ Γ_w^H u_1
//       (SVD identity), so U_nU_n^H = I − u_1u_1^H, V_nV_n^H = I − v_1v_1^H  Eqs.(7)-(11),(14)
//   a4  P(z) coefficients = diagonal sums of I − qq^H (autocorrelation of q)  Eqs.(12),(13)
//   a5  all 2M−2 roots by Aberth–Ehrlich from rotated noise-free templates; root
//       minimising |ln|z|| (≡ "closest to the unit circle, inside", P:L208 [R6])
//   a6  α = ∠ Σ_i conj(ẑ_y)^{o_i} Σ_k Γ_w(i,k) ẑ_x^{o_k}   (ẑ = z/|z| = e^{jω_y}, e^{-jω_x})
//   a7  out = wrap(α − φ_ref) ∈ (−π, π]; flags
//
// No tensor cores: these are tiny per-pixel systems (BASELINE north_star).  The path is
// FP32-FMA / MUFU bound.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "cx2.cuh"
#include "template_roots.h"

#ifndef BOS_SWEEP_UNROLL
#define BOS_SWEEP_UNROLL 1
#endif

namespace bos {

constexpr int kSweepUnroll = BOS_SWEEP_UNROLL;   // root-update loop unroll factor (A/B builds)
// the sweep's root loop is unrolled completely for K = N/2 ≤ BOS_SWEEP_FULL_MAX_K roots: the
// array rotation below then compiles to register renaming (no MOVs) at a code size the
// instruction cache still holds
#ifndef BOS_SWEEP_FULL_MAX_K
#define BOS_SWEEP_FULL_MAX_K 4
#endif
constexpr int sweep_unroll(int K) { return K <= BOS_SWEEP_FULL_MAX_K ? K : kSweepUnroll; }

constexpr int kBX = 32;               // pixels per CTA along x (one warp per row)
constexpr int kBY = 4;                // rows per CTA
constexpr int kThreads = kBX * kBY;

constexpr int kPowerMaxIt = 64;       // power-iteration cap (NONCONVERGED beyond)
#ifndef BOS_POWER_TOL
#define BOS_POWER_TOL 1e-8f
#endif
constexpr float kPowerTol = BOS_POWER_TOL;
// Clamped border windows [R1] (repeated rows / columns) leave α ill-conditioned: a held-out
// stress case (M = 17, −5 dB, a frame corner) missed the bar by 0.0012 rad with the 1e-8 stop
// and matched to 1.2e-4 rad at FP32 noise.  Border windows iterate to it (a few % of a large
// frame's pixels, in the warps of its edge strips only).
#ifndef BOS_POWER_TOL_BORDER
#define BOS_POWER_TOL_BORDER 1e-12f
#endif
constexpr float kPowerTolBorder = BOS_POWER_TOL_BORDER;    // ‖u_{k+1} − u_k‖² stop (error ≈ ‖Δu‖·λ2/(λ1−λ2) ≤ 3.3e-4 where σ1²/σ2² ≥ 1.3)
// Spatial smoothing (demod_ss.cuh): the order-m eigenvector feeds a degree-(2m−2) polynomial
// whose signal pair is a near-double root, so its angle is far more sensitive to u than at
// order M; a 3×3…m×m iteration is cheap, so it runs to FP32 noise (stress: 0.01–0.15 rad
// misses at −5…0 dB with 1e-8).
#ifndef BOS_POWER_TOL_SS
#define BOS_POWER_TOL_SS 1e-12f
#endif
constexpr float kPowerTolSS = BOS_POWER_TOL_SS;
// NEWTON_STOP sweeps also require every Newton ratio |P/P′|² < tol2, not only every Aberth
// step: an approximation repelled by its neighbours can take small steps far from any root
// (the repulsion term balances P/P′), and the loose stop then misses the root it is heading
// for.  Seen with the FB variant's polynomials (clamped border windows); always on there.
// The paper path needs it too: tools/stress_parity.py (random M, frame sizes, 0–40 dB and
// noise-free) found loose-stop misplacements at M = 17–20 (one noise-free) and, at −5 dB,
// M = 8 and 16.  It is compile-time on from M = BOS_STOP_NEWTON_MIN_M (12; cost ≤ 3 % there)
// and in the warp kernel (cost within noise); below, where it would cost 7 % at 10 dB (warps
// wait for their slowest lane), it is switched on per pixel for weak-tone windows only
// (λ1 < kLowSnrRatio·tr R_y, see below).  BOS_STOP_NEWTON_PAPER=1 forces it everywhere.
#ifndef BOS_PREFETCH
#define BOS_PREFETCH 1
#endif
#ifndef BOS_ITEMS_PER_CTA
#define BOS_ITEMS_PER_CTA 4
#endif
constexpr int kItemsPerCta = BOS_ITEMS_PER_CTA;   // (frame, row block) work items per CTA
#ifndef BOS_PREFETCH_MAX_M
#define BOS_PREFETCH_MAX_M 15   // M = 16: −9 % with prefetch (1 CTA/SM, 48 KB tiles), M = 15: +1.3 %
#endif
template <int M>
constexpr bool kPrefetch() { return BOS_PREFETCH != 0 && M <= BOS_PREFETCH_MAX_M; }   // 2 buffers ≤ 48 KB static SMEM (M ≤ 16)
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
#ifndef BOS_STOP_NEWTON_PAPER
#define BOS_STOP_NEWTON_PAPER 0
#endif
#ifndef BOS_STOP_NEWTON_MIN_M
#define BOS_STOP_NEWTON_MIN_M 12
#endif
template <bool FB, int M>
constexpr bool newton_stop() { return FB || BOS_STOP_NEWTON_PAPER != 0 || M >= BOS_STOP_NEWTON_MIN_M; }
constexpr int kAberthMaxIt = 40;      // Aberth sweep cap
// Loose sweep stop max_i |Δz_i|² < tol, then the Newton polish of the selected root.  The
// thread kernel (Gauss–Seidel sweeps) uses 2e-3 (|Δz| < 0.045): a warp runs as many sweeps as
// its slowest lane, and at 1e-3 the ~4 % of pixels needing a second sweep made most warps do
// two (C3 M = 8: 2725 → 3263 Mpixel/s; 3e-3: 3290 but −7 % at 0 dB from more tight re-runs;
// A/B vs 1e-3 over ~170 M pixels, 0–40 dB and noise-free: no pixel moved by > 1e-4 rad).
// The warp kernel (Jacobi sweeps) keeps 1e-3: at 3e-3 it misplaced 7 of 17 M pixels.
#ifndef BOS_ABERTH_TOL2
#define BOS_ABERTH_TOL2 2e-3f
#endif
constexpr float kAberthTol2 = BOS_ABERTH_TOL2;  // thread kernel (demod_kernel, demod_ss)
// Per-window-size loose tolerance of the thread / strip kernels' paper path: held-out stress
// seeds (tools/stress_r02_regressions.jsonl) found loose-stop misplacements at M = 4 (−5 dB,
// an approximation pair sharing one root, 1.39 rad) and M = 32 (10 dB, a clamped border window,
// 0.063 rad) that a tighter stop removes; the windows there are cheap (M ≤ 5: K ≤ 4 roots) or
// already long (M ≥ 21: the warp kernel used 1e-3 for the same reason).
#ifndef BOS_ABERTH_TOL2_SMALL_M
#define BOS_ABERTH_TOL2_SMALL_M 1e-4f
#endif
#ifndef BOS_ABERTH_SMALL_MAX_M
#define BOS_ABERTH_SMALL_MAX_M 5
#endif
#ifndef BOS_ABERTH_TOL2_LARGE_M
#define BOS_ABERTH_TOL2_LARGE_M 1e-3f
#endif
#ifndef BOS_ABERTH_LARGE_MIN_M
#define BOS_ABERTH_LARGE_MIN_M 21
#endif
template <int M>
constexpr float aberth_tol2() {
    return M <= BOS_ABERTH_SMALL_MAX_M ? BOS_ABERTH_TOL2_SMALL_M
                                       : (M >= BOS_ABERTH_LARGE_MIN_M ? BOS_ABERTH_TOL2_LARGE_M : kAberthTol2);
}
#ifndef BOS_ABERTH_TOL2_WIDE
#define BOS_ABERTH_TOL2_WIDE 1e-3f
#endif
constexpr float kAberthTol2Wide = BOS_ABERTH_TOL2_WIDE;   // warp kernel (demod_wide)
// Warp kernel, paper path: windows whose dominant eigenvalue λ1 is below kLowSnrRatio·tr(R_y)
// (a weak tone: λ1/tr ≈ (M·SNR + 1)/(M·(SNR + 1)), ≈ 0.91 at 10 dB, ≈ 0.5 at 0 dB) start from
// the tighter kAberthLowSnrTol2 — their polynomials have many roots near the unit circle and
// the loose stop misplaced the selected one in 5 of 400 random 0–5 dB cases at M ≥ 27
// (tools/stress_parity.py); the test is per pixel and warp-uniform, so ≥ 10 dB work is unchanged.
#ifndef BOS_LOWSNR_RATIO
#define BOS_LOWSNR_RATIO 0.9f
#endif
constexpr float kLowSnrRatio = BOS_LOWSNR_RATIO;
// Thread kernel, M < BOS_STOP_NEWTON_MIN_M: λ1 below this fraction of tr(R_y) switches the
// Newton-ratio stop on for that pixel (see newton_stop).
#ifndef BOS_WEAK_NEWTON_RATIO
#define BOS_WEAK_NEWTON_RATIO 0.7f
#endif
constexpr float kWeakNewtonRatio = BOS_WEAK_NEWTON_RATIO;
#ifndef BOS_WEAK_MODE
#define BOS_WEAK_MODE 0     // 1: weak pixels start from kAberthLowSnrTol2; 0: per-pixel Newton-ratio stop
#endif
constexpr float kAberthLowSnrTol2 = 1e-4f;
// From this window size the thread / strip kernels also apply the warp kernel's weak-tone rule
// (λ1 < kLowSnrRatio·tr R_y → start from kAberthLowSnrTol2) on top of the Newton-ratio stop:
// tools/stress_parity.py (M = 12…22, seed 7) found a 20 dB pixel at M = 20 on a small clamped
// frame 0.037 rad off, and tests/test_gpu_strip.py a 0 dB pixel at M = 22 2.4 rad off.
#ifndef BOS_WEAK_TIGHT_MIN_M
#define BOS_WEAK_TIGHT_MIN_M 16
#endif
constexpr int kWeakTightMinM = BOS_WEAK_TIGHT_MIN_M;
constexpr int kPolishMin = 2;         // Newton steps on the selected root after the sweeps:
constexpr int kPolishMax = 6;         // at least 2, then until |Δz|² < kPolishTol2, at most 6
constexpr float kPolishTol2 = 1e-12f;
// A first polish step already below this (|Δz| < 1e-4) ends the polish: Newton is quadratic,
// so the root is then within ≈ C·|Δz|² of its FP32 value (C = |P″/2P′|, ~1–10 away from
// double roots) — the second step would only confirm it.
#ifndef BOS_POLISH_ONE_STEP2
#define BOS_POLISH_ONE_STEP2 1e-8f
#endif
constexpr float kPolishOneStep2 = BOS_POLISH_ONE_STEP2;
__device__ __forceinline__ bool polish_done(int t, float w2) {
    return (t + 1 >= kPolishMin && !(w2 > kPolishTol2)) || w2 < kPolishOneStep2;
}
constexpr float kRefineMargin = 0.05f; // selection margin (|ln|z||) below which the runner-up is polished too
constexpr float kMoved2 = 1e-2f;       // polish displacement² (> 0.1) that triggers tight re-convergence
constexpr float kAberthTightTol2 = 1e-10f;

constexpr float kNearCircle = 1e-2f;  // |1 − |z|²| below which z and 1/z̄ are one cluster
constexpr float kReverse2 = 2.25f;    // |z|² beyond which P is evaluated through the reversed polynomial
constexpr float kCos2TauOmega = 0.99990000333f; // cos²(1e-2): "distinct frequency" test
constexpr float kTauSel = 1e-3f;      // AMBIGUOUS margin in |ln|z||
constexpr float kLowAmp = 1e-4f;      // LOW_AMPLITUDE threshold

enum : uint8_t {
    kFlagNonconverged = 1u << 0,
    kFlagAmbiguous = 1u << 1,
    kFlagLowAmplitude = 1u << 3,
    kFlagNonfinite = 1u << 4,
    kFlagBorder = 1u << 5,
    kFlagWeakInternal = 1u << 7,   // thread kernel scratch bit (weak-tone window), cleared before the store
};

// ---------------------------------------------------------------- complex helpers (FP32)
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
// a*b + c
__device__ __forceinline__ float2 cfma(float2 a, float2 b, float2 c) {
    return make_float2(fmaf(a.x, b.x, fmaf(-a.y, b.y, c.x)), fmaf(a.x, b.y, fmaf(a.y, b.x, c.y)));
}
// a*conj(b) + c
__device__ __forceinline__ float2 cfmac(float2 a, float2 b, float2 c) {
    return make_float2(fmaf(a.x, b.x, fmaf(a.y, b.y, c.x)), fmaf(a.y, b.x, fmaf(-a.x, b.y, c.y)));
}
__device__ __forceinline__ float cabs2(float2 a) { return fmaf(a.x, a.x, a.y * a.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
// 1/a with one MUFU.RCP (approximate reciprocal of |a|²)
__device__ __forceinline__ float2 crcp(float2 a) {
    const float r = __fdividef(1.0f, cabs2(a));
    return make_float2(a.x * r, -a.y * r);
}
// a/b
__device__ __forceinline__ float2 cdiv(float2 a, float2 b) {
    const float r = __fdividef(1.0f, cabs2(b));
    return make_float2(fmaf(a.x, b.x, a.y * b.y) * r, fmaf(a.y, b.x, -a.x * b.y) * r);
}

template <int M>
__device__ __forceinline__ constexpr int tri_off(int i, int j) {  // strict lower triangle, j < i
    return i * (i - 1) / 2 + j;
}

// Newton ratio P(z)/P′(z) of the conjugate-palindromic P (c_{N−k} = conj(c_k): C is
// Hermitian in Eqs.(12)-(13)).  For |z| > 1 it goes through the reversed polynomial
// Q(u) = z^{−N}P(z) = conj(P(conj u)), u = 1/z:  P/P′ = z·Q/(N·Q − u·Q′), so Horner always
// runs at |v| ≤ 1 (v = z or 1/z̄): no overflow for far roots, better relative accuracy.
template <int N>
__device__ __forceinline__ void newton_num_den(const cx2 (&c)[N + 1], float2 zi, float2& num, float2& den) {
    const float m2 = cabs2(zi);
    // direct Horner up to |z| = 1.5 (|z|^N stays tame); beyond, the reversed polynomial
    const bool outside = m2 > kReverse2;
    const float2 v = outside ? cscale(zi, __fdividef(1.0f, m2)) : zi;   // 1/z̄ or z
    // V and j·V as genuine 64-bit values (an f32x2 op result), so the register allocator keeps
    // each in one aligned pair instead of re-pairing scalars before every FFMA2.
    const cx2 V = cx2_make(v.x, v.y);
    const cx2 Vj = mul2(cx2_make(v.y, v.x), cx2_make(-1.0f, 1.0f));
    cx2 p = c[N];
    cx2 dp = 0ull;
#pragma unroll
    for (int k = N - 1; k >= 0; --k) {
        dp = cmad2(dp, V, Vj, p);
        p = cmad2(p, V, Vj, c[k]);
    }
    num = cx2_f2(p);
    den = cx2_f2(dp);
    if (outside) {
        const float2 q = cconj(num), dq = cconj(den), u = cconj(v);
        num = cmul(zi, q);
        den = csub(cscale(q, float(N)), cmul(u, dq));
    }
}

template <int N>
__device__ __forceinline__ float2 newton_ratio(const cx2 (&c)[N + 1], float2 zi) {
    float2 num, den;
    newton_num_den<N>(c, zi, num, den);
    return cdiv(num, den);
}

// P′(z)/P″(z): the Newton step for P′ (used for near-double roots on the unit circle).
// Horner with three accumulators: dp = P′(z), ddp = P″(z)/2.
template <int N>
__device__ __forceinline__ float2 newton_on_derivative(const cx2 (&c)[N + 1], float2 z) {
    const cx2 V = cx2_make(z.x, z.y);
    const cx2 Vj = mul2(cx2_make(z.y, z.x), cx2_make(-1.0f, 1.0f));
    cx2 p = c[N];
    cx2 dp = 0ull, ddp = 0ull;
#pragma unroll
    for (int k = N - 1; k >= 0; --k) {
        ddp = cmad2(ddp, V, Vj, dp);
        dp = cmad2(dp, V, Vj, p);
        p = cmad2(p, V, Vj, c[k]);
    }
    return cdiv(cx2_f2(dp), cscale(cx2_f2(ddp), 2.0f));
}

// One polish step on a single root, consistent with the sweeps: Newton on P, or on P′ for a
// root in the near-circle band (a near-double pair, whose centre carries the pair's arg).
template <int N>
__device__ __forceinline__ float2 polish_step(const cx2 (&c)[N + 1], float2 z) {
    return fabsf(1.0f - cabs2(z)) < kNearCircle ? newton_on_derivative<N>(c, z) : newton_ratio<N>(c, z);
}

// 1/|z|² · z = 1/z̄ (the mirror of z through the unit circle)
__device__ __forceinline__ cx2 mirror(cx2 z) {
    const float re = cx2_re(z), im = cx2_im(z);
    return mul2(z, cx2_bcast(rcp_approx(fmaf(re, re, im * im))));
}

// All roots of P (degree N = 2M−2) by a Gauss–Seidel Aberth–Ehrlich iteration that tracks
// only K = N/2 roots z_k and uses their mirrors 1/z̄_k for the other half.  On the unit circle
// P(e^{jθ})e^{−j(M−1)θ} = u^H(θ) C u(θ) ≥ 0 (C = U_nU_n^H is PSD), so roots on the circle have
// even multiplicity and the root multiset is exactly {z_k, 1/z̄_k} (Fejér–Riesz): the
// symmetric iteration finds the same root set as the companion matrix for half the
// Horner evaluations and half the reciprocal sums.
//
// Code size: the sweep over roots is a rolled loop that always updates z[0] and then
// rotates the arrays by one (after K steps they are back in order, and root k has seen the
// already-updated roots 0..k−1).  All register indices stay static; the I-cache holds one
// root update.  Complex values are packed (cx2.cuh): Horner and the reciprocal sum run on
// FFMA2.  Returns the number of sweeps; `ok` = converged or stagnated at FP32 noise.
template <int N, bool NEWTON_STOP = false>
__device__ __forceinline__ int aberth_sym(const cx2 (&c)[N + 1], cx2 (&z)[N / 2], bool& ok, float tol2,
                                          bool nstop = false) {
    constexpr int K = N / 2;
    cx2 zm[K];
#pragma unroll
    for (int k = 0; k < K; ++k) zm[k] = mirror(z[k]);
    const cx2 kNegPos = cx2_make(-1.0f, 1.0f);
    int it = 0;
    ok = false;
    for (; it < kAberthMaxIt; ++it) {
        float maxw = 0.0f;
        bool parked = false;               // some |P/P′|² ≥ tol2 (NEWTON_STOP)
#pragma unroll sweep_unroll(K)
        for (int r = 0; r < K; ++r) {
            const float2 zi = cx2_f2(z[0]);
            float2 num, den;                   // Newton ratio P/P′ = num/den
            newton_num_den<N>(c, zi, num, den);
            // Own-mirror term.  Near the unit circle z and 1/z̄ merge into one (near-)double
            // root: keeping the term there freezes the tangential (arg = ω) error.  There the
            // update is Newton on P′ instead (a double root of P is a simple root of P′;
            // quadratic), which lands on the pair's centre: same arg as the pair up to
            // O(η²) for a pair split by η ≤ kNearCircle/2.
            const bool near = fabsf(1.0f - cabs2(zi)) < kNearCircle;
            // s = Σ 1/(z_i − z_j) = Σ conj(d)/|d|², d = z_i − z_j; conj(d) = conj(z_i) + (−1,1)⊙z_j
            const cx2 ziC = mul2(z[0], cx2_make(1.0f, -1.0f));
            cx2 s = 0ull, sm = 0ull;           // two accumulators: halves the FFMA2 dependency chain
            {
                const cx2 dc = fma2(zm[0], kNegPos, ziC);
                const float q = fmaf(cx2_re(dc), cx2_re(dc), cx2_im(dc) * cx2_im(dc));
                sm = near ? 0ull : mul2(cx2_bcast(rcp_approx(q)), dc);
            }
#pragma unroll
            for (int j = 1; j < K; ++j) {
                const cx2 d1 = fma2(z[j], kNegPos, ziC);
                const float q1 = fmaf(cx2_re(d1), cx2_re(d1), cx2_im(d1) * cx2_im(d1));
                s = fma2(cx2_bcast(rcp_approx(q1)), d1, s);
                const cx2 d2 = fma2(zm[j], kNegPos, ziC);
                const float q2 = fmaf(cx2_re(d2), cx2_re(d2), cx2_im(d2) * cx2_im(d2));
                sm = fma2(cx2_bcast(rcp_approx(q2)), d2, sm);
            }
            const float2 sf = cx2_f2(add2(s, sm));
            // Aberth correction w = (P/P′) / (1 − (P/P′)·s) = num / (den − num·s): one division
            float2 w = cdiv(num, csub(den, cmul(num, sf)));
            if (near) w = newton_on_derivative<N>(c, zi);
            float w2 = cabs2(w);
            if (!(w2 < 1e30f)) {            // degenerate step (P′ = 0 or ratio·s = 1): skip
                w = make_float2(0.0f, 0.0f);
                w2 = 0.0f;
            }
            const cx2 zn = cx2_make(zi.x - w.x, zi.y - w.y);
            maxw = fmaxf(maxw, w2);
            if ((NEWTON_STOP || nstop) && !near) parked |= !(cabs2(num) < tol2 * cabs2(den));   // near: the P′ step is the test
#pragma unroll
            for (int j = 0; j + 1 < K; ++j) {
                z[j] = z[j + 1];
                zm[j] = zm[j + 1];
            }
            z[K - 1] = zn;
            zm[K - 1] = mirror(zn);
        }
        if (maxw < tol2 && !parked) { ok = true; ++it; break; }
    }
    return it;
}

// Root closest to the unit circle: argmin |ln|z|| = ½|ln|z|²| (one MUFU.LG2 per root, no
// division; a root and its mirror tie, P:L208 [R6]) and the margin, in |ln|z|| units, to the
// best root of a different frequency (|arg z − arg z_b| > τ_ω) for the AMBIGUOUS flag.
template <int K>
__device__ __forceinline__ float2 select_root(const cx2 (&zp)[K], float& margin, float2& z2) {
    float best = CUDART_INF_F, rb2 = 1.0f;
    float2 zb = make_float2(CUDART_NAN_F, CUDART_NAN_F);
    float d[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const float2 z = cx2_f2(zp[i]);
        const float r2 = cabs2(z);
        d[i] = fabsf(__log2f(r2));
        if (d[i] < best) { best = d[i]; zb = z; rb2 = r2; }
    }
    float second = CUDART_INF_F;
    z2 = zb;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const float2 z = cx2_f2(zp[i]);
        const float dot = fmaf(z.x, zb.x, z.y * zb.y);        // Re(z_i conj(z_b)) = |z_i||z_b| cos Δ
        const bool distinct = dot < 0.0f || dot * dot < kCos2TauOmega * cabs2(z) * rb2;
        if (distinct && d[i] < second) { second = d[i]; z2 = z; }
    }
    margin = (second - best) * 0.34657359f;                  // log2 → |ln r|: × ln2/2
    return zb;
}

// |ln|z|| of one root
__device__ __forceinline__ float ln_dist(float2 z) { return 0.34657359f * fabsf(__log2f(cabs2(z))); }

// Coefficients of P(z) = z^{M−1} q^H(z)(I − qq^H)q(z) for a unit vector q:
// c_{M−1} = M − ‖q‖², c_{M−1+d} = −r_d, c_{M−1−d} = −conj(r_d), r_d = Σ_i q_i conj(q_{i+d}).
// Also returns the rotation e^{jω̂} = conj(r_1)/|r_1| (tone estimate for the template).
template <int M>
__device__ __forceinline__ float2 music_coeffs(const float2 (&q)[M], cx2 (&c)[2 * M - 1]) {
    float n2 = 0.0f;
    cx2 qp[M], qnj[M];   // q_i and −j·q_i; q_i·conj(b) = re(b)·q_i + im(b)·(−j·q_i)
#pragma unroll
    for (int i = 0; i < M; ++i) {
        n2 += cabs2(q[i]);
        qp[i] = cx2_make(q[i].x, q[i].y);
        qnj[i] = cx2_make(q[i].y, -q[i].x);
    }
    c[M - 1] = cx2_make(float(M) - n2, 0.0f);
    float2 r1 = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int d = 1; d < M; ++d) {
        cx2 r = 0ull;
#pragma unroll
        for (int i = 0; i + d < M; ++i)
            r = fma2(cx2_bcast(q[i + d].x), qp[i], fma2(cx2_bcast(q[i + d].y), qnj[i], r));
        const float2 rf = cx2_f2(r);
        c[M - 1 + d] = cx2_make(-rf.x, -rf.y);
        c[M - 1 - d] = cx2_make(-rf.x, rf.y);
        if (d == 1) r1 = rf;
    }
    const float n = cabs2(r1);
    if (!(n > 0.0f)) return make_float2(1.0f, 0.0f);
    const float inv = rsqrtf(n);
    return make_float2(r1.x * inv, -r1.y * inv);
}

// Sum of outer products of M-vectors drawn from the window: ROWS = false → the columns
// Γ_w(:,k) (R = Γ_wΓ_w^H = R_y); ROWS = true → the rows Γ_w(i,:) (S = Σ_i row_i row_i^H =
// conj(Γ_w^HΓ_w)).  Real diagonal Rd + strict lower triangle Ro;  R_ij += a_i·conj(a_j) =
// re(a_j)·a_i + im(a_j)·(−j·a_i): two FFMA2 per entry.
template <int M, int TW, bool ROWS>
__device__ __forceinline__ void covariance(const float2* win, float (&Rd)[M], cx2 (&Ro)[M * (M - 1) / 2 > 0 ? M * (M - 1) / 2 : 1]) {
    constexpr int NOFF = M * (M - 1) / 2;
#pragma unroll
    for (int i = 0; i < M; ++i) Rd[i] = 0.0f;
#pragma unroll
    for (int t = 0; t < NOFF; ++t) Ro[t] = 0ull;
    const cx2 kPosNeg = cx2_make(1.0f, -1.0f);
#pragma unroll 1
    for (int k = 0; k < M; ++k) {   // rolled: one vector of Γ_w per trip (code size, regs)
        cx2 col[M], colnj[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const float2 g = ROWS ? win[k * TW + i] : win[i * TW + k];
            col[i] = cx2_make(g.x, g.y);
            colnj[i] = mul2(cx2_make(g.y, g.x), kPosNeg);     // −j·a = (im a, −re a)
            Rd[i] = fmaf(g.x, g.x, fmaf(g.y, g.y, Rd[i]));
        }
#pragma unroll
        for (int i = 1; i < M; ++i) {
#pragma unroll
            for (int j = 0; j < i; ++j) {
                cx2& r = Ro[tri_off<M>(i, j)];
                r = fma2(cx2_bcast(cx2_re(col[j])), col[i], fma2(cx2_bcast(cx2_im(col[j])), colnj[i], r));
            }
        }
    }
}

// Forward–backward average (variant f4, not in the paper): R ← ½(R + J conj(R) J), J the
// exchange matrix:  R_ij ← ½(R_ij + conj(R_{M−1−i, M−1−j})) = ½(R_ij + R_{M−1−j, M−1−i}).
template <int M>
__device__ __forceinline__ void fb_average(float (&Rd)[M], cx2 (&Ro)[M * (M - 1) / 2 > 0 ? M * (M - 1) / 2 : 1]) {
    float d2[M];
#pragma unroll
    for (int i = 0; i < M; ++i) d2[i] = 0.5f * (Rd[i] + Rd[M - 1 - i]);
#pragma unroll
    for (int i = 0; i < M; ++i) Rd[i] = d2[i];
    constexpr int NOFF = M * (M - 1) / 2;
    cx2 o2[NOFF > 0 ? NOFF : 1];
#pragma unroll
    for (int i = 1; i < M; ++i) {
#pragma unroll
        for (int j = 0; j < i; ++j)
            o2[tri_off<M>(i, j)] = mul2(add2(Ro[tri_off<M>(i, j)], Ro[tri_off<M>(M - 1 - j, M - 1 - i)]), cx2_bcast(0.5f));
    }
#pragma unroll
    for (int t = 0; t < NOFF; ++t) Ro[t] = o2[t];
}

// Dominant eigenvector of the Hermitian R (Rd, Ro) by power iteration from the lag-1 tone
// estimate u_i = e^{jω̂ i}, e^{jω̂} ∝ Σ_i R[i+1][i] (RAMP: u_i = (i − (M−1)/2)·e^{jω̂ i}, the
// second start of the FB variant), normalised; stops at ‖u_{k+1} − u_k‖² < kPowerTol.
// lam = ‖R u‖ of the last step (the Rayleigh quotient at convergence).
template <int M, bool RAMP = false>
__device__ __forceinline__ int power_iteration(const float (&Rd)[M], const cx2 (&Ro)[M * (M - 1) / 2 > 0 ? M * (M - 1) / 2 : 1],
                                               cx2 (&u)[M], bool& ok, float& lam, float tol = kPowerTol) {
    float2 r1 = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int i = 0; i + 1 < M; ++i) r1 = cadd(r1, cx2_f2(Ro[tri_off<M>(i + 1, i)]));
    float2 e = make_float2(1.0f, 0.0f);
    if (cabs2(r1) > 0.0f) e = cscale(r1, rsqrtf(cabs2(r1)));
    {
        // Σ_i (i − c)² = M(M²−1)/12
        const float s0 = RAMP ? rsqrtf(float(M) * float(M * M - 1) / 12.0f) : rsqrtf(float(M));
        float2 t = make_float2(1.0f, 0.0f);
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const float wgt = RAMP ? s0 * (float(i) - 0.5f * float(M - 1)) : s0;
            u[i] = cx2_make(wgt * t.x, wgt * t.y);
            t = cmul(t, e);
        }
    }
    lam = 0.0f;
    ok = false;
    int n = 0;
    for (; n < kPowerMaxIt;) {
        // y = R u with R Hermitian: y_i = Rd_i u_i + Σ_{j<i} R_ij u_j + Σ_{j>i} conj(R_ji) u_j
        cx2 uj[M];
#pragma unroll
        for (int j = 0; j < M; ++j) uj[j] = mul2(cx2_make(cx2_im(u[j]), cx2_re(u[j])), cx2_make(-1.0f, 1.0f));
        cx2 y[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            cx2 acc = mul2(cx2_bcast(Rd[i]), u[i]);
#pragma unroll
            for (int j = 0; j < i; ++j) {
                const cx2 r = Ro[tri_off<M>(i, j)];
                acc = fma2(cx2_bcast(cx2_re(r)), u[j], fma2(cx2_bcast(cx2_im(r)), uj[j], acc));
            }
#pragma unroll
            for (int j = i + 1; j < M; ++j) {
                const cx2 r = Ro[tri_off<M>(j, i)];
                acc = fma2(cx2_bcast(cx2_re(r)), u[j], fma2(cx2_bcast(-cx2_im(r)), uj[j], acc));
            }
            y[i] = acc;
        }
        float nrm2 = 0.0f;
#pragma unroll
        for (int i = 0; i < M; ++i) nrm2 += cabs2(cx2_f2(y[i]));
        const cx2 inv = cx2_bcast(rsqrtf(nrm2));
        lam = sqrtf(nrm2);
        float diff = 0.0f;
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const cx2 yn = mul2(y[i], inv);
            diff += cabs2(cx2_f2(sub2(yn, u[i])));
            u[i] = yn;
        }
        ++n;
        if (diff < tol) { ok = true; break; }
    }
    return n;
}

// Variant f4: the dominant eigenvector of a forward–backward averaged R.  The tone start can
// be (numerically) orthogonal to it — FB splits a window's tones into conjugate-symmetric and
// -antisymmetric combinations, e.g. on clamped border windows — and the step-size stop then
// accepts the runner-up.  Two starts (tone, ramp-weighted tone); the larger ‖R u‖ wins.
template <int M>
__device__ __forceinline__ int power_iteration_fb(const float (&Rd)[M], const cx2 (&Ro)[M * (M - 1) / 2 > 0 ? M * (M - 1) / 2 : 1],
                                                  cx2 (&u)[M], bool& ok, float tol = kPowerTol) {
    cx2 ua[M];
    bool oka = false;
    float l0, l1;
    int n = power_iteration<M, false>(Rd, Ro, u, ok, l0, tol);
    // R is PSD: if the converged eigenvalue exceeds half the trace no other eigenvalue can be
    // larger, so the tone start already found the top eigenvector (the usual case)
    float trace = 0.0f;
#pragma unroll
    for (int i = 0; i < M; ++i) trace += Rd[i];
    if (ok && l0 > 0.5005f * trace) return n;
    n += power_iteration<M, true>(Rd, Ro, ua, oka, l1, tol);
    if (l1 > l0) {
#pragma unroll
        for (int i = 0; i < M; ++i) u[i] = ua[i];
        ok = oka;
    }
    return n;
}

// ---- R_y in shared memory for larger windows (kRsmem): from M = 15 the strict lower triangle
// alone (M(M−1) registers) no longer fits beside the rest of the pixel's state and spilled to
// local memory.  Each thread keeps its triangle in a per-thread slice of dynamic shared memory
// (entry t at Rs[t·kThreads]: consecutive threads → consecutive words, conflict-free), built in
// two register-blocked passes over row ranges and read once per power-iteration matvec.
#ifndef BOS_RSMEM_MIN_M
#define BOS_RSMEM_MIN_M 17
#endif
template <int M, bool FB>
constexpr bool kRsmem() { return !FB && M >= BOS_RSMEM_MIN_M && M <= 20; }
// row boundaries of the register-blocked passes: P passes of ≈ equal entry counts
template <int M, int P, int B>
constexpr int rsmem_bound() {          // first row of pass B (B = 0 … P; bound P = M)
    if (B <= 0) return 1;
    if (B >= P) return M;
    int r = 1, acc = 0;
    const int target = (M * (M - 1) / 2) * B / P;
    while (r < M && acc + r <= target) acc += r++;
    return r;
}
// 4 passes (≈ M(M−1)/8 accumulators each): M = 18 +16 %, 19 +11 %, 20 +11 % over 2 passes
#ifndef BOS_RSMEM_PASSES
#define BOS_RSMEM_PASSES 4
#endif

// Rows [LO, HI) of the strict lower triangle of R_y (entries R_ij, j < i) accumulated over the
// M columns of the window in registers, then stored to the thread's shared-memory slice.
template <int M, int TW, int LO, int HI>
__device__ __forceinline__ void cov_pass_smem(const float2* win, cx2* Rs) {
    constexpr int E = (HI * (HI - 1) - LO * (LO - 1)) / 2;
    constexpr int B = LO * (LO - 1) / 2;               // tri_off(LO, 0)
    cx2 acc[E > 0 ? E : 1];
#pragma unroll
    for (int t = 0; t < E; ++t) acc[t] = 0ull;
    const cx2 kPosNeg = cx2_make(1.0f, -1.0f);
#pragma unroll 1
    for (int k = 0; k < M; ++k) {
        cx2 col[HI], colnj[HI];
#pragma unroll
        for (int i = 0; i < HI; ++i) {
            const float2 g = win[i * TW + k];
            col[i] = cx2_make(g.x, g.y);
            colnj[i] = mul2(cx2_make(g.y, g.x), kPosNeg);
        }
#pragma unroll
        for (int i = LO; i < HI; ++i) {
#pragma unroll
            for (int j = 0; j < i; ++j) {
                cx2& r = acc[tri_off<M>(i, j) - B];
                r = fma2(cx2_bcast(cx2_re(col[j])), col[i], fma2(cx2_bcast(cx2_im(col[j])), colnj[i], r));
            }
        }
    }
#pragma unroll
    for (int t = 0; t < E; ++t) Rs[(B + t) * kThreads] = acc[t];
}

// Power iteration as power_iteration() with R's strict lower triangle read from Rs.
// An empty asm with a memory clobber: the compiler may not move shared-memory accesses across
// it.  Unrolled sweeps over a triangle held in shared memory otherwise get all their loads
// hoisted to the top (independent addresses) and hold the whole triangle in registers.
__device__ __forceinline__ void compiler_fence() { asm volatile("" ::: "memory"); }

template <int M, int STRIDE = kThreads, bool FENCE = false>
__device__ __forceinline__ int power_iteration_smem(const float (&Rd)[M], const cx2* Rs, cx2 (&u)[M], bool& ok,
                                                    float* lam2_out = nullptr, float tol = kPowerTol) {
    float2 r1 = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int i = 0; i + 1 < M; ++i) r1 = cadd(r1, cx2_f2(Rs[tri_off<M>(i + 1, i) * STRIDE]));
    float2 e = make_float2(1.0f, 0.0f);
    if (cabs2(r1) > 0.0f) e = cscale(r1, rsqrtf(cabs2(r1)));
    {
        float2 t = make_float2(rsqrtf(float(M)), 0.0f);
#pragma unroll
        for (int i = 0; i < M; ++i) {
            u[i] = cx2_make(t.x, t.y);
            t = cmul(t, e);
        }
    }
    ok = false;
    int n = 0;
    for (; n < kPowerMaxIt;) {
        cx2 uj[M], y[M];
#pragma unroll
        for (int j = 0; j < M; ++j) {
            uj[j] = mul2(cx2_make(cx2_im(u[j]), cx2_re(u[j])), cx2_make(-1.0f, 1.0f));   // j·u
            y[j] = mul2(cx2_bcast(Rd[j]), u[j]);
        }
        // each stored R_ij (i > j) serves y_i += R_ij u_j and y_j += conj(R_ij) u_i
#pragma unroll
        for (int i = 1; i < M; ++i) {
            if constexpr (FENCE) compiler_fence();   // one row's loads in flight, not the whole triangle
#pragma unroll
            for (int j = 0; j < i; ++j) {
                const cx2 r = Rs[tri_off<M>(i, j) * STRIDE];
                y[i] = fma2(cx2_bcast(cx2_re(r)), u[j], fma2(cx2_bcast(cx2_im(r)), uj[j], y[i]));
                y[j] = fma2(cx2_bcast(cx2_re(r)), u[i], fma2(cx2_bcast(-cx2_im(r)), uj[i], y[j]));
            }
        }
        float nrm2 = 0.0f;
#pragma unroll
        for (int i = 0; i < M; ++i) nrm2 += cabs2(cx2_f2(y[i]));
        const cx2 inv = cx2_bcast(rsqrtf(nrm2));
        float diff = 0.0f;
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const cx2 yn = mul2(y[i], inv);
            diff += cabs2(cx2_f2(sub2(yn, u[i])));
            u[i] = yn;
        }
        ++n;
        if (diff < tol) {
            ok = true;
            if (lam2_out != nullptr) *lam2_out = nrm2;     // ‖R u‖² = λ1² at convergence
            break;
        }
    }
    return n;
}

// a3, second singular vector side: v_1 = Γ_w^H u_1 / ‖Γ_w^H u_1‖ (the SVD identity)
template <int M, int TW>
__device__ __forceinline__ void v1_from_window(const float2* win, const cx2 (&u)[M], float2 (&v)[M]) {
    const cx2 kPosNeg = cx2_make(1.0f, -1.0f);
    // v_1 ∝ Γ_w^H u_1:  v_k = Σ_i conj(Γ(i,k)) u_i = Σ_i re(g)·u_i + im(g)·(−j·u_i)
    cx2 unj[M];
#pragma unroll
    for (int i = 0; i < M; ++i) unj[i] = mul2(cx2_make(cx2_im(u[i]), cx2_re(u[i])), kPosNeg);
    cx2 vp[M];
    float vn = 0.0f;
#pragma unroll
    for (int k = 0; k < M; ++k) {
        cx2 acc = 0ull;
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const float2 g = win[i * TW + k];
            acc = fma2(cx2_bcast(g.x), u[i], fma2(cx2_bcast(g.y), unj[i], acc));
        }
        vp[k] = acc;
        vn += cabs2(cx2_f2(acc));
    }
    const cx2 vinv = cx2_bcast(rsqrtf(vn));
#pragma unroll
    for (int k = 0; k < M; ++k) v[k] = cx2_f2(mul2(vp[k], vinv));
}

// a4 + a5 (both axes) and a6 for one pixel, shared by the row kernel (demod_kernel) and the
// strip kernel (demod_strip.cuh): music_coeffs → symmetric Aberth from the rotated template →
// selection + polish (+ safety nets) → Eq.(15) least-squares phase.  Sets NONCONVERGED,
// AMBIGUOUS and LOW_AMPLITUDE in fl; returns the raw α (before the reference difference) and
// the selected roots zx (x axis, from v_1) and zy (y axis, from u_1).
template <int M, int TW, bool FB, bool WEAK_TIGHT = false>
__device__ __forceinline__ float roots_and_phase(const float2* win, const cx2 (&u)[M], const float2 (&v)[M], float trace,
                                                 bool pow_ok, uint8_t& fl, int& n_aby, int& n_abx, float2& zx_out,
                                                 float2& zy_out) {
    constexpr int N = 2 * M - 2;
    constexpr int O0 = (M - 1) / 2;
    float2 uf[M];
#pragma unroll
    for (int i = 0; i < M; ++i) uf[i] = cx2_f2(u[i]);

    // ---- a4 + a5, y axis (u_1) then x axis (v_1), one rolled loop ----
    float2 zy = make_float2(0.0f, 0.0f), zx = make_float2(0.0f, 0.0f);
    float my = CUDART_INF_F, mx = CUDART_INF_F;
    bool aby_ok = false, abx_ok = false;
#pragma unroll 1
    for (int axis = 0; axis < 2; ++axis) {
        float2 q[M];
#pragma unroll
        for (int i = 0; i < M; ++i) q[i] = axis ? v[i] : uf[i];
        cx2 c[N + 1];
        const float2 rot = music_coeffs<M>(q, c);
        cx2 z[N / 2];       // the inside half of the rotated template
#pragma unroll
        for (int j = 0; j < N / 2; ++j) z[j] = f2_cx2(cmul(kTemplateRoots[bos_template_offset(M) + j], rot));
        bool ok = false;
        int its = 0;
        float marg = CUDART_INF_F;
        float2 zs, z2;
        float tol2 = ((BOS_WEAK_MODE == 1 || WEAK_TIGHT) && (fl & kFlagWeakInternal)) ? fminf(kAberthLowSnrTol2, aberth_tol2<M>()) : aberth_tol2<M>();
#pragma unroll 1
        for (int attempt = 0;; ++attempt) {
            its += aberth_sym<N, newton_stop<FB, M>()>(c, z, ok, tol2, BOS_WEAK_MODE == 0 && (fl & kFlagWeakInternal));
            zs = select_root<N / 2>(z, marg, z2);
            // The sweeps stop once every root moved < 0.032 (cubic convergence leaves
            // ~1e-5 there); Newton steps on the selected root alone then make it
            // FP32-accurate (quadratic) at 1/(M−1) of a sweep each.
            const float2 zsel = zs;
#pragma unroll 1
            for (int t = 0; t < kPolishMax; ++t) {
                const float2 w = polish_step<N>(c, zs);
                const float w2 = cabs2(w);
                if (w2 < 1e30f) zs = csub(zs, w);
                if (polish_done(t, w2)) break;
            }
            // Loose sweeps can park an approximation between roots; polished, it lands on
            // a root that is no longer the closest (or moves far).  Then converge all
            // roots tightly and select again.  (Near-double roots legitimately move
            // ~0.02 toward the circle during the polish: that is not a fallback.)
            const float dsel = ln_dist(zs), dsec = ln_dist(z2) - 1e-3f;
            if (attempt == 0 && (!(dsel <= dsec || marg == CUDART_INF_F) ||
                                 !(cabs2(csub(zs, zsel)) <= kMoved2))) {
                tol2 = kAberthTightTol2;
                continue;
            }
            break;
        }
        // Near-tie between two frequencies: the loose sweeps may rank them wrongly, so
        // polish the runner-up too and re-select between the two converged roots.
        if (marg < kRefineMargin) {
#pragma unroll 1
            for (int t = 0; t < kPolishMax; ++t) {
                const float2 w = polish_step<N>(c, z2);
                const float w2 = cabs2(w);
                if (w2 < 1e30f) z2 = csub(z2, w);
                if (polish_done(t, w2)) break;
            }
            const float d1 = ln_dist(zs), d2 = ln_dist(z2);
            if (d2 < d1) zs = z2;
            marg = fabsf(d2 - d1);
        }
        if (axis == 0) { zy = zs; my = marg; aby_ok = ok; n_aby = its; }
        else { zx = zs; mx = marg; abx_ok = ok; n_abx = its; }
    }
    if (!pow_ok || !aby_ok || !abx_ok || !isfinite(zy.x + zy.y + zx.x + zx.y))
        fl |= kFlagNonconverged;
    if (fminf(my, mx) < kTauSel) fl |= kFlagAmbiguous;

    // ---- a6: Eq.(15) least-squares phase at the target pixel ----
    // ẑ_x = e^{-jω_x}, ẑ_y = e^{jω_y}; basis e^{-j(ω_x o_k + ω_y o_i)} = ẑ_x^{o_k} conj(ẑ_y)^{o_i}
    const float2 hx = cscale(zx, rsqrtf(cabs2(zx)));
    const float2 hy = cscale(zy, rsqrtf(cabs2(zy)));
    // row_i = Σ_k Γ(i,k)·tw_k = Σ_k re(g)·tw_k + im(g)·(j·tw_k)  (two FFMA2 per sample)
    cx2 tw[M], twj[M];
    {
        float2 p = make_float2(1.0f, 0.0f);
#pragma unroll
        for (int k = 0; k < O0; ++k) p = cmul(p, cconj(hx));
#pragma unroll
        for (int k = 0; k < M; ++k) {
            tw[k] = cx2_make(p.x, p.y);
            twj[k] = cx2_make(-p.y, p.x);
            p = cmul(p, hx);
        }
    }
    float2 q = make_float2(1.0f, 0.0f);
#pragma unroll
    for (int i = 0; i < O0; ++i) q = cmul(q, hy);
    float2 csum = make_float2(0.0f, 0.0f);
#pragma unroll 1
    for (int i = 0; i < M; ++i) {
        cx2 row = 0ull;
#pragma unroll
        for (int k = 0; k < M; ++k) {
            const float2 g = win[i * TW + k];
            row = fma2(cx2_bcast(g.x), tw[k], fma2(cx2_bcast(g.y), twj[k], row));
        }
        csum = cfma(cx2_f2(row), q, csum);
        q = cmul(q, cconj(hy));
    }
    if (!(cabs2(csum) >= kLowAmp * kLowAmp * float(M * M) * trace)) fl |= kFlagLowAmplitude;
    float a = atan2f(csum.y, csum.x);
    zx_out = zx;
    zy_out = zy;
    return a;
}

// roots_and_phase with the axis vectors supplied by qfn(axis, q) (axis 0: u_1, axis 1: v_1):
// the strip kernels form v_1 when the x axis starts (roots_and_phase_jit) or keep both vectors
// in shared memory (demod_strip_im_kernel), so no second M-vector is carried in registers
// through both Aberth runs.  Same arithmetic as roots_and_phase.
template <int M, int TW, bool FB, bool WEAK_TIGHT, class QFn>
__device__ __forceinline__ float roots_and_phase_q(const float2* win, QFn&& qfn, float trace, bool pow_ok, uint8_t& fl,
                                                   int& n_aby, int& n_abx, float2& zx_out, float2& zy_out) {
    constexpr int N = 2 * M - 2;
    constexpr int O0 = (M - 1) / 2;

    // ---- a4 + a5, y axis (u_1) then x axis (v_1), one rolled loop ----
    float2 zy = make_float2(0.0f, 0.0f), zx = make_float2(0.0f, 0.0f);
    float my = CUDART_INF_F, mx = CUDART_INF_F;
    bool aby_ok = false, abx_ok = false;
#pragma unroll 1
    for (int axis = 0; axis < 2; ++axis) {
        float2 q[M];
        qfn(axis, q);                              // u_1 (axis 0) or v_1 (axis 1), unit norm
        cx2 c[N + 1];
        const float2 rot = music_coeffs<M>(q, c);
        cx2 z[N / 2];       // the inside half of the rotated template
#pragma unroll
        for (int j = 0; j < N / 2; ++j) z[j] = f2_cx2(cmul(kTemplateRoots[bos_template_offset(M) + j], rot));
        bool ok = false;
        int its = 0;
        float marg = CUDART_INF_F;
        float2 zs, z2, zsel;
        // WEAK_TIGHT (large windows): a weak-tone window starts from the tight tolerance, the
        // warp kernel's rule (kLowSnrRatio) — with the Newton-ratio stop alone the loose sweeps
        // misplaced a 0 dB pixel at M = 22 (2.4 rad, tests/test_gpu_strip.py)
        float tol2 = ((BOS_WEAK_MODE == 1 || WEAK_TIGHT) && (fl & kFlagWeakInternal)) ? fminf(kAberthLowSnrTol2, aberth_tol2<M>()) : aberth_tol2<M>();
        // roots_and_phase's attempt loop and runner-up polish as one loop with ONE copy of the
        // polish code (the thread kernels are instruction-cache bound at M ≥ 13: ncu no_inst
        // stalls 23 %):  stage 0: loose sweeps, polish the selected root;  1: tight sweeps
        // after a failed check, polish again;  2: polish the runner-up of a near tie.
        int stage = 0;
#pragma unroll 1
        for (;;) {
            if (stage < 2) {
                its += aberth_sym<N, newton_stop<FB, M>()>(c, z, ok, tol2, BOS_WEAK_MODE == 0 && (fl & kFlagWeakInternal));
                zs = select_root<N / 2>(z, marg, z2);
                zsel = zs;
            }
            float2 zt = stage < 2 ? zs : z2;
#pragma unroll 1
            for (int t = 0; t < kPolishMax; ++t) {
                const float2 w = polish_step<N>(c, zt);
                const float w2 = cabs2(w);
                if (w2 < 1e30f) zt = csub(zt, w);
                if (polish_done(t, w2)) break;
            }
            if (stage < 2) {
                zs = zt;
                const float dsel = ln_dist(zs), dsec = ln_dist(z2) - 1e-3f;
                if (stage == 0 && (!(dsel <= dsec || marg == CUDART_INF_F) ||
                                   !(cabs2(csub(zs, zsel)) <= kMoved2))) {
                    tol2 = kAberthTightTol2;
                    stage = 1;
                    continue;
                }
                if (marg < kRefineMargin) {
                    stage = 2;
                    continue;
                }
                break;
            }
            z2 = zt;
            const float d1 = ln_dist(zs), d2 = ln_dist(z2);
            if (d2 < d1) zs = z2;
            marg = fabsf(d2 - d1);
            break;
        }
        if (axis == 0) { zy = zs; my = marg; aby_ok = ok; n_aby = its; }
        else { zx = zs; mx = marg; abx_ok = ok; n_abx = its; }
    }
    if (!pow_ok || !aby_ok || !abx_ok || !isfinite(zy.x + zy.y + zx.x + zx.y))
        fl |= kFlagNonconverged;
    if (fminf(my, mx) < kTauSel) fl |= kFlagAmbiguous;

    // ---- a6: Eq.(15) least-squares phase at the target pixel ----
    // ẑ_x = e^{-jω_x}, ẑ_y = e^{jω_y}; basis e^{-j(ω_x o_k + ω_y o_i)} = ẑ_x^{o_k} conj(ẑ_y)^{o_i}
    const float2 hx = cscale(zx, rsqrtf(cabs2(zx)));
    const float2 hy = cscale(zy, rsqrtf(cabs2(zy)));
    // row_i = Σ_k Γ(i,k)·tw_k = Σ_k re(g)·tw_k + im(g)·(j·tw_k)  (two FFMA2 per sample)
    cx2 tw[M], twj[M];
    {
        float2 p = make_float2(1.0f, 0.0f);
#pragma unroll
        for (int k = 0; k < O0; ++k) p = cmul(p, cconj(hx));
#pragma unroll
        for (int k = 0; k < M; ++k) {
            tw[k] = cx2_make(p.x, p.y);
            twj[k] = cx2_make(-p.y, p.x);
            p = cmul(p, hx);
        }
    }
    float2 q = make_float2(1.0f, 0.0f);
#pragma unroll
    for (int i = 0; i < O0; ++i) q = cmul(q, hy);
    float2 csum = make_float2(0.0f, 0.0f);
#pragma unroll 1
    for (int i = 0; i < M; ++i) {
        cx2 row = 0ull;
#pragma unroll
        for (int k = 0; k < M; ++k) {
            const float2 g = win[i * TW + k];
            row = fma2(cx2_bcast(g.x), tw[k], fma2(cx2_bcast(g.y), twj[k], row));
        }
        csum = cfma(cx2_f2(row), q, csum);
        q = cmul(q, cconj(hy));
    }
    if (!(cabs2(csum) >= kLowAmp * kLowAmp * float(M * M) * trace)) fl |= kFlagLowAmplitude;
    float a = atan2f(csum.y, csum.x);
    zx_out = zx;
    zy_out = zy;
    return a;
}

// roots_and_phase for the paper path with v_1 = Γ_w^H u_1/‖·‖ formed inside the axis loop when
// the x axis starts: only u stays live across the rooting of both axes — with v_1 and a copy
// of u both live (roots_and_phase) the rolled axis loop carried 4M extra registers through
// both Aberth runs.  Same arithmetic, bitwise the same result.
template <int M, int TW, bool FB, bool WEAK_TIGHT = false>
__device__ __forceinline__ float roots_and_phase_jit(const float2* win, const cx2 (&u)[M], float trace,
                                                     bool pow_ok, uint8_t& fl, int& n_aby, int& n_abx,
                                                     float2& zx_out, float2& zy_out) {
    return roots_and_phase_q<M, TW, FB, WEAK_TIGHT>(
        win,
        [&](int axis, float2 (&q)[M]) {
            if (axis == 0) {
#pragma unroll
                for (int i = 0; i < M; ++i) q[i] = cx2_f2(u[i]);
            } else {
                v1_from_window<M, TW>(win, u, q);      // v_1, formed when the x axis needs it
            }
        },
        trace, pow_ok, fl, n_aby, n_abx, zx_out, zy_out);
}

// CTAs per SM the register budget is tuned for (no spills at -O3; ptxas -v in the build log).
// (measured per M on C4: 4 CTAs/SM up to M = 9, 3 for M = 10, 11, 2 for 12, 13 — one more CTA
// costs 4–27 % at M = 10, 12, 13 through spills, one fewer is slower everywhere)
template <int M, bool FB = false>
constexpr int min_blocks_per_sm() {   // FB holds more state: its own (earlier) table — M = 11 FB: 1237 vs 1073 at 3 CTAs
    return FB ? (M <= 8 ? 4 : (M <= 10 ? 3 : (M <= 13 ? 2 : 1))) : (M <= 9 ? 4 : (M <= 11 ? 3 : (M <= 13 ? 2 : 1)));
}

template <int M, bool COUNT, bool FB = false>
__global__ void __launch_bounds__(kThreads, min_blocks_per_sm<M, FB>())
demod_kernel(const float2* __restrict__ frames, int n_frames, int H, int W,
             const float* __restrict__ ref, float* __restrict__ out, uint8_t* __restrict__ flags,
             float* __restrict__ omx, float* __restrict__ omy, unsigned long long* __restrict__ counters) {
    constexpr int N = 2 * M - 2;                 // polynomial degree
    constexpr int O0 = (M - 1) / 2;              // o_i = i − O0  [R2]
    constexpr int TW = kBX + M - 1;
    constexpr int NOFF = M * (M - 1) / 2;
    // One private halo tile per warp (row py, M rows × (32+M−1) columns): warps then move
    // through frames independently (__syncwarp only), so a warp with slow pixels never holds
    // the other three at a CTA barrier.  Re-staging the M−1 overlap rows per warp costs ~10
    // LDG/STS per pixel of a ~7k-instruction pixel.
    __shared__ float2 tiles[kPrefetch<M>() ? 2 : 1][kBY][M * TW];
    float2* tile = tiles[0][threadIdx.y];
    constexpr bool kRs = kRsmem<M, FB>();
    extern __shared__ cx2 rs_dyn[];                     // kRs: kThreads × NOFF (dynamic)
    cx2* Rs = rs_dyn + threadIdx.y * kBX + threadIdx.x;

    const int tx = threadIdx.x, ty = threadIdx.y;
    const int x0 = blockIdx.x * kBX;
    const int px = x0 + tx;
    const size_t plane = (size_t)H * (size_t)W;
    // work item = (frame, block of kBY rows); a CTA walks items blockIdx.y, +gridDim.y, … of its
    // 32-column strip (several per CTA, so the next item's halo can be prefetched)
    const int nby = (H + kBY - 1) / kBY;
    const long long nitems = (long long)n_frames * nby;
    // item → (frame, row block) advanced incrementally (no 64-bit division per item)
    const int step_f = (int)(gridDim.y / (unsigned)nby), step_b = (int)(gridDim.y % (unsigned)nby);
    auto advance = [&](int& fr, int& bl) {
        fr += step_f;
        bl += step_b;
        if (bl >= nby) { bl -= nby; ++fr; }
    };

    // a1: the clamped halo rows (Eq.(2) window support, [R1] clamp), row-wise: the clamped
    // column offsets are per lane and invariant, the row base is warp-uniform.  With prefetch
    // (kPrefetch) the next item's rows are copied by cp.async into the other buffer while this
    // item's pixels are computed.
    constexpr bool kPf = kPrefetch<M>();
    const int gx0 = min(max(x0 - O0 + tx, 0), W - 1);
    const int gx1 = min(max(x0 - O0 + tx + kBX, 0), W - 1);
    auto stage_async = [&](int fr, int bl, float2* dst) {
        const float2* __restrict__ fb = frames + (size_t)fr * plane;
        const int pyr = bl * kBY + ty;
#pragma unroll 2
        for (int r = 0; r < M; ++r) {
            const float2* __restrict__ row = fb + (size_t)min(max(pyr - O0 + r, 0), H - 1) * W;
            cp_async8(dst + r * TW + tx, row + gx0);
            if (tx + kBX < TW) cp_async8(dst + r * TW + tx + kBX, row + gx1);
        }
        cp_async_commit();
    };
    int buf = 0;
    int f = (int)(blockIdx.y / (unsigned)nby), blk = (int)(blockIdx.y % (unsigned)nby);
    if constexpr (kPf) {
        if ((long long)blockIdx.y < nitems) stage_async(f, blk, tiles[0][ty]);
    }
    for (long long it = blockIdx.y; it < nitems; it += gridDim.y, advance(f, blk)) {
        const int py = blk * kBY + ty;
        if constexpr (kPf) {
            cp_async_wait_all();
            __syncwarp();
            tile = tiles[buf][ty];
            if (it + (long long)gridDim.y < nitems) {
                int fn = f, bn = blk;
                advance(fn, bn);
                stage_async(fn, bn, tiles[buf ^ 1][ty]);
            }
            buf ^= 1;
        } else {
            const float2* __restrict__ frame = frames + (size_t)f * plane;
#pragma unroll 2
            for (int r = 0; r < M; ++r) {
                const float2* __restrict__ row = frame + (size_t)min(max(py - O0 + r, 0), H - 1) * W;
                tile[r * TW + tx] = __ldg(row + gx0);
                if (tx + kBX < TW) tile[r * TW + tx + kBX] = __ldg(row + gx1);
            }
            __syncwarp();
        }

        if (px < W && py < H) {             // warp-uniform in py
            const float2* win = tile + tx;             // Γ_w(i,k) = win[i*TW + k]
            uint8_t fl = 0;
            if (py - O0 < 0 || py + (M - 1 - O0) > H - 1 || px - O0 < 0 || px + (M - 1 - O0) > W - 1)
                fl |= kFlagBorder;

            // ---- a2: R_y = Γ_w Γ_w^H, diagonal (real) + strict lower triangle ----
            // R_ij += a·conj(b) (a = Γ(i,k), b = Γ(j,k)) = re(b)·a + im(b)·(−j·a): two FFMA2.
            float Rd[M];
            cx2 Ro[(NOFF > 0 && !kRs) ? NOFF : 1];
#pragma unroll
            for (int i = 0; i < M; ++i) Rd[i] = 0.0f;
            const cx2 kPosNeg = cx2_make(1.0f, -1.0f);
            if constexpr (kRs) {
#pragma unroll 1
                for (int k = 0; k < M; ++k) {
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        const float2 g = win[i * TW + k];
                        Rd[i] = fmaf(g.x, g.x, fmaf(g.y, g.y, Rd[i]));
                    }
                }
                constexpr int P = BOS_RSMEM_PASSES;
                cov_pass_smem<M, TW, rsmem_bound<M, P, 0>(), rsmem_bound<M, P, 1>()>(win, Rs);
                cov_pass_smem<M, TW, rsmem_bound<M, P, 1>(), rsmem_bound<M, P, 2>()>(win, Rs);
                if constexpr (P >= 3) cov_pass_smem<M, TW, rsmem_bound<M, P, 2>(), rsmem_bound<M, P, 3>()>(win, Rs);
                if constexpr (P >= 4) cov_pass_smem<M, TW, rsmem_bound<M, P, 3>(), rsmem_bound<M, P, 4>()>(win, Rs);
            } else {
#pragma unroll
            for (int t = 0; t < NOFF; ++t) Ro[t] = 0ull;
#pragma unroll 1
            for (int k = 0; k < M; ++k) {   // rolled: one column of Γ_w per trip (code size, regs)
                cx2 col[M], colnj[M];
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    const float2 g = win[i * TW + k];
                    col[i] = cx2_make(g.x, g.y);
                    colnj[i] = mul2(cx2_make(g.y, g.x), kPosNeg);     // −j·a = (im a, −re a)
                    Rd[i] = fmaf(g.x, g.x, fmaf(g.y, g.y, Rd[i]));
                }
#pragma unroll
                for (int i = 1; i < M; ++i) {
#pragma unroll
                    for (int j = 0; j < i; ++j) {
                        cx2& r = Ro[tri_off<M>(i, j)];
                        r = fma2(cx2_bcast(cx2_re(col[j])), col[i], fma2(cx2_bcast(cx2_im(col[j])), colnj[i], r));
                    }
                }
            }
            }
            float trace = 0.0f;
#pragma unroll
            for (int i = 0; i < M; ++i) trace += Rd[i];

            float result, wx = CUDART_NAN_F, wy = CUDART_NAN_F;
            int n_pow = 0, n_aby = 0, n_abx = 0;
            if (!isfinite(trace)) {
                fl |= kFlagNonfinite;
                result = CUDART_NAN_F;
            } else {
                cx2 u[M];
                bool pow_ok = false;
                float2 v[M];
                float lam2s = CUDART_INF_F;            // λ1² of the kRs power iteration
                if constexpr (kRs) {
                    n_pow = power_iteration_smem<M, kThreads, true>(Rd, Rs, u, pow_ok, &lam2s,
                                                            (fl & kFlagBorder) ? kPowerTolBorder : kPowerTol);
                    if constexpr (!FB && M >= kWeakTightMinM)
                        if (lam2s < kLowSnrRatio * kLowSnrRatio * trace * trace) fl |= kFlagWeakInternal;
                }
                if constexpr (!FB) {
                    // ---- a3: dominant eigenvector of R_y by power iteration ----
                    if constexpr (!kRs) {
                    // start: u_i = e^{jω̂ i}/√M with e^{jω̂} ∝ Σ_i R[i+1][i] (lag-1 correlation)
                    float2 r1 = make_float2(0.0f, 0.0f);
#pragma unroll
                    for (int i = 0; i + 1 < M; ++i) r1 = cadd(r1, cx2_f2(Ro[tri_off<M>(i + 1, i)]));
                    float2 e = make_float2(1.0f, 0.0f);
                    if (cabs2(r1) > 0.0f) e = cscale(r1, rsqrtf(cabs2(r1)));
                    {
                        float2 t = make_float2(rsqrtf(float(M)), 0.0f);
#pragma unroll
                        for (int i = 0; i < M; ++i) {
                            u[i] = cx2_make(t.x, t.y);
                            t = cmul(t, e);
                        }
                    }
                    float lam2 = CUDART_INF_F;   // ‖R u‖² of the converged step (λ1²); set at the break only
                    const float ptol = (fl & kFlagBorder) ? kPowerTolBorder : kPowerTol;
                    for (n_pow = 0; n_pow < kPowerMaxIt;) {
                        // y = R u with R Hermitian: y_i = Rd_i u_i + Σ_{j<i} R_ij u_j + Σ_{j>i} conj(R_ji) u_j
                        cx2 uj[M];
#pragma unroll
                        for (int j = 0; j < M; ++j) uj[j] = mul2(cx2_make(cx2_im(u[j]), cx2_re(u[j])), cx2_make(-1.0f, 1.0f));
                        cx2 y[M];
#pragma unroll
                        for (int i = 0; i < M; ++i) {
                            cx2 acc = mul2(cx2_bcast(Rd[i]), u[i]);
#pragma unroll
                            for (int j = 0; j < i; ++j) {
                                const cx2 r = Ro[tri_off<M>(i, j)];
                                acc = fma2(cx2_bcast(cx2_re(r)), u[j], fma2(cx2_bcast(cx2_im(r)), uj[j], acc));
                            }
#pragma unroll
                            for (int j = i + 1; j < M; ++j) {
                                const cx2 r = Ro[tri_off<M>(j, i)];
                                acc = fma2(cx2_bcast(cx2_re(r)), u[j], fma2(cx2_bcast(-cx2_im(r)), uj[j], acc));
                            }
                            y[i] = acc;
                        }
                        float nrm2 = 0.0f;
#pragma unroll
                        for (int i = 0; i < M; ++i) nrm2 += cabs2(cx2_f2(y[i]));
                        const cx2 inv = cx2_bcast(rsqrtf(nrm2));
                        float diff = 0.0f;
#pragma unroll
                        for (int i = 0; i < M; ++i) {
                            const cx2 yn = mul2(y[i], inv);
                            diff += cabs2(cx2_f2(sub2(yn, u[i])));
                            u[i] = yn;
                        }
                        ++n_pow;
                        if (diff < ptol) { pow_ok = true; lam2 = nrm2; break; }
                    }
                    if constexpr (!newton_stop<FB, M>()) {  // weak-tone window (see newton_stop); a flag bit, not a register
                        if (lam2 < kWeakNewtonRatio * kWeakNewtonRatio * trace * trace) fl |= kFlagWeakInternal;
                    } else if constexpr (M >= kWeakTightMinM) {   // see kWeakTightMinM
                        if (lam2 < kLowSnrRatio * kLowSnrRatio * trace * trace) fl |= kFlagWeakInternal;
                    }
                    }
                    v1_from_window<M, TW>(win, u, v);
                } else {
                    // variant f4 (not in the paper): dominant eigenvectors of the FB-averaged
                    // R_y and of FB(S), S = Σ_i row_i row_i^H = conj(R_x); v_1 = conj(eigvec of FB(S))
                    fb_average<M>(Rd, Ro);
                    n_pow = power_iteration_fb<M>(Rd, Ro, u, pow_ok);
                    covariance<M, TW, true>(win, Rd, Ro);
                    fb_average<M>(Rd, Ro);
                    cx2 sv[M];
                    bool pow2_ok = false;
                    n_pow += power_iteration_fb<M>(Rd, Ro, sv, pow2_ok);
                    pow_ok = pow_ok && pow2_ok;
#pragma unroll
                    for (int k = 0; k < M; ++k) v[k] = cconj(cx2_f2(sv[k]));
                }
                float2 zx, zy;
                float a = roots_and_phase<M, TW, FB, (!FB && M >= kWeakTightMinM)>(win, u, v, trace, pow_ok, fl, n_aby,
                                                                                   n_abx, zx, zy);
                // ---- a7: reference difference, wrap into (−π, π] ----
                if (omx != nullptr) wx = -atan2f(zx.y, zx.x);       // Eq.(15): ω_x = −arg z_x
                if (omy != nullptr) wy = atan2f(zy.y, zy.x);        //          ω_y =  arg z_y
                if (ref != nullptr) a -= __ldg(ref + (size_t)py * W + px);
                if (a > CUDART_PI_F) a -= 2.0f * CUDART_PI_F;
                if (a <= -CUDART_PI_F) a += 2.0f * CUDART_PI_F;
                result = a;
            }
            const size_t o = (size_t)f * plane + (size_t)py * W + px;
            out[o] = result;
            if (flags != nullptr) flags[o] = fl & uint8_t(~kFlagWeakInternal);
            if (omx != nullptr) omx[o] = wx;
            if (omy != nullptr) omy[o] = wy;
            if (COUNT) {
                atomicAdd(counters + 0, 1ull);
                atomicAdd(counters + 1, (unsigned long long)n_pow);
                atomicAdd(counters + 2, (unsigned long long)n_aby);
                atomicAdd(counters + 3, (unsigned long long)n_abx);
            }
        }
        __syncwarp();
    }
}

}  // namespace bos
