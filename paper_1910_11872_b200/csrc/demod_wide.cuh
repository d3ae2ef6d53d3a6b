// demod_wide.cuh — warp-per-pixel root-MUSIC demodulation for large windows (M = 21…32 by default;
// the FB variant from 19).
//
// Same algorithm and arithmetic as demod_kernel.cuh (a1–a7, symmetric Aberth, Newton polish),
// laid out for M where a thread can no longer hold R_y (M(M+1)/2 complex) in registers:
//
// * one CTA = 4 warps = 4 image rows × a 32-pixel row segment; the CTA stages the clamped
//   (4+M−1)×(32+M−1) halo once per frame (odd row stride → conflict-free column reads);
// * each warp walks its 32 pixels left to right; lane i owns row i of R_y.  R_y is formed in
//   full at the first pixel of the segment and then slid one column per pixel with a rank-2
//   update  R += a_new a_new^H − a_old a_old^H  (2M instead of M² complex MACs per lane; the
//   refresh every 32 pixels bounds FP32 drift to ~32 ε‖R‖ — cf. parity tests);
// * power iteration, v_1 = Γ^H u_1 and the autocorrelation coefficients use lane-distributed
//   vectors and warp shuffles; the polynomial coefficients go to a per-warp SMEM buffer that
//   every lane reads by broadcast during Horner;
// * Aberth: lane k owns tracked root z_k (K = M−1 ≤ 31 roots), simultaneous (Jacobi) update,
//   the other roots and mirrors arrive through per-warp SMEM buffers; warp-reduced stop test,
//   argmin selection and margin; Newton polish of the selected root with the whole warp;
// * per-root loops unrolled 8× (≤ 128 registers → 4 CTAs/SM without spills);
// * Eq.(15) row sums per lane, warp reduction, lane 0 stores phase + flags.
#pragma once

#include "demod_kernel.cuh"

namespace bos {

// Smallest window handled warp-per-pixel by the row-kernel dispatch (small launches of the
// paper path and the FB variant; FB switches at 19).  Large paper-path launches of M ≤ 22 run
// the strip kernels (demod_strip.cuh) instead: round-2 C3 1024² ×8, 10 dB: M = 21 286 vs 156,
// M = 22 260 vs 149 Mpixel/s (profiles/r02_c4_sweep.md); from M = 23 this kernel is faster
// (the strip kernel's shared-memory R_y leaves 2 warps per SM).
#ifndef BOS_WIDE_MIN_M
#define BOS_WIDE_MIN_M 21
#endif
constexpr int kWideMinM = BOS_WIDE_MIN_M;
// unroll factor of the warp kernel's per-root loops (Horner over N, reciprocal sums over K):
// unroll 8 instead of full unrolling shrinks the code (the kernel showed instruction-fetch
// stalls) and the registers (≤ 128 → 4 CTAs/SM without spills): M = 21 +6 %, 24 +4 %, 25…32
// +12…16 % over full unroll with 2–3 CTAs/SM
#ifndef BOS_WIDE_UNROLL
#define BOS_WIDE_UNROLL 8
#endif
#ifndef BOS_WIDE_UNROLL_MAX_M
#define BOS_WIDE_UNROLL_MAX_M 32
#endif
template <int N>
constexpr int wide_unroll() { return N <= 2 * BOS_WIDE_UNROLL_MAX_M - 2 ? BOS_WIDE_UNROLL : 64; }
template <bool FB>
constexpr int wide_min_m() { return FB ? (BOS_WIDE_MIN_M < 19 ? BOS_WIDE_MIN_M : 19) : BOS_WIDE_MIN_M; }

__device__ __forceinline__ cx2 shfl_cx2(cx2 v, int src) {
    return (cx2)__shfl_sync(0xffffffffu, (unsigned long long)v, src);
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float2 warp_sum2(float2 v) { return make_float2(warp_sum(v.x), warp_sum(v.y)); }

// Horner on coefficients in shared memory (broadcast reads): Newton ratio P/P′ with the
// reversed-polynomial evaluation for |z| > 1 (see newton_ratio).
template <int N>
__device__ __forceinline__ float2 newton_ratio_smem(const cx2* __restrict__ c, float2 zi) {
    const float m2 = cabs2(zi);
    const bool outside = m2 > 1.0f;
    const float2 v = outside ? cscale(zi, __fdividef(1.0f, m2)) : zi;
    const cx2 V = cx2_make(v.x, v.y);
    const cx2 Vj = mul2(cx2_make(v.y, v.x), cx2_make(-1.0f, 1.0f));
    cx2 p = c[N];
    cx2 dp = 0ull;
#pragma unroll (wide_unroll<N>())
    for (int k = N - 1; k >= 0; --k) {
        dp = cmad2(dp, V, Vj, p);
        p = cmad2(p, V, Vj, c[k]);
    }
    float2 num = cx2_f2(p), den = cx2_f2(dp);
    if (outside) {
        const float2 q = cconj(num), dq = cconj(den), u = cconj(v);
        num = cmul(zi, q);
        den = csub(cscale(q, float(N)), cmul(u, dq));
    }
    return cdiv(num, den);
}

template <int N>
__device__ __forceinline__ float2 newton_on_derivative_smem(const cx2* __restrict__ c, float2 z) {
    const cx2 V = cx2_make(z.x, z.y);
    const cx2 Vj = mul2(cx2_make(z.y, z.x), cx2_make(-1.0f, 1.0f));
    cx2 p = c[N];
    cx2 dp = 0ull, ddp = 0ull;
#pragma unroll (wide_unroll<N>())
    for (int k = N - 1; k >= 0; --k) {
        ddp = cmad2(ddp, V, Vj, dp);
        dp = cmad2(dp, V, Vj, p);
        p = cmad2(p, V, Vj, c[k]);
    }
    return cdiv(cx2_f2(dp), cscale(cx2_f2(ddp), 2.0f));
}

// P(z)/P′(z) at ONE point z with the whole warp: lane l sums the terms k = 2l, 2l+1 (the
// coefficient buffer is zero-padded to 64), v^{2l−1} by binary exponentiation, then a warp
// reduction — ~5 dependent complex products + 5 shuffle levels instead of an N-step Horner
// chain on every lane.  Reversed evaluation for |z| > 1 as in newton_ratio.
template <int N>
__device__ __forceinline__ float2 newton_ratio_warp(const cx2* __restrict__ c, float2 zi, int lane) {
    const float m2 = cabs2(zi);
    const bool near = fabsf(1.0f - m2) < kNearCircle;    // near-double pair: Newton on P′ (see polish_step)
    const bool outside = !near && m2 > 1.0f;
    const float2 v = outside ? cscale(zi, __fdividef(1.0f, m2)) : zi;
    const float2 v2 = cmul(v, v);
    // q = (v²)^{l−1} = v^{2l−2} for l ≥ 1 (5-bit exponent)
    const int e = lane > 0 ? lane - 1 : 0;
    float2 q = make_float2(1.0f, 0.0f), b = v2;
#pragma unroll
    for (int bit = 0; bit < 5; ++bit) {
        if ((e >> bit) & 1) q = cmul(q, b);
        b = cmul(b, b);
    }
    const float2 pm1 = cmul(q, v);                                  // v^{2l−1}
    const float2 pw = lane > 0 ? cmul(pm1, v) : make_float2(1.0f, 0.0f);   // v^{2l}
    const float2 c0 = cx2_f2(c[2 * lane]), c1 = cx2_f2(c[2 * lane + 1]);
    const float a = float(2 * lane);
    // terms k = 2l, 2l+1 of P, P′ and P″
    const float2 pp = cmul(pw, cfma(c1, v, c0));
    const float2 dterm = cfma(cscale(c1, a + 1.0f), v, cscale(c0, a));          // 2l·c0 + (2l+1)·c1·v
    const float2 dd = lane > 0 ? cmul(pm1, dterm) : c1;
    float2 num, den;
    if (near) {                                                          // warp-uniform (zi is)
        const float2 d2term = cfma(cscale(c1, (a + 1.0f) * a), v, cscale(c0, a * (a - 1.0f)));
        const float2 dd2 = lane > 0 ? cmul(q, d2term) : make_float2(0.0f, 0.0f);
        num = warp_sum2(dd);
        den = warp_sum2(dd2);
    } else {
        num = warp_sum2(pp);
        den = warp_sum2(dd);
        if (outside) {
            const float2 qq = cconj(num), dq = cconj(den), u = cconj(v);
            num = cmul(zi, qq);
            den = csub(cscale(qq, float(N)), cmul(u, dq));
        }
    }
    return cdiv(num, den);
}

// Variant f4 (forward–backward averaging, not in the paper), lane i holding row i of the
// Hermitian R:  R_ij ← ½(R_ij + conj(R_{M−1−i, M−1−j})).  Register j of lane M−1−i is R_{M−1−i, j},
// so for a fixed register index every lane reads the same index from its mirror lane (one
// shuffle per register); pairs (j, M−1−j) are updated together so no read sees a new value.
template <int M>
__device__ __forceinline__ void fb_average_rows(cx2 (&R)[M], int ri) {
    const int src = M - 1 - ri;
#pragma unroll
    for (int j = 0; j < M / 2; ++j) {
        const float2 a = cx2_f2(shfl_cx2(R[M - 1 - j], src));   // R_{M−1−i, M−1−j}
        const float2 b = cx2_f2(shfl_cx2(R[j], src));           // R_{M−1−i, j}
        R[j] = mul2(add2(R[j], f2_cx2(cconj(a))), cx2_bcast(0.5f));
        R[M - 1 - j] = mul2(add2(R[M - 1 - j], f2_cx2(cconj(b))), cx2_bcast(0.5f));
    }
    if (M & 1) {
        const float2 a = cx2_f2(shfl_cx2(R[M / 2], src));
        R[M / 2] = mul2(add2(R[M / 2], f2_cx2(cconj(a))), cx2_bcast(0.5f));
    }
}

// Dominant eigenvector of the Hermitian R (lane i: row i) by power iteration from the lag-1
// tone estimate (as the thread kernel); lane i returns u_i (0 on lanes ≥ M).  `va` is the
// warp's broadcast buffer.  Returns the iteration count; ok = converged.
template <int M, bool RAMP = false>
__device__ __forceinline__ int power_iteration_warp(const cx2 (&R)[M], int lane, bool rl, cx2* va, cx2& u, bool& ok,
                                                    float& lam) {
    const cx2 kNegPos = cx2_make(-1.0f, 1.0f);
    float2 sub = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int j = 0; j < M; ++j)
        if (j + 1 == lane) sub = cx2_f2(R[j]);
    const float2 r1 = warp_sum2(rl ? sub : make_float2(0.0f, 0.0f));   // Σ_i R[i+1][i]
    float2 e = make_float2(1.0f, 0.0f);
    if (cabs2(r1) > 0.0f) e = cscale(r1, rsqrtf(cabs2(r1)));
    {
        float2 t = make_float2(1.0f, 0.0f), ul = t;
#pragma unroll
        for (int j = 0; j < M; ++j) {
            if (j == lane) ul = t;
            t = cmul(t, e);
        }
        // RAMP (second FB start): weight (i − (M−1)/2); Σ_i (i − c)² = M(M²−1)/12
        const float wgt = RAMP ? rsqrtf(float(M) * float(M * M - 1) / 12.0f) * (float(lane) - 0.5f * float(M - 1))
                               : rsqrtf(float(M));
        u = rl ? cx2_make(wgt * ul.x, wgt * ul.y) : 0ull;
    }
    ok = false;
    lam = 0.0f;
    int n = 0;
    for (; n < kPowerMaxIt;) {
        if (rl) va[lane] = u;
        __syncwarp();
        cx2 y = 0ull;
#pragma unroll
        for (int j = 0; j < M; ++j) {
            const cx2 uj = va[j];                                   // broadcast
            const cx2 ujj = mul2(cx2_make(cx2_im(uj), cx2_re(uj)), kNegPos);
            y = fma2(cx2_bcast(cx2_re(R[j])), uj, fma2(cx2_bcast(cx2_im(R[j])), ujj, y));
        }
        __syncwarp();
        if (!rl) y = 0ull;
        const float nrm2 = warp_sum(cabs2(cx2_f2(y)));
        const cx2 yn = mul2(y, cx2_bcast(rsqrtf(nrm2)));
        lam = sqrtf(nrm2);
        const float diff = warp_sum(cabs2(cx2_f2(sub2(yn, u))));
        u = yn;
        ++n;
        if (diff < kPowerTol) { ok = true; break; }
    }
    return n;
}

// Variant f4: two starts (tone, ramp-weighted tone), the larger ‖R u‖ wins (see the thread
// kernel's power_iteration_fb for why one start is not enough under FB averaging).
template <int M>
__device__ __forceinline__ int power_iteration_warp_fb(const cx2 (&R)[M], int lane, bool rl, cx2* va, cx2& u,
                                                       bool& ok, float trace, float& lam) {
    cx2 ua;
    bool oka = false;
    float l0, l1;
    int n = power_iteration_warp<M, false>(R, lane, rl, va, u, ok, l0);
    lam = l0;
    if (ok && l0 > 0.5005f * trace) return n;     // > half the trace of a PSD R: the top one
    n += power_iteration_warp<M, true>(R, lane, rl, va, ua, oka, l1);
    if (l1 > l0) {          // warp-uniform (warp sums)
        u = ua;
        ok = oka;
        lam = l1;
    }
    return n;
}

#ifndef BOS_WIDE_BLOCKS
#define BOS_WIDE_BLOCKS 0
#endif
template <int M>
constexpr int wide_min_blocks() {   // measured: 4 CTAs/SM (≤ 128 registers, no spills) best for M = 21…32
    return BOS_WIDE_BLOCKS > 0 ? BOS_WIDE_BLOCKS : 4;
}

template <int M, bool COUNT, bool FB = false>
__global__ void __launch_bounds__(kThreads, wide_min_blocks<M>())
demod_wide_kernel(const float2* __restrict__ frames, int n_frames, int H, int W,
                  const float* __restrict__ ref, float* __restrict__ out, uint8_t* __restrict__ flags,
                  float* __restrict__ omx, float* __restrict__ omy, unsigned long long* __restrict__ counters) {
    static_assert(M >= 3 && M <= 32, "wide kernel: M <= 32");
    constexpr int N = 2 * M - 2;                 // polynomial degree
    constexpr int K = N / 2;                     // tracked (inside) roots, one per lane
    constexpr int O0 = (M - 1) / 2;              // o_i = i − O0  [R2]
    constexpr int TW = (kBX + M - 1) | 1;        // odd float2 stride: conflict-free row-per-lane reads
    constexpr int TH = kBY + M - 1;
    __shared__ float2 tile[TH * TW];
    __shared__ cx2 coef_s[kBY][64];              // P coefficients, zero-padded to 64 (lane-parallel polish)
    __shared__ cx2 vec_s[kBY][2][64];            // per-warp broadcast vectors (u / q / roots, mirrors)

    const int lane = threadIdx.x, warp = threadIdx.y;
    const int x0 = blockIdx.x * kBX, y0 = blockIdx.y * kBY;
    const int py = y0 + warp;
    const size_t plane = (size_t)H * (size_t)W;
    const int ri = lane < M ? lane : M - 1;      // lane's row / column of the window (clamped)
    const bool rl = lane < M;
    const bool kl = lane < K;
    cx2* coef = coef_s[warp];
    cx2* va = vec_s[warp][0];
    cx2* vb = vec_s[warp][1];
    const cx2 kPosNeg = cx2_make(1.0f, -1.0f);
    const cx2 kNegPos = cx2_make(-1.0f, 1.0f);
    // zero padding: coef[N+1..63], va/vb[M..63] stay 0 (only indices < N+1 / < M are written)
    for (int t = lane; t < 64; t += kBX) {
        coef[t] = 0ull;
        va[t] = 0ull;
        vb[t] = 0ull;
    }
    __syncwarp();

    for (int f = blockIdx.z; f < n_frames; f += gridDim.z) {
        const float2* __restrict__ frame = frames + (size_t)f * plane;
        // ---- a1: stage the clamped halo tile ----
        for (int idx = warp * kBX + lane; idx < TH * (kBX + M - 1); idx += kThreads) {
            const int r = idx / (kBX + M - 1), cc = idx - r * (kBX + M - 1);
            const int gy = min(max(y0 - O0 + r, 0), H - 1);
            const int gx = min(max(x0 - O0 + cc, 0), W - 1);
            tile[r * TW + cc] = __ldg(frame + (size_t)gy * W + gx);
        }
        __syncthreads();

        if (py < H) {
            const float2* wrow = tile + warp * TW;   // window of pixel p: Γ(i,k) = wrow[i*TW + p + k]
            cx2 R[M];                                // lane i: row i of R_y
            bool rebuild = true;                     // full R at the segment start / after non-finite data
#pragma unroll 1
            for (int p = 0; p < kBX; ++p) {
                const int px = x0 + p;
                if (px >= W) break;                  // warp-uniform
                // ---- a2: R_y row `ri` (full at the segment start, then rank-2 slides) ----
                if (rebuild) {
#pragma unroll
                    for (int j = 0; j < M; ++j) R[j] = 0ull;
#pragma unroll 1
                    for (int k = p; k < p + M; ++k) {
                        const float2 g = wrow[ri * TW + k];
                        const cx2 A = cx2_make(g.x, g.y), Anj = cx2_make(g.y, -g.x);
#pragma unroll
                        for (int j = 0; j < M; ++j) {
                            const float2 b = wrow[j * TW + k];
                            R[j] = fma2(cx2_bcast(b.x), A, fma2(cx2_bcast(b.y), Anj, R[j]));
                        }
                    }
                } else {
                    const float2 go = wrow[ri * TW + p - 1], gn = wrow[ri * TW + p + M - 1];
                    const cx2 Ao = cx2_make(go.x, go.y), Aonj = cx2_make(go.y, -go.x);
                    const cx2 An = cx2_make(gn.x, gn.y), Annj = cx2_make(gn.y, -gn.x);
#pragma unroll
                    for (int j = 0; j < M; ++j) {
                        const float2 bo = wrow[j * TW + p - 1], bn = wrow[j * TW + p + M - 1];
                        R[j] = fma2(cx2_bcast(bn.x), An, fma2(cx2_bcast(bn.y), Annj, R[j]));
                        R[j] = fma2(cx2_bcast(-bo.x), Ao, fma2(cx2_bcast(-bo.y), Aonj, R[j]));
                    }
                }
                // diagonal element R_ii of this lane's row
                float dii = 0.0f;
#pragma unroll
                for (int j = 0; j < M; ++j)
                    if (j == lane) dii = cx2_re(R[j]);
                const float trace = warp_sum(rl ? dii : 0.0f);

                uint8_t fl = 0;
                if (py - O0 < 0 || py + (M - 1 - O0) > H - 1 || px - O0 < 0 || px + (M - 1 - O0) > W - 1)
                    fl |= kFlagBorder;
                float result, wx = CUDART_NAN_F, wy = CUDART_NAN_F;
                int n_pow = 0, n_aby = 0, n_abx = 0;
                // NaN/Inf never leave R by subtraction; the FB variant overwrites R (no slide)
                rebuild = FB || !isfinite(trace);
                if (!isfinite(trace)) {
                    fl |= kFlagNonfinite;
                    result = CUDART_NAN_F;
                } else {
                    // ---- a3: power iteration, lane i holds u_i ----
                    if (FB) fb_average_rows<M>(R, ri);
                    cx2 u;
                    bool pow_ok = false;
                    bool weak = false;                          // see kLowSnrRatio
                    if constexpr (FB) {
                        float lam;
                        n_pow = power_iteration_warp_fb<M>(R, lane, rl, va, u, pow_ok, trace, lam);
                        weak = lam < kLowSnrRatio * trace;
                    } else {
                        float lam;
                        n_pow = power_iteration_warp<M>(R, lane, rl, va, u, pow_ok, lam);
                        weak = lam < kLowSnrRatio * trace;
                    }
                    cx2 v = 0ull;
                    if (!FB) {
                        // v_1 ∝ Γ_w^H u_1, lane k holds v_k
                        if (rl) va[lane] = u;
                        __syncwarp();
#pragma unroll
                        for (int i = 0; i < M; ++i) {
                            const float2 g = wrow[i * TW + p + ri];
                            const cx2 ui = va[i];
                            const cx2 uinj = mul2(cx2_make(cx2_im(ui), cx2_re(ui)), kPosNeg);
                            v = fma2(cx2_bcast(g.x), ui, fma2(cx2_bcast(g.y), uinj, v));
                        }
                        if (!rl) v = 0ull;
                        v = mul2(v, cx2_bcast(rsqrtf(warp_sum(cabs2(cx2_f2(v))))));
                    } else {
                        // variant f4: S = Σ_i row_i row_i^H = conj(Γ_w^H Γ_w), lane k holds row k:
                        // S_kl = Σ_i Γ(i,k) conj(Γ(i,l)); v_1 = conj(dominant eigenvector of FB(S))
#pragma unroll
                        for (int j = 0; j < M; ++j) R[j] = 0ull;
#pragma unroll 1
                        for (int i = 0; i < M; ++i) {
                            const float2 g = wrow[i * TW + p + ri];
                            const cx2 A = cx2_make(g.x, g.y), Anj = cx2_make(g.y, -g.x);
#pragma unroll
                            for (int j = 0; j < M; ++j) {
                                const float2 b = wrow[i * TW + p + j];
                                R[j] = fma2(cx2_bcast(b.x), A, fma2(cx2_bcast(b.y), Anj, R[j]));
                            }
                        }
                        fb_average_rows<M>(R, ri);
                        bool pow2_ok = false;
                        float lam2;
                        n_pow += power_iteration_warp_fb<M>(R, lane, rl, va, v, pow2_ok, trace, lam2);
                        pow_ok = pow_ok && pow2_ok;
                        v = f2_cx2(cconj(cx2_f2(v)));
                    }
                    __syncwarp();

                    // ---- a4 + a5 per axis ----
                    float2 zy = make_float2(0.0f, 0.0f), zx = make_float2(0.0f, 0.0f);
                    float my = CUDART_INF_F, mx = CUDART_INF_F;
                    bool aby_ok = false, abx_ok = false;
#pragma unroll 1
                    for (int axis = 0; axis < 2; ++axis) {
                        const cx2 q = axis ? v : u;
                        if (rl) va[lane] = q;                    // va[M..63] = 0
                        __syncwarp();
                        // lane d: r_d = Σ_i q_i conj(q_{i+d}) = Σ_i re(q_{i+d})·q_i + im(q_{i+d})·(−j q_i)
                        const int d = lane;
                        cx2 r = 0ull;
#pragma unroll
                        for (int i = 0; i < M - 1; ++i) {
                            const cx2 qi = va[i];                                    // broadcast
                            const cx2 qinj = mul2(cx2_make(cx2_im(qi), cx2_re(qi)), kPosNeg);   // −j·q_i
                            const cx2 qid = va[i + d];                               // 0 beyond M
                            r = fma2(cx2_bcast(cx2_re(qid)), qi, fma2(cx2_bcast(cx2_im(qid)), qinj, r));
                        }
                        const float n2 = warp_sum(cabs2(cx2_f2(q)));
                        const float2 rf = cx2_f2(r);
                        if (lane == 0) coef[M - 1] = cx2_make(float(M) - n2, 0.0f);
                        if (d >= 1 && d < M) {
                            coef[M - 1 + d] = cx2_make(-rf.x, -rf.y);
                            coef[M - 1 - d] = cx2_make(-rf.x, rf.y);
                        }
                        const float2 r1q = cx2_f2(shfl_cx2(r, 1));
                        float2 rot = make_float2(1.0f, 0.0f);
                        if (cabs2(r1q) > 0.0f) rot = cscale(cconj(r1q), rsqrtf(cabs2(r1q)));
                        __syncwarp();                          // coef written, va free again
                        // Aberth–Ehrlich, lane k owns root k (simultaneous update)
                        float2 z = kl ? cmul(kTemplateRoots[bos_template_offset(M) + lane], rot) : make_float2(0.0f, 0.0f);
                        cx2 zp = f2_cx2(z);
                        int it = 0;
                        bool ok = false;
                        float tol2 = weak ? kAberthLowSnrTol2 : kAberthTol2Wide;
                        float2 zb, z2;
                        float marg;
                        int sl;
#pragma unroll 1
                        for (int attempt = 0;; ++attempt) {      // warp-uniform (see demod_kernel.cuh)
                        for (int sweep = 0; sweep < kAberthMaxIt; ++sweep, ++it) {
                            if (kl) {
                                va[lane] = zp;
                                vb[lane] = mirror(zp);
                            }
                            __syncwarp();
                            const float2 ratio = newton_ratio_smem<N>(coef, z);
                            const bool near = fabsf(1.0f - cabs2(z)) < kNearCircle;
                            const cx2 ziC = mul2(zp, kPosNeg);
                            cx2 s = 0ull;
#pragma unroll (wide_unroll<N>())
                            for (int j = 0; j < K; ++j) {
                                // 1/(z − z_j) = conj(d)/|d|²; the own term gets |d|² = ∞ → 0
                                const cx2 d1 = fma2(va[j], kNegPos, ziC);
                                float q1 = fmaf(cx2_re(d1), cx2_re(d1), cx2_im(d1) * cx2_im(d1));
                                q1 = (j == lane) ? CUDART_INF_F : q1;
                                s = fma2(cx2_bcast(rcp_approx(q1)), d1, s);
                                const cx2 d2 = fma2(vb[j], kNegPos, ziC);
                                float q2 = fmaf(cx2_re(d2), cx2_re(d2), cx2_im(d2) * cx2_im(d2));
                                q2 = (j == lane && near) ? CUDART_INF_F : q2;
                                s = fma2(cx2_bcast(rcp_approx(q2)), d2, s);
                            }
                            const float2 sf = cx2_f2(s);
                            const float2 dd = make_float2(1.0f - (ratio.x * sf.x - ratio.y * sf.y),
                                                          -(ratio.x * sf.y + ratio.y * sf.x));
                            float2 w = cdiv(ratio, dd);
                            if (near) w = newton_on_derivative_smem<N>(coef, z);
                            float w2 = cabs2(w);
                            if (!(w2 < 1e30f) || !kl) {
                                w = make_float2(0.0f, 0.0f);
                                w2 = 0.0f;
                            }
                            z = csub(z, w);
                            zp = f2_cx2(z);
                            __syncwarp();                      // everyone has read va/vb
                            const float n2 = (kl && !near) ? cabs2(ratio) : 0.0f;   // Newton-ratio stop always on here (see newton_stop)
                            if (warp_max(fmaxf(w2, n2 < 1e30f ? n2 : CUDART_INF_F)) < tol2) { ok = true; ++it; break; }
                        }
                        // selection: argmin |log2 |z|²| over lanes, margin to a different frequency
                        const float r2 = cabs2(z);
                        const float dl = kl ? fabsf(__log2f(r2)) : CUDART_INF_F;
                        const float best = warp_min(dl);
                        const int bl = __ffs(__ballot_sync(0xffffffffu, dl == best)) - 1;
                        zb = cx2_f2(shfl_cx2(zp, bl < 0 ? 0 : bl));
                        if (!(best < CUDART_INF_F)) zb = make_float2(CUDART_NAN_F, CUDART_NAN_F);
                        const float rb2 = cabs2(zb);
                        const float dot = fmaf(z.x, zb.x, z.y * zb.y);
                        const bool distinct = kl && (dot < 0.0f || dot * dot < kCos2TauOmega * r2 * rb2);
                        const float dd2 = distinct ? dl : CUDART_INF_F;
                        const float second = warp_min(dd2);
                        marg = (second - best) * 0.34657359f;
                        sl = __ffs(__ballot_sync(0xffffffffu, dd2 == second && second < CUDART_INF_F)) - 1;
                        z2 = cx2_f2(shfl_cx2(zp, sl < 0 ? 0 : sl));
                        const float2 zsel = zb;
#pragma unroll 1
                        for (int t = 0; t < kPolishMax; ++t) {   // warp-uniform: zb is the same on all lanes
                            const float2 wp = newton_ratio_warp<N>(coef, zb, lane);
                            const float w2 = cabs2(wp);
                            if (w2 < 1e30f) zb = csub(zb, wp);
                            if (polish_done(t, w2)) break;
                        }
                        const float dsel = ln_dist(zb), dsec = ln_dist(z2) - 1e-3f;   // see demod_kernel.cuh
                        if (attempt == 0 && (!(dsel <= dsec || !(second < CUDART_INF_F)) ||
                                             !(cabs2(csub(zb, zsel)) <= kMoved2))) {
                            tol2 = kAberthTightTol2;
                            continue;
                        }
                        break;
                        }
                        if (marg < kRefineMargin && sl >= 0) {     // warp-uniform (see demod_kernel.cuh)
#pragma unroll 1
                            for (int t = 0; t < kPolishMax; ++t) {
                                const float2 wp = newton_ratio_warp<N>(coef, z2, lane);
                                const float w2 = cabs2(wp);
                                if (w2 < 1e30f) z2 = csub(z2, wp);
                                if (polish_done(t, w2)) break;
                            }
                            const float d1 = ln_dist(zb), d2 = ln_dist(z2);
                            if (d2 < d1) zb = z2;
                            marg = fabsf(d2 - d1);
                        }
                        __syncwarp();                // coefficient buffer reused by the next axis
                        if (axis == 0) { zy = zb; my = marg; aby_ok = ok; n_aby = it; }
                        else { zx = zb; mx = marg; abx_ok = ok; n_abx = it; }
                    }
                    if (!pow_ok || !aby_ok || !abx_ok || !isfinite(zy.x + zy.y + zx.x + zx.y))
                        fl |= kFlagNonconverged;
                    if (fminf(my, mx) < kTauSel) fl |= kFlagAmbiguous;

                    // ---- a6: Eq.(15); lane i forms row_i = Σ_k Γ(i,k) ẑ_x^{o_k} ----
                    const float2 hx = cscale(zx, rsqrtf(cabs2(zx)));
                    const float2 hy = cscale(zy, rsqrtf(cabs2(zy)));
                    float2 tw = make_float2(1.0f, 0.0f);
#pragma unroll
                    for (int k = 0; k < O0; ++k) tw = cmul(tw, cconj(hx));
                    cx2 row = 0ull;
#pragma unroll
                    for (int k = 0; k < M; ++k) {
                        const float2 g = wrow[ri * TW + p + k];
                        const cx2 T = cx2_make(tw.x, tw.y), Tj = cx2_make(-tw.y, tw.x);
                        row = fma2(cx2_bcast(g.x), T, fma2(cx2_bcast(g.y), Tj, row));
                        tw = cmul(tw, hx);
                    }
                    // q_i = conj(ẑ_y)^{o_i} for this lane's row
                    float2 qy = make_float2(1.0f, 0.0f), qi = qy;
#pragma unroll
                    for (int i = 0; i < O0; ++i) qy = cmul(qy, hy);
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        if (i == lane) qi = qy;
                        qy = cmul(qy, cconj(hy));
                    }
                    float2 cs = rl ? cmul(cx2_f2(row), qi) : make_float2(0.0f, 0.0f);
                    cs = warp_sum2(cs);
                    if (!(cabs2(cs) >= kLowAmp * kLowAmp * float(M * M) * trace)) fl |= kFlagLowAmplitude;
                    float a = atan2f(cs.y, cs.x);
                    if (omx != nullptr) wx = -atan2f(zx.y, zx.x);   // Eq.(15)
                    if (omy != nullptr) wy = atan2f(zy.y, zy.x);
                    if (ref != nullptr) a -= __ldg(ref + (size_t)py * W + px);
                    if (a > CUDART_PI_F) a -= 2.0f * CUDART_PI_F;
                    if (a <= -CUDART_PI_F) a += 2.0f * CUDART_PI_F;
                    result = a;
                }
                if (lane == 0) {
                    const size_t o = (size_t)f * plane + (size_t)py * W + px;
                    out[o] = result;
                    if (flags != nullptr) flags[o] = fl;
                    if (omx != nullptr) omx[o] = wx;
                    if (omy != nullptr) omy[o] = wy;
                    if (COUNT) {
                        atomicAdd(counters + 0, 1ull);
                        atomicAdd(counters + 1, (unsigned long long)n_pow);
                        atomicAdd(counters + 2, (unsigned long long)n_aby);
                        atomicAdd(counters + 3, (unsigned long long)n_abx);
                    }
                }
            }
        }
        __syncthreads();
    }
}

}  // namespace bos
