// demod_ss.cuh — SURVEY §8 row f4, the reduced-order (spatially smoothed) covariance variant
// (NOT in the paper, [R14]): FP32, thread per pixel, for a window of any M ≤ 32 (runtime) and
// a subarray order m = MS ≤ 16 (compile time).  The covariances of order m average the outer
// products of all length-m segments of the window's columns (R_y) and conjugated rows (R_x);
// their dominant eigenvectors (power iteration) give polynomials of degree 2m − 2 instead of
// 2M − 2, so the rooting — the dominant cost of the paper path — shrinks with m, and m = 3
// needs no iteration at all: the quartic is solved in closed form (Ferrari, FP64 — a few
// hundred double operations per axis) and the selected root is polished in FP32.  Eq.(15)
// still uses the whole M×M window.  Staging: per-warp clamped halo rows in dynamic shared
// memory, as in demod_kernel.cuh.  Shares that file's helpers (included first).
#pragma once
#include "demod_kernel.cuh"

namespace bos {
namespace ss {

// ---- FP64 complex helpers for the closed-form quartic ----
struct zd {
    double re, im;
};
__device__ __forceinline__ zd zmk(double r, double i) { return zd{r, i}; }
__device__ __forceinline__ zd zadd(zd a, zd b) { return zmk(a.re + b.re, a.im + b.im); }
__device__ __forceinline__ zd zsub(zd a, zd b) { return zmk(a.re - b.re, a.im - b.im); }
__device__ __forceinline__ zd zmul(zd a, zd b) { return zmk(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re); }
__device__ __forceinline__ zd zscl(zd a, double s) { return zmk(a.re * s, a.im * s); }
__device__ __forceinline__ double zabs(zd a) { return hypot(a.re, a.im); }
__device__ __forceinline__ zd zdiv(zd a, zd b) {
    const double d = b.re * b.re + b.im * b.im;
    return zmk((a.re * b.re + a.im * b.im) / d, (a.im * b.re - a.re * b.im) / d);
}
__device__ __forceinline__ zd zsqrt(zd a) {        // principal branch
    const double r = zabs(a);
    const double re = sqrt(fmax(0.5 * (r + a.re), 0.0));
    const double im = copysign(sqrt(fmax(0.5 * (r - a.re), 0.0)), a.im);
    return zmk(re, im);
}
__device__ __forceinline__ zd zcbrt(zd a) {        // principal branch
    const double r = cbrt(zabs(a)), t = atan2(a.im, a.re) / 3.0;
    double s, c;
    sincos(t, &s, &c);
    return zmk(r * c, r * s);
}

// Roots of c0 + c1 z + c2 z² + c3 z³ + c4 z⁴ (Ferrari): depressed quartic y⁴ + p y² + q y + r
// (z = y − A/4), resolvent cubic m³ + p m² + (p²/4 − r) m − q²/8 = 0 (Cardano; the cube root
// of the largest |m| of the three is used), then the two quadratics
// y² ∓ s y + p/2 + m ± q/(2s) = 0, s = √(2m).  q = 0: the biquadratic.
__device__ inline void quartic_roots(const cx2 (&c)[5], float2 (&z)[4]) {
    zd k[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) k[i] = zmk(cx2_re(c[i]), cx2_im(c[i]));
    const zd A = zdiv(k[3], k[4]), B = zdiv(k[2], k[4]), C = zdiv(k[1], k[4]), D = zdiv(k[0], k[4]);
    const zd A2 = zmul(A, A);
    const zd p = zsub(B, zscl(A2, 3.0 / 8.0));
    const zd q = zadd(zsub(C, zscl(zmul(A, B), 0.5)), zscl(zmul(A2, A), 1.0 / 8.0));
    const zd r = zadd(zsub(D, zscl(zmul(A, C), 0.25)),
                      zsub(zscl(zmul(A2, B), 1.0 / 16.0), zscl(zmul(A2, A2), 3.0 / 256.0)));
    zd y[4];
    const double scale = zabs(p) * zabs(p) + zabs(r) + 1e-300;
    if (zabs(q) * zabs(q) <= 1e-28 * scale * zabs(p) + 1e-300) {
        const zd d = zsqrt(zsub(zmul(p, p), zscl(r, 4.0)));
        const zd w1 = zscl(zsub(d, p), 0.5), w2 = zscl(zadd(d, p), -0.5);
        y[0] = zsqrt(w1);
        y[1] = zscl(y[0], -1.0);
        y[2] = zsqrt(w2);
        y[3] = zscl(y[2], -1.0);
    } else {
        const zd a2 = p, a1 = zsub(zscl(zmul(p, p), 0.25), r), a0 = zscl(zmul(q, q), -1.0 / 8.0);
        const zd P = zsub(a1, zscl(zmul(a2, a2), 1.0 / 3.0));
        const zd Q = zadd(zsub(zscl(zmul(zmul(a2, a2), a2), 2.0 / 27.0), zscl(zmul(a2, a1), 1.0 / 3.0)), a0);
        const zd sd = zsqrt(zadd(zscl(zmul(Q, Q), 0.25), zscl(zmul(zmul(P, P), P), 1.0 / 27.0)));
        const zd wa = zadd(zscl(Q, -0.5), sd), wb = zsub(zscl(Q, -0.5), sd);
        const zd u0 = zcbrt(zabs(wa) >= zabs(wb) ? wa : wb);
        const zd om = zmk(-0.5, 0.86602540378443865);
        zd m = zmk(0.0, 0.0), u = u0;
#pragma unroll 1
        for (int b = 0; b < 3; ++b) {
            const zd t = zabs(u) > 0.0 ? zsub(u, zdiv(P, zscl(u, 3.0))) : zmk(0.0, 0.0);
            const zd mb = zsub(t, zscl(a2, 1.0 / 3.0));
            if (zabs(mb) > zabs(m)) m = mb;
            u = zmul(u, om);
        }
        const zd s = zsqrt(zscl(m, 2.0));
        const zd h = zadd(zscl(p, 0.5), m), qs = zdiv(q, zscl(s, 2.0));
        const zd e1 = zadd(h, qs), e2 = zsub(h, qs);          // y² − s y + e1,  y² + s y + e2
        const zd d1 = zsqrt(zsub(zmul(s, s), zscl(e1, 4.0))), d2 = zsqrt(zsub(zmul(s, s), zscl(e2, 4.0)));
        y[0] = zscl(zadd(s, d1), 0.5);
        y[1] = zscl(zsub(s, d1), 0.5);
        y[2] = zscl(zadd(zscl(s, -1.0), d2), 0.5);
        y[3] = zscl(zsub(zscl(s, -1.0), d2), 0.5);
    }
    const zd sh = zscl(A, 0.25);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const zd zz = zsub(y[i], sh);
        z[i] = make_float2((float)zz.re, (float)zz.im);
    }
}

// Order-MS covariance from the per-warp halo tile (runtime window M, row stride TW):
// ROWS = false: R_y = Σ_{s,k} x x^H, x_i = Γ(s+i, k);  ROWS = true: R_x = Σ_{s,i} y y^H,
// y_k = conj(Γ(i, s+k)).  Diagonal + strict lower triangle, two FFMA2 per entry.
template <int MS, bool ROWS>
__device__ __forceinline__ void ss_covariance(const float2* win, int M, int TW, float (&Rd)[MS],
                                              cx2 (&Ro)[MS * (MS - 1) / 2 > 0 ? MS * (MS - 1) / 2 : 1]) {
    constexpr int NOFF = MS * (MS - 1) / 2;
#pragma unroll
    for (int i = 0; i < MS; ++i) Rd[i] = 0.0f;
#pragma unroll
    for (int t = 0; t < NOFF; ++t) Ro[t] = 0ull;
    const cx2 kPosNeg = cx2_make(1.0f, -1.0f);
#pragma unroll 1
    for (int k = 0; k < M; ++k) {
#pragma unroll 1
        for (int s = 0; s + MS <= M; ++s) {
            cx2 col[MS], colnj[MS];
#pragma unroll
            for (int i = 0; i < MS; ++i) {
                float2 g = ROWS ? win[k * TW + s + i] : win[(s + i) * TW + k];
                if (ROWS) g.y = -g.y;                                // conjugated row segment
                col[i] = cx2_make(g.x, g.y);
                colnj[i] = mul2(cx2_make(g.y, g.x), kPosNeg);
                Rd[i] = fmaf(g.x, g.x, fmaf(g.y, g.y, Rd[i]));
            }
#pragma unroll
            for (int i = 1; i < MS; ++i) {
#pragma unroll
                for (int j = 0; j < i; ++j) {
                    cx2& r = Ro[tri_off<MS>(i, j)];
                    r = fma2(cx2_bcast(cx2_re(col[j])), col[i], fma2(cx2_bcast(cx2_im(col[j])), colnj[i], r));
                }
            }
        }
    }
}

// One axis: q (the order-MS eigenvector) → polynomial → roots → selected root, margin.
template <int MS>
__device__ __forceinline__ float2 ss_root(const float2 (&q)[MS], float& marg, bool& ok, int& its) {
    constexpr int N = 2 * MS - 2;
    cx2 c[N + 1];
    const float2 rot = music_coeffs<MS>(q, c);
    float2 zs, z2;
    marg = CUDART_INF_F;
    if constexpr (MS == 3) {
        float2 zr[4];
        quartic_roots(c, zr);
        // the two inside members of the mirror pairs (z, 1/z̄): the two smallest |z|
        int a = 0;
#pragma unroll
        for (int i = 1; i < 4; ++i)
            if (cabs2(zr[i]) < cabs2(zr[a])) a = i;
        int b = a == 0 ? 1 : 0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (i != a && cabs2(zr[i]) < cabs2(zr[b])) b = i;
        cx2 zin[2] = {f2_cx2(zr[a]), f2_cx2(zr[b])};
        zs = select_root<2>(zin, marg, z2);
        ok = isfinite(zs.x + zs.y);
        its = 0;
        for (int t = 0; t < kPolishMax; ++t) {
            const float2 w = polish_step<N>(c, zs);
            const float w2 = cabs2(w);
            if (w2 < 1e30f) zs = csub(zs, w);
            if (polish_done(t, w2)) break;
        }
    } else {
        cx2 z[N / 2];
#pragma unroll
        for (int j = 0; j < N / 2; ++j) z[j] = f2_cx2(cmul(kTemplateRoots[bos_template_offset(MS) + j], rot));
        float tol2 = kAberthTol2;
        its = 0;
#pragma unroll 1
        for (int attempt = 0;; ++attempt) {
            its += aberth_sym<N, true>(c, z, ok, tol2);
            zs = select_root<N / 2>(z, marg, z2);
            const float2 zsel = zs;
#pragma unroll 1
            for (int t = 0; t < kPolishMax; ++t) {
                const float2 w = polish_step<N>(c, zs);
                const float w2 = cabs2(w);
                if (w2 < 1e30f) zs = csub(zs, w);
                if (polish_done(t, w2)) break;
            }
            const float dsel = ln_dist(zs), dsec = ln_dist(z2) - 1e-3f;
            if (attempt == 0 && (!(dsel <= dsec || marg == CUDART_INF_F) || !(cabs2(csub(zs, zsel)) <= kMoved2))) {
                tol2 = kAberthTightTol2;
                continue;
            }
            break;
        }
    }
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
    return zs;
}

template <int MS, bool FB>
__global__ void __launch_bounds__(kThreads, min_blocks_per_sm<MS>())
demod_ss_kernel(const float2* __restrict__ frames, int n_frames, int H, int W, int M,
                const float* __restrict__ ref, float* __restrict__ out, uint8_t* __restrict__ flags,
                float* __restrict__ omx, float* __restrict__ omy) {
    constexpr int NOFF = MS * (MS - 1) / 2;
    extern __shared__ float2 ss_tiles[];
    const int O0 = (M - 1) / 2;                  // o_i = i − O0  [R2]
    const int TW = kBX + M - 1;
    float2* tile = ss_tiles + (size_t)threadIdx.y * M * TW;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int x0 = blockIdx.x * kBX, y0 = blockIdx.y * kBY;
    const int px = x0 + tx, py = y0 + ty;
    const size_t plane = (size_t)H * (size_t)W;
    if (py >= H) return;                         // warp-uniform

    for (int f = blockIdx.z; f < n_frames; f += gridDim.z) {
        const float2* __restrict__ frame = frames + (size_t)f * plane;
        {   // ---- a1: clamped halo rows of this warp ----
            const int gx0 = min(max(x0 - O0 + tx, 0), W - 1);
            const int gx1 = min(max(x0 - O0 + tx + kBX, 0), W - 1);
#pragma unroll 1
            for (int r = 0; r < M; ++r) {
                const float2* __restrict__ row = frame + (size_t)min(max(py - O0 + r, 0), H - 1) * W;
                tile[r * TW + tx] = __ldg(row + gx0);
                if (tx + kBX < TW) tile[r * TW + tx + kBX] = __ldg(row + gx1);
            }
        }
        __syncwarp();
        if (px < W) {
            const float2* win = tile + tx;
            uint8_t fl = 0;
            if (py - O0 < 0 || py + (M - 1 - O0) > H - 1 || px - O0 < 0 || px + (M - 1 - O0) > W - 1)
                fl |= kFlagBorder;
            float Rd[MS];
            cx2 Ro[NOFF > 0 ? NOFF : 1];
            ss_covariance<MS, false>(win, M, TW, Rd, Ro);
            float trace = 0.0f;
#pragma unroll
            for (int i = 0; i < MS; ++i) trace += Rd[i];
            float result, wx = CUDART_NAN_F, wy = CUDART_NAN_F;
            if (!isfinite(trace)) {             // every window sample is in some snapshot
                fl |= kFlagNonfinite;
                result = CUDART_NAN_F;
            } else {
                // ---- a3: dominant eigenvectors of the order-m covariances ----
                cx2 e[MS];
                bool ok_y = false, ok_x = false;
                float lam;
                if (FB) fb_average<MS>(Rd, Ro);
                if (FB) power_iteration_fb<MS>(Rd, Ro, e, ok_y, kPowerTolSS);
                else power_iteration<MS>(Rd, Ro, e, ok_y, lam, kPowerTolSS);
                float2 u[MS], v[MS];
#pragma unroll
                for (int i = 0; i < MS; ++i) u[i] = cx2_f2(e[i]);
                ss_covariance<MS, true>(win, M, TW, Rd, Ro);
                if (FB) fb_average<MS>(Rd, Ro);
                if (FB) power_iteration_fb<MS>(Rd, Ro, e, ok_x, kPowerTolSS);
                else power_iteration<MS>(Rd, Ro, e, ok_x, lam, kPowerTolSS);
#pragma unroll
                for (int i = 0; i < MS; ++i) v[i] = cx2_f2(e[i]);
                // ---- a4 + a5 ----
                float my, mx;
                bool aby_ok, abx_ok;
                int its;
                const float2 zy = ss_root<MS>(u, my, aby_ok, its);
                const float2 zx = ss_root<MS>(v, mx, abx_ok, its);
                if (!ok_y || !ok_x || !aby_ok || !abx_ok || !isfinite(zy.x + zy.y + zx.x + zx.y))
                    fl |= kFlagNonconverged;
                if (fminf(my, mx) < kTauSel) fl |= kFlagAmbiguous;
                // ---- a6: Eq.(15) over the whole M×M window ----
                const float2 hx = cscale(zx, rsqrtf(cabs2(zx)));
                const float2 hy = cscale(zy, rsqrtf(cabs2(zy)));
                float2 tx0 = make_float2(1.0f, 0.0f), qy = make_float2(1.0f, 0.0f);
#pragma unroll 1
                for (int k = 0; k < O0; ++k) {
                    tx0 = cmul(tx0, cconj(hx));
                    qy = cmul(qy, hy);
                }
                float2 csum = make_float2(0.0f, 0.0f);
                float fro = 0.0f;
#pragma unroll 1
                for (int i = 0; i < M; ++i) {
                    float2 row = make_float2(0.0f, 0.0f), tw = tx0;
#pragma unroll 4
                    for (int k = 0; k < M; ++k) {
                        const float2 g = win[i * TW + k];
                        row = cfma(g, tw, row);
                        fro = fmaf(g.x, g.x, fmaf(g.y, g.y, fro));
                        tw = cmul(tw, hx);
                    }
                    csum = cfma(row, qy, csum);
                    qy = cmul(qy, cconj(hy));
                }
                if (!(cabs2(csum) >= kLowAmp * kLowAmp * float(M) * float(M) * fro)) fl |= kFlagLowAmplitude;
                float a = atan2f(csum.y, csum.x);
                if (omx != nullptr) wx = -atan2f(zx.y, zx.x);
                if (omy != nullptr) wy = atan2f(zy.y, zy.x);
                if (ref != nullptr) a -= __ldg(ref + (size_t)py * W + px);
                if (a > CUDART_PI_F) a -= 2.0f * CUDART_PI_F;
                if (a <= -CUDART_PI_F) a += 2.0f * CUDART_PI_F;
                result = a;
            }
            const size_t o = (size_t)f * plane + (size_t)py * W + px;
            out[o] = result;
            if (flags != nullptr) flags[o] = fl;
            if (omx != nullptr) omx[o] = wx;
            if (omy != nullptr) omy[o] = wy;
        }
        __syncwarp();                            // tile reused by the next frame
    }
}

}  // namespace ss
}  // namespace bos
