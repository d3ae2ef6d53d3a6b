// demod_f64.cuh — SURVEY §8 row f4, "an FP64 GPU path" (not in the paper, whose GPU code is
// FP32): Algorithm 1 per pixel in double precision, written for accuracy, not
// speed — the high-accuracy companion of the FP32 hot path (demod_kernel.cuh,
// demod_wide.cuh).  One thread per pixel; the window, the Hermitian matrices and the roots
// live in thread-local arrays (local memory, L1-cached):
//
//   a1  Γ_w: M×M clamped window [R1], promoted to double;
//   a2  R_y = Γ_wΓ_w^H and R_x = Γ_w^HΓ_w (Eq.(4) and its x counterpart; the eigenvectors of
//       these are the SVD's U and V), or their spatially smoothed order-m versions
//       ([R14]), optionally forward–backward averaged (FB, [R13]);
//   a3  cyclic complex Jacobi eigen-decomposition of each (rotations until the off-diagonal
//       norm is below 1e-15 of the Frobenius norm) → u_1, v_1 = eigenvectors of the largest
//       eigenvalue, and λ1/λ2 for the SMALL_GAP flag (the FP32 kernels cannot emit it);
//   a4  polynomial coefficients from the autocorrelation of u_1 / v_1 (Eqs.(12),(13));
//   a5  all 2M−2 roots by Gauss–Seidel Aberth–Ehrlich in double, each root frozen once
//       |P(z)| is within the Horner rounding bound 4nε·Σ|c_k||z|^k (the attainable accuracy,
//       so near-double roots stop at their √ε split like the oracle's QR); selection
//       argmin |ln|z|| [R6] with the distinct-frequency margin [R8];
//   a6  Eq.(15) with twiddles = powers of z/|z|;  a7 reference difference, wrap, flags.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "template_roots.h"

namespace bos {
namespace f64 {

struct cd {
    double re, im;
};
__device__ __forceinline__ cd mk(double r, double i) { return cd{r, i}; }
__device__ __forceinline__ cd add(cd a, cd b) { return mk(a.re + b.re, a.im + b.im); }
__device__ __forceinline__ cd sub(cd a, cd b) { return mk(a.re - b.re, a.im - b.im); }
__device__ __forceinline__ cd mul(cd a, cd b) { return mk(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re); }
__device__ __forceinline__ cd cj(cd a) { return mk(a.re, -a.im); }
__device__ __forceinline__ cd scl(cd a, double s) { return mk(a.re * s, a.im * s); }
__device__ __forceinline__ double abs2(cd a) { return a.re * a.re + a.im * a.im; }
__device__ __forceinline__ cd dvd(cd a, cd b) {
    const double d = abs2(b);
    return mk((a.re * b.re + a.im * b.im) / d, (a.im * b.re - a.re * b.im) / d);
}
__device__ __forceinline__ double wrap_pi(double a) {
    return a - 2.0 * CUDART_PI * ceil((a - CUDART_PI) / (2.0 * CUDART_PI));
}

constexpr int kJacobiMaxSweeps = 40;
constexpr double kJacobiTol2 = 1e-30;     // off² ≤ 1e-30·‖R‖_F²  (1e-15 relative)
constexpr int kAberthMaxIt = 500;
constexpr double kEps = 1.1102230246251565e-16;
constexpr double kTauSel = 1e-3, kTauOmega = 1e-2, kGammaMin = 1.3, kLowAmp = 1e-4;

// Covariance of order m ≤ M from the window g (M×M, row-major), full Hermitian storage
// (row-major m×m).  ROWS = false: R_y = Σ_{s,k} x x^H with x = Γ[s:s+m, k] (m = M: Γ Γ^H);
// ROWS = true: R_x = Σ_{s,i} y y^H with y = conj(Γ[i, s:s+m]) (m = M: Γ^H Γ).  m < M is the
// spatially smoothed covariance of row f4 ([R14]).
template <int M, bool ROWS>
__device__ void gram(const cd* __restrict__ g, int m, cd* __restrict__ R) {
#pragma unroll 1
    for (int a = 0; a < m; ++a) {
#pragma unroll 1
        for (int b = 0; b <= a; ++b) {
            cd s = mk(0.0, 0.0);
#pragma unroll 1
            for (int o = 0; o + m <= M; ++o) {
#pragma unroll 4
                for (int t = 0; t < M; ++t) {
                    const cd x = ROWS ? cj(g[t * M + o + a]) : g[(o + a) * M + t];
                    const cd y = ROWS ? cj(g[t * M + o + b]) : g[(o + b) * M + t];
                    s = add(s, mul(x, cj(y)));
                }
            }
            R[a * m + b] = s;
            R[b * m + a] = cj(s);
        }
        R[a * m + a].im = 0.0;
    }
}

// Forward–backward average ½(R + J R* J): R_ij ← ½(R_ij + conj(R_{M−1−i, M−1−j})).
__device__ inline void fb_average(cd* R, int M) {
#pragma unroll 1
    for (int i = 0; i < M; ++i) {
#pragma unroll 1
        for (int j = 0; j < M; ++j) {
            const int i2 = M - 1 - i, j2 = M - 1 - j;
            if (i * M + j > i2 * M + j2) continue;                // each mirror pair once
            const cd a = R[i * M + j], b = R[i2 * M + j2];
            const cd n = scl(add(a, cj(b)), 0.5);
            R[i * M + j] = n;
            R[i2 * M + j2] = cj(n);
        }
    }
}

// Cyclic Jacobi for a Hermitian R (destroyed: diagonal → eigenvalues); V ← eigenvectors in
// columns.  Each rotation: phase column/row q so that R_pq = |R_pq| is real, then the real
// symmetric rotation t = sgn(θ)/(|θ| + √(θ²+1)), θ = (R_qq − R_pp)/(2|R_pq|).
__device__ inline bool jacobi(cd* R, cd* V, int M) {
#pragma unroll 1
    for (int i = 0; i < M * M; ++i) V[i] = mk(0.0, 0.0);
#pragma unroll 1
    for (int i = 0; i < M; ++i) V[i * M + i] = mk(1.0, 0.0);
#pragma unroll 1
    for (int sweep = 0; sweep < kJacobiMaxSweeps; ++sweep) {
        double off = 0.0, dia = 0.0;
#pragma unroll 1
        for (int p = 0; p < M; ++p) {
            dia += R[p * M + p].re * R[p * M + p].re;
#pragma unroll 1
            for (int q = p + 1; q < M; ++q) off += 2.0 * abs2(R[p * M + q]);
        }
        if (off <= kJacobiTol2 * (dia + off)) return true;
#pragma unroll 1
        for (int p = 0; p < M - 1; ++p) {
#pragma unroll 1
            for (int q = p + 1; q < M; ++q) {
                const cd apq = R[p * M + q];
                const double g = sqrt(abs2(apq));
                if (!(g > 0.0)) continue;
                const cd w = scl(apq, 1.0 / g);                  // e^{jφ}
                // phase: column q × conj(w), row q × w (R_qq unchanged), V column q × conj(w)
#pragma unroll 1
                for (int r = 0; r < M; ++r) {
                    if (r != q) {
                        R[r * M + q] = mul(R[r * M + q], cj(w));
                        R[q * M + r] = mul(R[q * M + r], w);
                    }
                    V[r * M + q] = mul(V[r * M + q], cj(w));
                }
                const double app = R[p * M + p].re, aqq = R[q * M + q].re;
                const double th = (aqq - app) / (2.0 * g);
                const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
#pragma unroll 1
                for (int r = 0; r < M; ++r) {
                    if (r != p && r != q) {
                        const cd arp = R[r * M + p], arq = R[r * M + q];
                        const cd np = sub(scl(arp, c), scl(arq, s));
                        const cd nq = add(scl(arp, s), scl(arq, c));
                        R[r * M + p] = np;
                        R[p * M + r] = cj(np);
                        R[r * M + q] = nq;
                        R[q * M + r] = cj(nq);
                    }
                    const cd vrp = V[r * M + p], vrq = V[r * M + q];
                    V[r * M + p] = sub(scl(vrp, c), scl(vrq, s));
                    V[r * M + q] = add(scl(vrp, s), scl(vrq, c));
                }
                R[p * M + p] = mk(app - t * g, 0.0);
                R[q * M + q] = mk(aqq + t * g, 0.0);
                R[p * M + q] = mk(0.0, 0.0);
                R[q * M + p] = mk(0.0, 0.0);
            }
        }
    }
    return false;
}

// Column of V with the largest eigenvalue → q (normalised); gap = λ1/λ2 (∞ if λ2 ≤ 0).
__device__ inline void top_eigvec(const cd* R, const cd* V, int M, cd* q, double& gap) {
    int b = 0;
#pragma unroll 1
    for (int i = 1; i < M; ++i)
        if (R[i * M + i].re > R[b * M + b].re) b = i;
    double l2 = -CUDART_INF;
#pragma unroll 1
    for (int i = 0; i < M; ++i)
        if (i != b && R[i * M + i].re > l2) l2 = R[i * M + i].re;
    const double l1 = R[b * M + b].re;
    gap = (l2 > 0.0) ? l1 / l2 : CUDART_INF;
#pragma unroll 1
    for (int i = 0; i < M; ++i) q[i] = V[i * M + b];
}

// Eqs.(12),(13): c_{M−1} = M − ‖q‖², c_{M−1+d} = −r_d, c_{M−1−d} = −conj(r_d),
// r_d = Σ_i q_i conj(q_{i+d}) (ascending powers); rot = conj(r_1)/|r_1| (template rotation).
__device__ inline cd coefficients(const cd* q, int M, cd* c) {
    double n2 = 0.0;
#pragma unroll 1
    for (int i = 0; i < M; ++i) n2 += abs2(q[i]);
    c[M - 1] = mk(double(M) - n2, 0.0);
    cd rot = mk(1.0, 0.0);
#pragma unroll 1
    for (int d = 1; d < M; ++d) {
        cd r = mk(0.0, 0.0);
#pragma unroll 1
        for (int i = 0; i + d < M; ++i) r = add(r, mul(q[i], cj(q[i + d])));
        c[M - 1 + d] = mk(-r.re, -r.im);
        c[M - 1 - d] = mk(-r.re, r.im);
        if (d == 1 && abs2(r) > 0.0) rot = scl(cj(r), 1.0 / sqrt(abs2(r)));
    }
    return rot;
}

// All N roots of Σ c_k z^k: Gauss–Seidel Aberth–Ehrlich from the rotated template; a root is
// frozen when |P(z)| ≤ 4Nε·Σ|c_k||z|^k.  Returns false at the iteration cap.
__device__ inline bool aberth_all(const cd* c, int N, cd* z, int toff, cd rot) {
#pragma unroll 1
    for (int k = 0; k < N; ++k) {
        const float2 t = kTemplateRoots[toff + k];
        z[k] = mul(mk(t.x, t.y), rot);
    }
    uint64_t frozen = 0;
    const uint64_t all = (N >= 64) ? ~0ull : ((1ull << N) - 1ull);   // N ≤ 62
#pragma unroll 1
    for (int it = 0; it < kAberthMaxIt; ++it) {
#pragma unroll 1
        for (int k = 0; k < N; ++k) {
            if ((frozen >> k) & 1ull) continue;
            const cd zk = z[k];
            const double az = sqrt(abs2(zk));
            cd p = c[N], dp = mk(0.0, 0.0);
            double bound = sqrt(abs2(c[N]));
#pragma unroll 1
            for (int j = N - 1; j >= 0; --j) {
                dp = add(mul(dp, zk), p);
                p = add(mul(p, zk), c[j]);
                bound = bound * az + sqrt(abs2(c[j]));
            }
            if (sqrt(abs2(p)) <= 4.0 * double(N) * kEps * bound) {
                frozen |= 1ull << k;
                continue;
            }
            cd s = mk(0.0, 0.0);
#pragma unroll 1
            for (int j = 0; j < N; ++j)
                if (j != k) s = add(s, dvd(mk(1.0, 0.0), sub(zk, z[j])));
            const cd nr = dvd(p, dp);                                   // Newton ratio
            const cd w = dvd(nr, sub(mk(1.0, 0.0), mul(nr, s)));        // Aberth correction
            if (abs2(w) < 1e300) z[k] = sub(zk, w);
        }
        if (frozen == all) return true;
    }
    return false;
}

// argmin |ln|z||; margin = min over roots of a different frequency (|wrap(arg − arg_sel)| > τ_ω)
// of |ln|z|| − |ln|z_sel|| ([R6], [R8]).
__device__ inline cd select(const cd* z, int N, double& margin) {
    int b = -1;
    double best = CUDART_INF;
#pragma unroll 1
    for (int k = 0; k < N; ++k) {
        const double d = fabs(0.5 * log(abs2(z[k])));
        if (d < best) { best = d; b = k; }
    }
    if (b < 0) {
        margin = CUDART_INF;
        return mk(CUDART_NAN, CUDART_NAN);
    }
    const double ab = atan2(z[b].im, z[b].re);
    double sec = CUDART_INF;
#pragma unroll 1
    for (int k = 0; k < N; ++k) {
        const double d = fabs(0.5 * log(abs2(z[k])));
        if (fabs(wrap_pi(atan2(z[k].im, z[k].re) - ab)) > kTauOmega && d < sec) sec = d;
    }
    margin = sec - best;
    return z[b];
}

// Local storage per thread: window M², two matrices M², coefficients, roots.
template <int M, bool FB>
__global__ void __launch_bounds__(128)
demod_f64_kernel(const float2* __restrict__ frames, int n_frames, int H, int W, int m, const float* __restrict__ ref,
                 float* __restrict__ out, uint8_t* __restrict__ flags, float* __restrict__ omx,
                 float* __restrict__ omy) {
    constexpr int O0 = (M - 1) / 2;              // o_i = i − O0 [R2]
    const int px = blockIdx.x * 32 + threadIdx.x, py = blockIdx.y * 4 + threadIdx.y;
    if (px >= W || py >= H) return;
    const size_t plane = (size_t)H * (size_t)W;
    cd g[M * M], A[M * M], V[M * M], c[2 * M - 1], z[2 * M - 2], u[M], v[M];   // 50 KB at M = 32
    for (int f = blockIdx.z; f < n_frames; f += gridDim.z) {
        const float2* __restrict__ frame = frames + (size_t)f * plane;
        uint8_t fl = 0;
        if (py - O0 < 0 || py + (M - 1 - O0) > H - 1 || px - O0 < 0 || px + (M - 1 - O0) > W - 1) fl |= 1u << 5;
        // ---- a1 ----
        bool finite = true;
        double fro2 = 0.0;
#pragma unroll 1
        for (int i = 0; i < M; ++i) {
            const int gy = min(max(py - O0 + i, 0), H - 1);
#pragma unroll 1
            for (int k = 0; k < M; ++k) {
                const int gx = min(max(px - O0 + k, 0), W - 1);
                const float2 s = __ldg(frame + (size_t)gy * W + gx);
                finite = finite && isfinite(s.x) && isfinite(s.y);
                g[i * M + k] = mk(s.x, s.y);
                fro2 += double(s.x) * s.x + double(s.y) * s.y;
            }
        }
        double result = CUDART_NAN, wx = CUDART_NAN, wy = CUDART_NAN;
        if (!finite) {
            fl |= 1u << 4;
        } else {
            // ---- a2 + a3 (order m covariances; m = M is Algorithm 1 line 4) ----
            double gap_y, gap_x;
            gram<M, false>(g, m, A);
            if (FB) fb_average(A, m);
            bool ok = jacobi(A, V, m);
            top_eigvec(A, V, m, u, gap_y);
            gram<M, true>(g, m, A);
            if (FB) fb_average(A, m);
            ok = jacobi(A, V, m) && ok;
            top_eigvec(A, V, m, v, gap_x);
            // ---- a4 + a5 per axis (degree 2m − 2) ----
            const int N = 2 * m - 2;
            cd zsel[2];
            double marg = CUDART_INF;
#pragma unroll 1
            for (int axis = 0; axis < 2; ++axis) {
                const cd rot = coefficients(axis ? v : u, m, c);
                ok = aberth_all(c, N, z, bos_template_offset(m), rot) && ok;
                double mg;
                zsel[axis] = select(z, N, mg);
                marg = fmin(marg, mg);
            }
            const cd zy = zsel[0], zx = zsel[1];
            if (!ok || !isfinite(zy.re + zy.im + zx.re + zx.im)) fl |= 1u << 0;
            if (marg < kTauSel) fl |= 1u << 1;
            if (fmin(gap_y, (FB || m < M) ? gap_x : gap_y) < kGammaMin) fl |= 1u << 2;
            // ---- a6: Eq.(15); ẑ_x = e^{−jω_x}, ẑ_y = e^{jω_y} ----
            const cd hx = scl(zx, 1.0 / sqrt(abs2(zx))), hy = scl(zy, 1.0 / sqrt(abs2(zy)));
            cd qy = mk(1.0, 0.0), tx0 = mk(1.0, 0.0);
#pragma unroll 1
            for (int i = 0; i < O0; ++i) {
                qy = mul(qy, hy);
                tx0 = mul(tx0, cj(hx));
            }
            cd sum = mk(0.0, 0.0);
#pragma unroll 1
            for (int i = 0; i < M; ++i) {
                cd row = mk(0.0, 0.0), tw = tx0;
#pragma unroll 1
                for (int k = 0; k < M; ++k) {
                    row = add(row, mul(g[i * M + k], tw));
                    tw = mul(tw, hx);
                }
                sum = add(sum, mul(row, qy));
                qy = mul(qy, cj(hy));
            }
            // |mean| < LOW_AMP·‖Γ_w‖_F / M  ⇔  |Σ| < LOW_AMP·M·‖Γ_w‖_F
            if (fro2 == 0.0 || !(sqrt(abs2(sum)) >= kLowAmp * double(M) * sqrt(fro2))) fl |= 1u << 3;
            double a = atan2(sum.im, sum.re);
            wx = -atan2(zx.im, zx.re);
            wy = atan2(zy.im, zy.re);
            if (ref != nullptr) a = wrap_pi(a - (double)__ldg(ref + (size_t)py * W + px));
            result = a;
        }
        const size_t o = (size_t)f * plane + (size_t)py * W + px;
        out[o] = (float)result;
        if (flags != nullptr) flags[o] = fl;
        if (omx != nullptr) omx[o] = (float)wx;
        if (omy != nullptr) omy[o] = (float)wy;
    }
}

}  // namespace f64
}  // namespace bos
