// demod_strip.cuh — the paper-path thread-per-pixel kernel with a sliding covariance
// ("strip kernels": R_y slid in registers, or no R_y at all for the larger windows).
//
// Same per-pixel chain as demod_kernel.cuh (Algorithm 1: a2 R_y = Γ_wΓ_w^H,
// a3 power iteration + v_1 = Γ_w^H u_1, a4 coefficients, a5 symmetric Aberth + selection,
// a6 Eq.(15), a7 wrap(α − φ_ref)) and the same FP32 arithmetic, but a warp walks DOWN a
// vertical strip of S image rows × 32 columns instead of across one row, so consecutive
// pixels of a thread share M−1 of the M window rows:
//
//   R_y(py+1)(i, j) = R_y(py)(i+1, j+1)          for i, j ≤ M−2      (Eq.(4), rows ↔ y [R4])
//
// exactly — each entry is Σ_k Γ(row_a, k)·conj(Γ(row_b, k)) over the window's M columns, and
// clamped border rows [R1] shift the same way.  Per pixel only the new last row R(M−1, ·) is
// formed (M² complex MACs instead of M²(M+1)/2): the covariance drops from ≈17 % (M = 8) … 30 %
// (M = 16) of the per-pixel flops to ≈3 %.  Each entry is summed over k in the same order as
// the row kernel's full build, so R — and with it every output — is bitwise identical to
// demod_kernel<M, false, false> (tests/test_gpu_strip.py).  A non-finite sample poisons exactly
// the entries of its row and leaves with it: no rebuild is needed.
//
// Layout (one warp = 32 columns, lanes independent after staging):
//  * halo tile per warp: (M+1) rows × (32+M−1) complex in shared memory — rows 0…M−1 the
//    current window rows, row M the next row, prefetched with cp.async one step ahead; per
//    step every lane shifts its own two columns up by one row (no cross-lane hazard);
//  * R_y in registers while the pixel forms it and runs the power iteration (as in the row
//    kernel); between pixels the (M−1)(M−2)/2 + M−1 entries that survive the shift wait in the
//    thread's shared-memory slice (stride = threads per CTA: consecutive lanes → consecutive
//    words), stored already shifted.  (A first version kept all of R_y in shared memory and ran
//    the power iteration from there: 2·NOFF loads per iteration doubled the kernel's shared
//    traffic and it measured 7 % slower than the row kernel at M = 8.);
//  * work item = (frame, strip of S rows, 32-column block), one per 1-warp CTA: the hardware
//    block scheduler refills an SM slot as soon as a warp finishes, so fast and slow strips
//    balance (a persistent grid with equal row shares per warp reached 20.5 % of the 25 %
//    theoretical occupancy at M = 8 — warps that finished early left their slots idle).
#pragma once

#include "demod_kernel.cuh"

namespace bos {

// Which paper-path kernel runs window M on a large launch (measured per M, round 2, C3 1024²,
// 10 and 0 dB: profiles/r02_strip.md):  1 = strip kernel with R_y in registers (faster up to
// M = 10 and at 12, 13);  2 = implicit-power-iteration strip kernel (M = 11 and 14…32: equal
// at 11 and without the register kernel's 160-byte spill, +1…+130 % from 14);  0 = none (the
// row kernel).  BOS_STRIP_KIND_OVERRIDE=k forces kind k for every M (A/B builds).
template <int M>
constexpr int strip_kind() {
#ifdef BOS_STRIP_KIND_OVERRIDE
    return BOS_STRIP_KIND_OVERRIDE;
#else
    return (M <= 10 || M == 12 || M == 13) ? 1 : 2;
#endif
}
#ifndef BOS_POWER_ERR_STOP_MIN_M
#define BOS_POWER_ERR_STOP_MIN_M 20   // implicit strip kernel from this M: error-based power-iteration stop
#endif
#ifndef BOS_POWER_ERR_TOL
#define BOS_POWER_ERR_TOL 1e-10f // squared estimated eigenvector error at the error-based stop
#endif
constexpr int kPowerErrStopMinM = BOS_POWER_ERR_STOP_MIN_M;
#ifndef BOS_POWER_SHIFT
#define BOS_POWER_SHIFT 0        // implicit strip kernel: shifted power iteration (see there)
#endif
constexpr bool kPowerShift = BOS_POWER_SHIFT != 0;
constexpr float kPowerErrTol = BOS_POWER_ERR_TOL;
#ifndef BOS_STRIP_ROWS
#define BOS_STRIP_ROWS 16        // S: rows per work item (fewer for small launches, see launch_strip)
#endif
#ifndef BOS_STRIP_MIN_ROWS
#define BOS_STRIP_MIN_ROWS 8     // smaller launches run on the row kernel (launch_strip)
#endif
#ifndef BOS_STRIP_SMALL_MIN_M
#define BOS_STRIP_SMALL_MIN_M 17 // from this M the implicit kernel also runs launches too small for 8-row strips
#endif
#ifndef BOS_STRIP_WARPS
#define BOS_STRIP_WARPS 1
#endif
template <int M>
constexpr int strip_warps() { return BOS_STRIP_WARPS; }
// resident warps per SM the register budget is sized for (4 per SM partition → 128 registers,
// 3 → 168, 2 → 255)
template <int M>
constexpr int strip_warps_per_sm() { return M <= 8 ? 16 : (M <= 11 ? 12 : 8); }   // 8: 255 registers
template <int M>
constexpr int strip_min_blocks() { return strip_warps_per_sm<M>() / strip_warps<M>(); }
template <int M>
constexpr size_t strip_smem_bytes() {
    constexpr int NT = strip_warps<M>() * 32;
    return (size_t)strip_warps<M>() * (M + 1) * (32 + M - 1) * sizeof(float2) +
           (size_t)NT * ((M - 1) * (M - 2) / 2) * sizeof(cx2) + (size_t)NT * (M - 1) * sizeof(float);
}

// Row I of R_y over the window's M columns — entries (I, j), j < I, and the diagonal entry I —
// summed over k in the row kernel's order (so every entry is bitwise the row kernel's).
template <int M, int TW, int I>
__device__ __forceinline__ void strip_new_row(const float2* win, float (&Rd)[M], cx2 (&Ro)[M * (M - 1) / 2]) {
    constexpr int B = I * (I - 1) / 2;                 // tri_off(I, 0)
    float d = 0.0f;
#pragma unroll
    for (int j = 0; j < I; ++j) Ro[B + j] = 0ull;
#pragma unroll 1
    for (int k = 0; k < M; ++k) {
        const float2 gi = win[I * TW + k];
        d = fmaf(gi.x, gi.x, fmaf(gi.y, gi.y, d));
        const cx2 ci = cx2_make(gi.x, gi.y);
        const cx2 cnj = mul2(cx2_make(gi.y, gi.x), cx2_make(1.0f, -1.0f));   // −j·a
#pragma unroll
        for (int j = 0; j < I; ++j) {
            const float2 gj = win[j * TW + k];
            Ro[B + j] = fma2(cx2_bcast(gj.x), ci, fma2(cx2_bcast(gj.y), cnj, Ro[B + j]));
        }
    }
    Rd[I] = d;
}

// The carry between consecutive pixels of a thread, in its shared-memory slice (stride NT):
// slot (i, j) of the next pixel = entry (i+1, j+1) of this one, i.e. only the (M−1)(M−2)/2
// entries and M−1 diagonal values that survive the shift.
template <int M, int NT>
__device__ __forceinline__ void strip_store_carry(const float (&Rd)[M], const cx2 (&Ro)[M * (M - 1) / 2], cx2* Cs,
                                                  float* Cds) {
#pragma unroll
    for (int i = 0; i + 1 < M; ++i) Cds[i * NT] = Rd[i + 1];
#pragma unroll
    for (int i = 1; i + 1 < M; ++i) {
#pragma unroll
        for (int j = 0; j < i; ++j) Cs[tri_off<M>(i, j) * NT] = Ro[tri_off<M>(i + 1, j + 1)];
    }
}

template <int M, int NT>
__device__ __forceinline__ void strip_load_carry(float (&Rd)[M], cx2 (&Ro)[M * (M - 1) / 2], const cx2* Cs,
                                                 const float* Cds) {
#pragma unroll
    for (int i = 0; i + 1 < M; ++i) Rd[i] = Cds[i * NT];
#pragma unroll
    for (int i = 1; i + 1 < M; ++i) {
#pragma unroll
        for (int j = 0; j < i; ++j) Ro[tri_off<M>(i, j)] = Cs[tri_off<M>(i, j) * NT];
    }
}

// The row kernel's power iteration (demod_kernel.cuh, a3) on R_y in registers: start
// u_i = e^{jω̂ i}/√M from the lag-1 correlation, y = R u, stop at ‖Δu‖² < kPowerTol.
// lam2 = ‖R u‖² of the converged step (λ1²), +inf when the cap was hit.
template <int M>
__device__ __forceinline__ int strip_power_iteration(const float (&Rd)[M], const cx2 (&Ro)[M * (M - 1) / 2],
                                                     cx2 (&u)[M], bool& ok, float& lam2, float tol) {
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
    lam2 = CUDART_INF_F;
    ok = false;
    int n = 0;
    for (; n < kPowerMaxIt;) {
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
        ++n;
        if (diff < tol) { ok = true; lam2 = nrm2; break; }
    }
    return n;
}

template <int M, bool COUNT>
__global__ void __launch_bounds__(strip_warps<M>() * 32, strip_min_blocks<M>())
demod_strip_kernel(const float2* __restrict__ frames, int n_frames, int H, int W, int S,
                   const float* __restrict__ ref, float* __restrict__ out, uint8_t* __restrict__ flags,
                   float* __restrict__ omx, float* __restrict__ omy, unsigned long long* __restrict__ counters) {
    constexpr int WARPS = strip_warps<M>();
    constexpr int NT = WARPS * 32;
    constexpr int O0 = (M - 1) / 2;                 // o_i = i − O0  [R2]
    constexpr int TW = kBX + M - 1;
    constexpr int NOFF = M * (M - 1) / 2;
    extern __shared__ __align__(16) unsigned char strip_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float2* tile = reinterpret_cast<float2*>(strip_smem) + warp * (M + 1) * TW;
    constexpr int NCARRY = (M - 1) * (M - 2) / 2;
    cx2* Cs = reinterpret_cast<cx2*>(reinterpret_cast<float2*>(strip_smem) + WARPS * (M + 1) * TW) + threadIdx.x;
    float* Cds = reinterpret_cast<float*>(reinterpret_cast<cx2*>(reinterpret_cast<float2*>(strip_smem) +
                                                                  WARPS * (M + 1) * TW) + NCARRY * NT) + threadIdx.x;
    const size_t plane = (size_t)H * (size_t)W;
    const int nbx = (W + kBX - 1) / kBX;
    const int nstrip = (H + S - 1) / S;
    const long long items = (long long)n_frames * nstrip * nbx;     // (frame, strip of S rows, 32-column block)
    const long long wstride = (long long)gridDim.x * WARPS;

    for (long long item = (long long)blockIdx.x * WARPS + warp; item < items; item += wstride) {
        const int bx = (int)(item % nbx);
        const long long rest = item / nbx;
        const int f = (int)(rest / nstrip);
        const int py0 = (int)(rest % nstrip) * S;
        const int rows = min(S, H - py0);
        const int x0 = bx * kBX, px = x0 + lane;
        const float2* __restrict__ frame = frames + (size_t)f * plane;
        const int gx0 = min(max(x0 - O0 + lane, 0), W - 1);
        const int gx1 = min(max(x0 - O0 + lane + kBX, 0), W - 1);
        // strip row r (0 … rows+M−2) ↔ image row clamp(py0 − O0 + r)  (a1, [R1])
        auto load_row = [&](int r, float2* dst) {
            const float2* __restrict__ row = frame + (size_t)min(max(py0 - O0 + r, 0), H - 1) * W;
            cp_async8(dst + lane, row + gx0);
            if (lane + kBX < TW) cp_async8(dst + lane + kBX, row + gx1);
        };
        __syncwarp();                                  // the previous item's reads of the tile are done
#pragma unroll 1
        for (int r = 0; r < M; ++r) load_row(r, tile + r * TW);
        cp_async_commit();
        for (int s = 0; s < rows; ++s) {
            cp_async_wait_all();
            __syncwarp();
            if (s > 0) {                               // window moves down one row: rows 1…M → 0…M−1
#pragma unroll
                for (int r = 0; r < M; ++r) {
                    tile[r * TW + lane] = tile[(r + 1) * TW + lane];
                    if (lane + kBX < TW) tile[r * TW + lane + kBX] = tile[(r + 1) * TW + lane + kBX];
                }
                __syncwarp();
            }
            if (s + 1 < rows) load_row(s + M, tile + M * TW);     // next step's new row (row M)
            cp_async_commit();

            const int py = py0 + s;
            if (px < W) {
                const float2* win = tile + lane;       // Γ_w(i,k) = win[i*TW + k]
                uint8_t fl = 0;
                if (py - O0 < 0 || py + (M - 1 - O0) > H - 1 || px - O0 < 0 || px + (M - 1 - O0) > W - 1)
                    fl |= kFlagBorder;
                // ---- a2: R_y in registers: in full at the strip start, else the carry (the
                // previous pixel's entries shifted by one row) + the new last row ----
                float Rd[M];
                cx2 Ro[NOFF > 0 ? NOFF : 1];
                if (s == 0) {
#pragma unroll
                    for (int i = 0; i < M; ++i) Rd[i] = 0.0f;
#pragma unroll
                    for (int t = 0; t < NOFF; ++t) Ro[t] = 0ull;
                    const cx2 kPosNeg = cx2_make(1.0f, -1.0f);
#pragma unroll 1
                    for (int k = 0; k < M; ++k) {   // the row kernel's full build (same order)
                        cx2 col[M], colnj[M];
#pragma unroll
                        for (int i = 0; i < M; ++i) {
                            const float2 g = win[i * TW + k];
                            col[i] = cx2_make(g.x, g.y);
                            colnj[i] = mul2(cx2_make(g.y, g.x), kPosNeg);
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
                } else {
                    strip_load_carry<M, NT>(Rd, Ro, Cs, Cds);
                    strip_new_row<M, TW, M - 1>(win, Rd, Ro);
                }
                if (s + 1 < rows) strip_store_carry<M, NT>(Rd, Ro, Cs, Cds);
                float trace = 0.0f;
#pragma unroll
                for (int i = 0; i < M; ++i) trace += Rd[i];

                float result, wx = CUDART_NAN_F, wy = CUDART_NAN_F;
                int n_pow = 0, n_aby = 0, n_abx = 0;
                if (!isfinite(trace)) {
                    fl |= kFlagNonfinite;
                    result = CUDART_NAN_F;
                } else {
                    // ---- a3: u_1 by power iteration (the row kernel's), v_1 = Γ_w^H u_1 / ‖·‖ ----
                    cx2 u[M];
                    bool pow_ok = false;
                    float lam2;
                    n_pow = strip_power_iteration<M>(Rd, Ro, u, pow_ok, lam2, (fl & kFlagBorder) ? kPowerTolBorder : kPowerTol);
                    if constexpr (!newton_stop<false, M>()) {
                        if (lam2 < kWeakNewtonRatio * kWeakNewtonRatio * trace * trace) fl |= kFlagWeakInternal;
                    } else if constexpr (M >= kWeakTightMinM) {
                        if (lam2 < kLowSnrRatio * kLowSnrRatio * trace * trace) fl |= kFlagWeakInternal;
                    }
                    // ---- v_1 = Γ_w^H u_1/‖·‖, a4 + a5 + a6 ----
                    float2 zx, zy;
                    float a = roots_and_phase_jit<M, TW, false, (M >= kWeakTightMinM)>(win, u, trace, pow_ok, fl, n_aby,
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
        }
        cp_async_wait_all();
    }
}


// ---- Larger windows (strip_kind<M>() == 2): no R_y at all.  From M ≈ 11 R_y no longer fits
// the registers beside the rooting state (the row kernel spills 0.1–2.4 KB per thread at
// M = 11…20), and a per-thread shared-memory copy of it (M(M−1)/2 entries, slid in place — an
// intermediate version) limits a B200 SM to 6…2 warps at M = 15…24.  Here the power iteration
// applies R_y = Γ_wΓ_w^H as Γ_w(Γ_w^H u) straight from the window tile (2M² instead of M²
// complex MACs per iteration, no M³/2 build, no slide), the
// trace and the lag-1 sum Σ_i R[i+1][i] come from one pass over the window, and u_1, v_1 wait
// in the thread's shared-memory slice while the other axis is rooted.  The loops over the
// window run rolled over one index (loop-carried vectors go through the slice), which keeps
// the kernel's code — and its instruction-cache footprint — O(M) instead of O(M²).
// Same FP32 chain otherwise; parity against the FP64 oracle (tests/test_gpu_strip.py).

// M-vectors per lane the implicit kernel keeps in shared memory.  2: u_1 and v_1 in two
// slices.  1 (M ≥ BOS_STRIP_IM_ONE_SLOT_MIN_M): one slice holds the power iteration's scratch,
// then u_1; v_1 = Γ_w^H u_1/‖·‖ is formed in registers when the x axis starts (u_1 is dead by
// then) — 8 KB less per warp at M = 32, which lifts the SM from 6 to 8 resident warps at
// M = 31, 32 (measured +8 % at M = 32, 10 and 0 dB; at M = 30 — 7 → 8 warps — −3 %…0, so the
// two-slice layout stays below).
#ifndef BOS_STRIP_IM_ONE_SLOT_MIN_M
#define BOS_STRIP_IM_ONE_SLOT_MIN_M 31
#endif
template <int M>
constexpr int strip_im_slots() { return M >= BOS_STRIP_IM_ONE_SLOT_MIN_M ? 1 : 2; }
template <int M>
constexpr size_t strip_im_smem_bytes() {      // one warp: tile (M+1 rows) + strip_im_slots M-vectors per lane
    return (size_t)(M + 1) * (32 + M - 1) * sizeof(float2) + (size_t)32 * strip_im_slots<M>() * M * sizeof(cx2);
}

// t = Γ_w^H u column by column (t_k = Σ_i conj(Γ(i,k)) u_i, v1_from_window's arithmetic) into
// the slice T (entry k at T[k·32]); returns ‖t‖²
template <int M, int TW>
__device__ __forceinline__ float im_gamma_h(const float2* win, const cx2 (&u)[M], cx2* T) {
    const cx2 kPosNeg = cx2_make(1.0f, -1.0f);
    cx2 unj[M];
#pragma unroll
    for (int i = 0; i < M; ++i) unj[i] = mul2(cx2_make(cx2_im(u[i]), cx2_re(u[i])), kPosNeg);   // −j·u_i
    float n2 = 0.0f;
#pragma unroll 1
    for (int k = 0; k < M; ++k) {
        cx2 acc = 0ull;
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const float2 g = win[i * TW + k];
            acc = fma2(cx2_bcast(g.x), u[i], fma2(cx2_bcast(g.y), unj[i], acc));
        }
        T[k * 32] = acc;
        n2 += cabs2(cx2_f2(acc));
    }
    return n2;
}

// the same t = Γ_w^H u with u read from the slice U one entry per row and t kept in registers
// (row-outer order: one u_i live instead of u and −j·u; per-k sums in the same order and
// nesting as im_gamma_h, so bitwise equal); returns ‖t‖²
template <int M, int TW>
__device__ __forceinline__ float im_gamma_h_rows(const float2* win, const cx2* U, cx2 (&t)[M]) {
    const cx2 kPosNeg = cx2_make(1.0f, -1.0f);
#pragma unroll
    for (int k = 0; k < M; ++k) t[k] = 0ull;
#pragma unroll 1
    for (int i = 0; i < M; ++i) {
        const cx2 ui = U[i * 32];
        const cx2 uj = mul2(cx2_make(cx2_im(ui), cx2_re(ui)), kPosNeg);   // −j·u_i
#pragma unroll
        for (int k = 0; k < M; ++k) {
            const float2 g = win[i * TW + k];
            t[k] = fma2(cx2_bcast(g.x), ui, fma2(cx2_bcast(g.y), uj, t[k]));
        }
    }
    float n2 = 0.0f;
#pragma unroll
    for (int k = 0; k < M; ++k) n2 += cabs2(cx2_f2(t[k]));
    return n2;
}

// resident warps per SM the implicit kernel's register budget is sized for (12 → ≤ 168
// registers, 8 → ≤ 255); BOS_STRIP_IM_WARPS_MAX_M12 = the largest M given 12
#ifndef BOS_STRIP_IM_WARPS_MAX_M12
#define BOS_STRIP_IM_WARPS_MAX_M12 18   // measured: M = 15, 16 +6 %, 17 +3 %, 18 +2 %; M = 20 −4 % (shared memory caps it at 11 warps)
#endif
#ifndef BOS_STRIP_IM_WARPS_MAX_M16
#define BOS_STRIP_IM_WARPS_MAX_M16 11   // largest M given 16 warps/SM (128 registers): M = 11 +5 %; 14…16 spill there and lose 2…13 %
#endif
template <int M>
constexpr int strip_im_min_blocks() {
    return M <= BOS_STRIP_IM_WARPS_MAX_M16 ? 16 : (M <= BOS_STRIP_IM_WARPS_MAX_M12 ? 12 : 8);
}

template <int M, bool COUNT>
__global__ void __launch_bounds__(32, strip_im_min_blocks<M>())
demod_strip_im_kernel(const float2* __restrict__ frames, int n_frames, int H, int W, int S,
                      const float* __restrict__ ref, float* __restrict__ out, uint8_t* __restrict__ flags,
                      float* __restrict__ omx, float* __restrict__ omy, unsigned long long* __restrict__ counters) {
    constexpr int O0 = (M - 1) / 2;
    constexpr int TW = kBX + M - 1;
    extern __shared__ __align__(16) unsigned char strip_smem[];
    const int lane = threadIdx.x;
    float2* tile = reinterpret_cast<float2*>(strip_smem);
    cx2* Us = reinterpret_cast<cx2*>(tile + (M + 1) * TW) + lane;   // u_1: entry i at Us[i·32]
    cx2* Vs = strip_im_slots<M>() == 1 ? Us : Us + M * 32;           // v_1 (and the iteration's scratch)
    const size_t plane = (size_t)H * (size_t)W;
    const int nbx = (W + kBX - 1) / kBX;
    const int nstrip = (H + S - 1) / S;
    const long long items = (long long)n_frames * nstrip * nbx;

    for (long long item = blockIdx.x; item < items; item += gridDim.x) {
        const int bx = (int)(item % nbx);
        const long long rest = item / nbx;
        const int f = (int)(rest / nstrip);
        const int py0 = (int)(rest % nstrip) * S;
        const int rows = min(S, H - py0);
        const int x0 = bx * kBX, px = x0 + lane;
        const float2* __restrict__ frame = frames + (size_t)f * plane;
        const int gx0 = min(max(x0 - O0 + lane, 0), W - 1);
        const int gx1 = min(max(x0 - O0 + lane + kBX, 0), W - 1);
        auto load_row = [&](int r, float2* dst) {
            const float2* __restrict__ row = frame + (size_t)min(max(py0 - O0 + r, 0), H - 1) * W;
            cp_async8(dst + lane, row + gx0);
            if (lane + kBX < TW) cp_async8(dst + lane + kBX, row + gx1);
        };
        __syncwarp();
#pragma unroll 1
        for (int r = 0; r < M; ++r) load_row(r, tile + r * TW);
        cp_async_commit();
        for (int s = 0; s < rows; ++s) {
            cp_async_wait_all();
            __syncwarp();
            if (s > 0) {
#pragma unroll 1
                for (int r = 0; r < M; ++r) {
                    tile[r * TW + lane] = tile[(r + 1) * TW + lane];
                    if (lane + kBX < TW) tile[r * TW + lane + kBX] = tile[(r + 1) * TW + lane + kBX];
                }
                __syncwarp();
            }
            if (s + 1 < rows) load_row(s + M, tile + M * TW);
            cp_async_commit();

            const int py = py0 + s;
            if (px < W) {
                const float2* win = tile + lane;
                uint8_t fl = 0;
                if (py - O0 < 0 || py + (M - 1 - O0) > H - 1 || px - O0 < 0 || px + (M - 1 - O0) > W - 1)
                    fl |= kFlagBorder;
                // ---- tr R_y = ‖Γ_w‖_F² and r1 = Σ_i R[i+1][i] = Σ_k Σ_i Γ(i+1,k) conj(Γ(i,k)), one pass ----
                float trace = 0.0f;
                float2 r1 = make_float2(0.0f, 0.0f);
                {
                    float2 prev[M];
#pragma unroll
                    for (int k = 0; k < M; ++k) {
                        prev[k] = win[k];
                        trace = fmaf(prev[k].x, prev[k].x, fmaf(prev[k].y, prev[k].y, trace));
                    }
#pragma unroll 1
                    for (int i = 1; i < M; ++i) {
                        float2 racc = make_float2(0.0f, 0.0f);
#pragma unroll
                        for (int k = 0; k < M; ++k) {
                            const float2 g = win[i * TW + k];
                            trace = fmaf(g.x, g.x, fmaf(g.y, g.y, trace));
                            racc = cfmac(g, prev[k], racc);            // g · conj(prev)
                            prev[k] = g;
                        }
                        r1 = cadd(r1, racc);
                    }
                }
                float result, wx = CUDART_NAN_F, wy = CUDART_NAN_F;
                int n_pow = 0, n_aby = 0, n_abx = 0;
                if (!isfinite(trace)) {
                    fl |= kFlagNonfinite;
                    result = CUDART_NAN_F;
                } else {
                    // ---- a3: power iteration y = Γ_w(Γ_w^H u) from the lag-1 tone start ----
                    cx2 u[M];
                    {
                        float2 e = make_float2(1.0f, 0.0f);
                        if (cabs2(r1) > 0.0f) e = cscale(r1, rsqrtf(cabs2(r1)));
                        float2 t = make_float2(rsqrtf(float(M)), 0.0f);
#pragma unroll
                        for (int i = 0; i < M; ++i) {
                            u[i] = cx2_make(t.x, t.y);
                            t = cmul(t, e);
                        }
                    }
                    bool pow_ok = false;
                    float lam2 = CUDART_INF_F;
                    float prev_diff = CUDART_INF_F;
                    const float ptol = (fl & kFlagBorder) ? kPowerTolBorder : kPowerTol;
                    for (n_pow = 0; n_pow < kPowerMaxIt;) {
                        im_gamma_h<M, TW>(win, u, Vs);                 // t = Γ^H u → slice
                        cx2 t[M], tj[M];
#pragma unroll
                        for (int k = 0; k < M; ++k) {
                            t[k] = Vs[k * 32];
                            tj[k] = mul2(cx2_make(cx2_im(t[k]), cx2_re(t[k])), cx2_make(-1.0f, 1.0f));   // j·t
                        }
                        // y_i = Σ_k Γ(i,k) t_k, row by row → slice
#pragma unroll 1
                        for (int i = 0; i < M; ++i) {
                            cx2 acc = 0ull;
#pragma unroll
                            for (int k = 0; k < M; ++k) {
                                const float2 g = win[i * TW + k];
                                acc = fma2(cx2_bcast(g.x), t[k], fma2(cx2_bcast(g.y), tj[k], acc));
                            }
                            Vs[i * 32] = acc;
                        }
                        cx2 y[M];
                        float nrm2 = 0.0f, rq = 0.0f;            // ‖R u‖², Rayleigh quotient u^H R u
#pragma unroll
                        for (int i = 0; i < M; ++i) {
                            y[i] = Vs[i * 32];
                            nrm2 += cabs2(cx2_f2(y[i]));
                            rq = fmaf(cx2_re(u[i]), cx2_re(y[i]), fmaf(cx2_im(u[i]), cx2_im(y[i]), rq));
                        }
                        // shifted step (R − μI)u with μ = the mean of the other eigenvalues,
                        // (tr − λ1)/(M−1), once λ1 > 3μ: the step ratio (λ2 − μ)/(λ1 − μ) instead of
                        // λ2/λ1 — fewer iterations for weak-tone windows; same eigenvector
                        float nrm2s = nrm2;
                        if constexpr (kPowerShift) {
                            const float mu = (trace - rq) * (1.0f / float(M - 1));
                            if (rq > 3.0f * mu && mu > 0.0f) {
                                nrm2s = 0.0f;
#pragma unroll
                                for (int i = 0; i < M; ++i) {
                                    y[i] = fma2(cx2_bcast(-mu), u[i], y[i]);
                                    nrm2s += cabs2(cx2_f2(y[i]));
                                }
                            }
                        }
                        const cx2 inv = cx2_bcast(rsqrtf(nrm2s));
                        float diff = 0.0f;
#pragma unroll
                        for (int i = 0; i < M; ++i) {
                            const cx2 yn = mul2(y[i], inv);
                            diff += cabs2(cx2_f2(sub2(yn, u[i])));
                            u[i] = yn;
                        }
                        ++n_pow;
                        if (diff < ptol) { pow_ok = true; lam2 = nrm2; break; }
                        // error-based stop: in the asymptotic regime the step shrinks by ρ = λ2/λ1
                        // per iteration (ρ² ≈ diff/prev_diff) and the remaining error is
                        // ≈ ‖Δu‖·ρ/(1−ρ); stop once that is below kPowerErrTol^½ with ρ ≤ ½.
                        // High-SNR windows then stop after 2 iterations instead of the 3rd that
                        // only confirmed a < 1e-4 step (emulated: error ≤ 3e-5; measured 2.0 vs
                        // 3.0 iterations, +4…6 % at M = 20…32, none below: a warp still runs its
                        // slowest lane's 3rd iteration, so the rule starts at M = 20).
                        if constexpr (M >= kPowerErrStopMinM) {
                            const float r2 = diff / prev_diff;   // 0 after the first iteration (prev = ∞)
                            if (n_pow >= 2 && r2 < 0.25f && !(fl & kFlagBorder)) {
                                const float rr = sqrtf(r2);
                                if (diff * r2 < kPowerErrTol * (1.0f - rr) * (1.0f - rr)) { pow_ok = true; lam2 = nrm2; break; }
                            }
                        }
                        prev_diff = diff;
                    }
                    if constexpr (M >= kWeakTightMinM)
                        if (lam2 < kLowSnrRatio * kLowSnrRatio * trace * trace) fl |= kFlagWeakInternal;
                    // u_1 and v_1 = Γ_w^H u_1/‖·‖ to the slice(s) (v1_from_window's arithmetic);
                    // one slice: u_1 now, v_1 formed in registers when the x axis starts
                    if constexpr (strip_im_slots<M>() == 1) {
#pragma unroll
                        for (int k = 0; k < M; ++k) Us[k * 32] = u[k];
                        compiler_fence();       // no store-to-load forwarding: u must not stay live into the axis loop
                    } else {
                        const float vn = im_gamma_h<M, TW>(win, u, Vs);
                        const cx2 vinv = cx2_bcast(rsqrtf(vn));
#pragma unroll
                        for (int k = 0; k < M; ++k) {
                            Vs[k * 32] = mul2(Vs[k * 32], vinv);
                            Us[k * 32] = u[k];
                        }
                    }
                    float2 zx, zy;
                    float a = roots_and_phase_q<M, TW, false, (M >= kWeakTightMinM)>(
                        win,
                        [&](int axis, float2 (&q)[M]) {
                            if constexpr (strip_im_slots<M>() == 1) {
                                if (axis) {
                                    cx2 t[M];
                                    const float vn = im_gamma_h_rows<M, TW>(win, Us, t);
                                    const cx2 vinv = cx2_bcast(rsqrtf(vn));
#pragma unroll
                                    for (int i = 0; i < M; ++i) q[i] = cx2_f2(mul2(t[i], vinv));
                                } else {
#pragma unroll
                                    for (int i = 0; i < M; ++i) q[i] = cx2_f2(Us[i * 32]);
                                }
                            } else {
                                const cx2* Q = axis ? Vs : Us;
#pragma unroll
                                for (int i = 0; i < M; ++i) q[i] = cx2_f2(Q[i * 32]);
                            }
                        },
                        trace, pow_ok, fl, n_aby, n_abx, zx, zy);
                    if (omx != nullptr) wx = -atan2f(zx.y, zx.x);
                    if (omy != nullptr) wy = atan2f(zy.y, zy.x);
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
        }
        cp_async_wait_all();
    }
}


// ---- Row f4, forward–backward averaging (BOS_VARIANT_FB, [R13]; not in the paper) on the
// implicit strip kernel: the FB-averaged R_y and S = Γ_w^TΓ_w* = conj(R_x) are never formed;
// their matvecs run from the tile:
//   FB(R_y) u = ½[Γ(Γ^H u) + J Γ*(Γ^T (J u))],   FB(S) w = ½[Γ^T(Γ* w) + J Γ^H(Γ (J w))]
// (J the exchange matrix), four window passes per matvec.  As the row / warp kernels' FB path:
// two power-iteration starts per axis (tone, ramp-weighted tone; the larger ‖Au‖ wins, the
// second skipped once λ > ½ tr), u_1 = the FB(R_y) eigenvector, v_1 = conj(the FB(S) one),
// then the paper's rooting and Eq.(15); weak-tone windows (λ1 < kLowSnrRatio·tr) start the
// rooting from the tight tolerance (the warp kernel's FB rule).  Parity vs the FP64 oracle's
// FB variant (tests/test_gpu_strip.py, tools/stress_parity.py --variant fb).
// measured on C3 1024² ×8 at 10 dB (Mpixel/s, FB implicit strip vs the row / warp kernels):
// M = 11 818 vs 1220, 16 320 vs 343, 20 223 vs 74, 24 119 vs 55, 26 92 vs 48, 28 51 vs 43, 32 19 vs 32
// (it spills from M = 22)
#ifndef BOS_STRIP_FB_MIN_M
#define BOS_STRIP_FB_MIN_M 17
#endif
#ifndef BOS_STRIP_FB_MAX_M
#define BOS_STRIP_FB_MAX_M 28
#endif
constexpr int kStripFbMinM = BOS_STRIP_FB_MIN_M;
constexpr int kStripFbMaxM = BOS_STRIP_FB_MAX_M;

template <int M>
constexpr size_t strip_imfb_smem_bytes() {    // one warp: tile + 3 M-vectors per lane (u, v, scratch)
    return (size_t)(M + 1) * (32 + M - 1) * sizeof(float2) + (size_t)32 * 3 * M * sizeof(cx2);
}

// T[k] = Σ_i g(i,k)·a_i, or Σ_i conj(g(i,k))·a_i (CONJ) — column sums, a indexed by row
template <int M, int TW, bool CONJ>
__device__ __forceinline__ void im_colsum(const float2* win, const cx2 (&a)[M], cx2* T) {
    cx2 aj[M];
#pragma unroll
    for (int i = 0; i < M; ++i)       // CONJ: −j·a (conj(g)a = gx·a + gy·(−ja));  else j·a
        aj[i] = CONJ ? mul2(cx2_make(cx2_im(a[i]), cx2_re(a[i])), cx2_make(1.0f, -1.0f))
                     : mul2(cx2_make(cx2_im(a[i]), cx2_re(a[i])), cx2_make(-1.0f, 1.0f));
#pragma unroll 1
    for (int k = 0; k < M; ++k) {
        cx2 acc = 0ull;
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const float2 g = win[i * TW + k];
            acc = fma2(cx2_bcast(g.x), a[i], fma2(cx2_bcast(g.y), aj[i], acc));
        }
        T[k * 32] = acc;
    }
}
// Y[i] = Σ_k g(i,k)·t_k, or Σ_k conj(g(i,k))·t_k (CONJ) — row sums, t indexed by column
template <int M, int TW, bool CONJ>
__device__ __forceinline__ void im_rowsum(const float2* win, const cx2 (&t)[M], cx2* Y) {
    cx2 tj[M];
#pragma unroll
    for (int k = 0; k < M; ++k)
        tj[k] = CONJ ? mul2(cx2_make(cx2_im(t[k]), cx2_re(t[k])), cx2_make(1.0f, -1.0f))
                     : mul2(cx2_make(cx2_im(t[k]), cx2_re(t[k])), cx2_make(-1.0f, 1.0f));
#pragma unroll 1
    for (int i = 0; i < M; ++i) {
        cx2 acc = 0ull;
#pragma unroll
        for (int k = 0; k < M; ++k) {
            const float2 g = win[i * TW + k];
            acc = fma2(cx2_bcast(g.x), t[k], fma2(cx2_bcast(g.y), tj[k], acc));
        }
        Y[i * 32] = acc;
    }
}
template <int M>
__device__ __forceinline__ void slice_load(const cx2* S, cx2 (&v)[M]) {
#pragma unroll
    for (int i = 0; i < M; ++i) v[i] = S[i * 32];
}

// y = FB(R_y) u (AXIS 0) or FB(S) u (AXIS 1), through the scratch slice T
template <int M, int TW, int AXIS>
__device__ __forceinline__ void fb_apply(const float2* win, const cx2 (&u)[M], cx2* T, cx2 (&y)[M]) {
    cx2 a[M];
    if constexpr (AXIS == 0) {
        im_colsum<M, TW, true>(win, u, T);     // Γ^H u
        slice_load<M>(T, a);
        im_rowsum<M, TW, false>(win, a, T);    // Γ(Γ^H u)
        slice_load<M>(T, y);
#pragma unroll
        for (int i = 0; i < M; ++i) a[i] = u[M - 1 - i];
        im_colsum<M, TW, false>(win, a, T);    // Γ^T (J u)
        slice_load<M>(T, a);
        im_rowsum<M, TW, true>(win, a, T);     // Γ*(Γ^T J u)
    } else {
        im_rowsum<M, TW, true>(win, u, T);     // Γ* w
        slice_load<M>(T, a);
        im_colsum<M, TW, false>(win, a, T);    // Γ^T(Γ* w)
        slice_load<M>(T, y);
#pragma unroll
        for (int k = 0; k < M; ++k) a[k] = u[M - 1 - k];
        im_rowsum<M, TW, false>(win, a, T);    // Γ (J w)
        slice_load<M>(T, a);
        im_colsum<M, TW, true>(win, a, T);     // Γ^H(Γ J w)
    }
    slice_load<M>(T, a);
#pragma unroll
    for (int i = 0; i < M; ++i) y[i] = mul2(add2(y[i], a[M - 1 - i]), cx2_bcast(0.5f));
}

// power iteration on the FB operator of AXIS from the tone e^{jω̂ i} (RAMP: weighted by
// i − (M−1)/2), stop at ‖Δu‖² < kPowerTol; lam = ‖A u‖ of the last step
template <int M, int TW, int AXIS, bool RAMP>
__device__ __forceinline__ int fb_power(const float2* win, float2 e, cx2* T, cx2 (&u)[M], bool& ok, float& lam) {
    {
        const float s0 = RAMP ? rsqrtf(float(M) * float(M * M - 1) / 12.0f) : rsqrtf(float(M));
        float2 t = make_float2(1.0f, 0.0f);
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const float wgt = RAMP ? s0 * (float(i) - 0.5f * float(M - 1)) : s0;
            u[i] = cx2_make(wgt * t.x, wgt * t.y);
            t = cmul(t, e);
        }
    }
    ok = false;
    lam = 0.0f;
    int n = 0;
#pragma unroll 1
    for (; n < kPowerMaxIt;) {
        cx2 y[M];
        fb_apply<M, TW, AXIS>(win, u, T, y);
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
        if (diff < kPowerTol) { ok = true; break; }
    }
    return n;
}

// dominant eigenvector of the FB operator of AXIS, two starts (see above) → slice OUT
template <int M, int TW, int AXIS>
__device__ __forceinline__ int fb_eigvec(const float2* win, float2 e, float trace, cx2* T, cx2* OUT, bool& ok,
                                         float& lam) {
    cx2 u[M];
    int n = fb_power<M, TW, AXIS, false>(win, e, T, u, ok, lam);
#pragma unroll
    for (int i = 0; i < M; ++i) OUT[i * 32] = u[i];
    if (ok && lam > 0.5005f * trace) return n;       // > half the trace of a PSD operator: the top one
    bool ok2 = false;
    float lam2 = 0.0f;
    n += fb_power<M, TW, AXIS, true>(win, e, T, u, ok2, lam2);
    if (lam2 > lam) {
#pragma unroll
        for (int i = 0; i < M; ++i) OUT[i * 32] = u[i];
        ok = ok2;
        lam = lam2;
    }
    return n;
}

template <int M, bool COUNT>
__global__ void __launch_bounds__(32, 8)
demod_strip_imfb_kernel(const float2* __restrict__ frames, int n_frames, int H, int W, int S,
                        const float* __restrict__ ref, float* __restrict__ out, uint8_t* __restrict__ flags,
                        float* __restrict__ omx, float* __restrict__ omy, unsigned long long* __restrict__ counters) {
    constexpr int O0 = (M - 1) / 2;
    constexpr int TW = kBX + M - 1;
    extern __shared__ __align__(16) unsigned char strip_smem[];
    const int lane = threadIdx.x;
    float2* tile = reinterpret_cast<float2*>(strip_smem);
    cx2* Us = reinterpret_cast<cx2*>(tile + (M + 1) * TW) + lane;
    cx2* Vs = Us + M * 32;
    cx2* Ts = Vs + M * 32;
    const size_t plane = (size_t)H * (size_t)W;
    const int nbx = (W + kBX - 1) / kBX;
    const int nstrip = (H + S - 1) / S;
    const long long items = (long long)n_frames * nstrip * nbx;

    for (long long item = blockIdx.x; item < items; item += gridDim.x) {
        const int bx = (int)(item % nbx);
        const long long rest = item / nbx;
        const int f = (int)(rest / nstrip);
        const int py0 = (int)(rest % nstrip) * S;
        const int rows = min(S, H - py0);
        const int x0 = bx * kBX, px = x0 + lane;
        const float2* __restrict__ frame = frames + (size_t)f * plane;
        const int gx0 = min(max(x0 - O0 + lane, 0), W - 1);
        const int gx1 = min(max(x0 - O0 + lane + kBX, 0), W - 1);
        auto load_row = [&](int r, float2* dst) {
            const float2* __restrict__ row = frame + (size_t)min(max(py0 - O0 + r, 0), H - 1) * W;
            cp_async8(dst + lane, row + gx0);
            if (lane + kBX < TW) cp_async8(dst + lane + kBX, row + gx1);
        };
        __syncwarp();
#pragma unroll 1
        for (int r = 0; r < M; ++r) load_row(r, tile + r * TW);
        cp_async_commit();
        for (int s = 0; s < rows; ++s) {
            cp_async_wait_all();
            __syncwarp();
            if (s > 0) {
#pragma unroll 1
                for (int r = 0; r < M; ++r) {
                    tile[r * TW + lane] = tile[(r + 1) * TW + lane];
                    if (lane + kBX < TW) tile[r * TW + lane + kBX] = tile[(r + 1) * TW + lane + kBX];
                }
                __syncwarp();
            }
            if (s + 1 < rows) load_row(s + M, tile + M * TW);
            cp_async_commit();

            const int py = py0 + s;
            if (px < W) {
                const float2* win = tile + lane;
                uint8_t fl = 0;
                if (py - O0 < 0 || py + (M - 1 - O0) > H - 1 || px - O0 < 0 || px + (M - 1 - O0) > W - 1)
                    fl |= kFlagBorder;
                // tr = ‖Γ_w‖_F²; lag-1 sums of R_y (Σ_i R[i+1][i]) and of S (Σ_k S[k+1][k]) — FB
                // averaging leaves both unchanged, so they seed the tone starts of both axes
                float trace = 0.0f;
                float2 r1y = make_float2(0.0f, 0.0f), r1x = make_float2(0.0f, 0.0f);
                {
                    float2 prev[M];
#pragma unroll
                    for (int k = 0; k < M; ++k) {
                        prev[k] = win[k];
                        trace = fmaf(prev[k].x, prev[k].x, fmaf(prev[k].y, prev[k].y, trace));
                        if (k > 0) r1x = cfmac(prev[k], prev[k - 1], r1x);
                    }
#pragma unroll 1
                    for (int i = 1; i < M; ++i) {
                        float2 ry = make_float2(0.0f, 0.0f), rx = make_float2(0.0f, 0.0f);
                        float2 gl = make_float2(0.0f, 0.0f);
#pragma unroll
                        for (int k = 0; k < M; ++k) {
                            const float2 g = win[i * TW + k];
                            trace = fmaf(g.x, g.x, fmaf(g.y, g.y, trace));
                            ry = cfmac(g, prev[k], ry);                // g·conj(row above)
                            if (k > 0) rx = cfmac(g, gl, rx);          // g·conj(left neighbour)
                            gl = g;
                            prev[k] = g;
                        }
                        r1y = cadd(r1y, ry);
                        r1x = cadd(r1x, rx);
                    }
                }
                float result, wx = CUDART_NAN_F, wy = CUDART_NAN_F;
                int n_pow = 0, n_aby = 0, n_abx = 0;
                if (!isfinite(trace)) {
                    fl |= kFlagNonfinite;
                    result = CUDART_NAN_F;
                } else {
                    const float2 ey = cabs2(r1y) > 0.0f ? cscale(r1y, rsqrtf(cabs2(r1y))) : make_float2(1.0f, 0.0f);
                    const float2 ex = cabs2(r1x) > 0.0f ? cscale(r1x, rsqrtf(cabs2(r1x))) : make_float2(1.0f, 0.0f);
                    bool oky = false, okx = false;
                    float lamy = 0.0f, lamx = 0.0f;
                    n_pow = fb_eigvec<M, TW, 0>(win, ey, trace, Ts, Us, oky, lamy);
                    n_pow += fb_eigvec<M, TW, 1>(win, ex, trace, Ts, Vs, okx, lamx);
#pragma unroll 1
                    for (int k = 0; k < M; ++k) Vs[k * 32] = mul2(Vs[k * 32], cx2_make(1.0f, -1.0f));   // v_1 = conj
                    if constexpr (M >= kWeakTightMinM)
                        if (lamy < kLowSnrRatio * trace) fl |= kFlagWeakInternal;
                    float2 zx, zy;
                    auto qfn = [&](int axis, float2 (&q)[M]) {
                        const cx2* Q = axis ? Vs : Us;
#pragma unroll
                        for (int i = 0; i < M; ++i) q[i] = cx2_f2(Q[i * 32]);
                    };
                    float a = roots_and_phase_q<M, TW, true, (M >= kWeakTightMinM), decltype(qfn)&>(
                        win, qfn, trace, oky && okx, fl, n_aby, n_abx, zx, zy);
                    if (omx != nullptr) wx = -atan2f(zx.y, zx.x);
                    if (omy != nullptr) wy = atan2f(zy.y, zy.x);
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
        }
        cp_async_wait_all();
    }
}

}  // namespace bos
