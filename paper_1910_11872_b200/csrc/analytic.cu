// analytic.cu — SURVEY §8 row f1: the analytic (complex) fringe signal from 8-bit intensity
// frames, the step before the root-MUSIC path: "by using bandpass filtering and carrier
// removal, the analytic or complex fringe signal is obtained" (Eq.(1)).
//
// Per frame:  I/255 → 2-D FFT (cuFFT, C2C, in place) → keep the +1 spectral lobe, a disc of
// radius r (cycles/px) around the carrier (f_x, f_y), scaled by 1/(H·W) → inverse FFT →
// optionally × e^{−j2π(f_x x + f_y y)} (carrier removal; a spatial-domain shift is exact for any
// carrier, integer bin or not).  The hard circular mask follows SPEC S:L126 ([R11] in
// the paper does not specify the filter).  Bin frequencies follow the DFT
// convention f_k = k/N for k ≤ ⌊(N−1)/2⌋, (k−N)/N otherwise; the disc test is done in FP64
// with explicit round-to-nearest operations so the oracle's numpy mask is matched bit for bit.
#include <cuda_runtime.h>
#include <cufft.h>

#include <algorithm>
#include <cstdint>
#include <new>

#include "bos_rootmusic.h"

namespace {

constexpr int kChunk = 8;   // frames per cuFFT batch (bounds the work area)

__global__ void u8_to_complex(const uint8_t* __restrict__ in, size_t n, float2* __restrict__ out) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = make_float2((float)in[i] * (1.0f / 255.0f), 0.0f);
}

__device__ __forceinline__ double bin_freq(int k, int n) {
    const int kk = (k <= (n - 1) / 2) ? k : k - n;
    return __dmul_rn((double)kk, 1.0 / (double)n);
}

// zero every bin outside the disc |f − f_c| ≤ r, scale the kept ones by 1/(H·W)
__global__ void lobe_mask(float2* __restrict__ spec, int T, int H, int W, double fx, double fy, double r2) {
    const size_t plane = (size_t)H * (size_t)W;
    const size_t n = plane * (size_t)T;
    const float scale = 1.0f / (float)plane;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const size_t q = i % plane;
        const int ky = (int)(q / (size_t)W), kx = (int)(q % (size_t)W);
        const double dx = __dadd_rn(bin_freq(kx, W), -fx);
        const double dy = __dadd_rn(bin_freq(ky, H), -fy);
        const double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
        float2 v = spec[i];
        if (d2 <= r2) {
            v.x *= scale;
            v.y *= scale;
        } else {
            v = make_float2(0.0f, 0.0f);
        }
        spec[i] = v;
    }
}

// Γ ← Γ · e^{−j2π(f_x x + f_y y)}; the phase cycle count is reduced mod 1 in FP64 first
__global__ void remove_carrier(float2* __restrict__ g, int T, int H, int W, double fx, double fy) {
    const size_t plane = (size_t)H * (size_t)W;
    const size_t n = plane * (size_t)T;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const size_t q = i % plane;
        const int y = (int)(q / (size_t)W), x = (int)(q % (size_t)W);
        double c = fx * (double)x + fy * (double)y;
        c -= floor(c);
        float s, co;
        sincospif(-2.0f * (float)c, &s, &co);
        const float2 v = g[i];
        g[i] = make_float2(v.x * co - v.y * s, v.x * s + v.y * co);
    }
}

bool is_dev(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int make_plan(cufftHandle* plan, int H, int W, int batch, size_t* work) {
    if (cufftCreate(plan) != CUFFT_SUCCESS) return BOS_ERR_CUDA;
    if (cufftSetAutoAllocation(*plan, 0) != CUFFT_SUCCESS) {
        cufftDestroy(*plan);
        return BOS_ERR_CUDA;
    }
    long long n[2] = {H, W};
    const long long dist = (long long)H * W;
    if (cufftMakePlanMany64(*plan, 2, n, nullptr, 1, dist, nullptr, 1, dist, CUFFT_C2C, batch, work) !=
        CUFFT_SUCCESS) {
        cufftDestroy(*plan);
        return BOS_ERR_CUDA;
    }
    return BOS_OK;
}

unsigned grid_for(size_t n) { return (unsigned)std::min<size_t>((n + 255) / 256, 148 * 32); }

}  // namespace

// Caller-owned plan object (opaque in the ABI): the cuFFT plans for a chunk of kChunk frames
// and for single frames (ragged tails), made once instead of per call.
struct bos_analytic_plan {
    int H, W, batch;
    cufftHandle full, one;
    size_t work;
};

namespace {

int run_planned(bos_analytic_plan* pl, const uint8_t* frames_u8, int n_frames, double fx, double fy, double radius,
                int remove, bos_cf32* out, void* d_workspace, size_t workspace_bytes, cudaStream_t s) {
    const int H = pl->H, W = pl->W;
    if (frames_u8 == nullptr || out == nullptr || d_workspace == nullptr) return BOS_ERR_INVALID_ARG;
    if (n_frames < 1 || !(radius > 0.0)) return BOS_ERR_INVALID_ARG;
    if (!(fx >= -0.5 && fx <= 0.5 && fy >= -0.5 && fy <= 0.5)) return BOS_ERR_INVALID_ARG;
    if (fx * fx + fy * fy <= radius * radius) return BOS_ERR_INVALID_ARG;   // the disc must exclude DC
    if (workspace_bytes < pl->work) return BOS_ERR_INVALID_ARG;
    if (!is_dev(frames_u8) || !is_dev(out) || !is_dev(d_workspace)) return BOS_ERR_INVALID_ARG;
    const size_t plane = (size_t)H * (size_t)W;
    const uintptr_t a = (uintptr_t)frames_u8, b = (uintptr_t)out;
    if (a < b + plane * (size_t)n_frames * sizeof(bos_cf32) && b < a + plane * (size_t)n_frames)
        return BOS_ERR_INVALID_ARG;
    for (cufftHandle h : {pl->full, pl->one})
        if (cufftSetWorkArea(h, d_workspace) != CUFFT_SUCCESS || cufftSetStream(h, s) != CUFFT_SUCCESS)
            return BOS_ERR_CUDA;
    for (int f0 = 0; f0 < n_frames;) {
        const int nb = (n_frames - f0 >= pl->batch) ? pl->batch : 1;     // ragged tail: frame by frame
        const cufftHandle p = (nb == pl->batch) ? pl->full : pl->one;
        float2* g = reinterpret_cast<float2*>(out) + (size_t)f0 * plane;
        const size_t n = plane * (size_t)nb;
        u8_to_complex<<<grid_for(n), 256, 0, s>>>(frames_u8 + (size_t)f0 * plane, n, g);
        if (cufftExecC2C(p, (cufftComplex*)g, (cufftComplex*)g, CUFFT_FORWARD) != CUFFT_SUCCESS) return BOS_ERR_CUDA;
        lobe_mask<<<grid_for(n), 256, 0, s>>>(g, nb, H, W, fx, fy, radius * radius);
        if (cufftExecC2C(p, (cufftComplex*)g, (cufftComplex*)g, CUFFT_INVERSE) != CUFFT_SUCCESS) return BOS_ERR_CUDA;
        if (remove) remove_carrier<<<grid_for(n), 256, 0, s>>>(g, nb, H, W, fx, fy);
        if (cudaGetLastError() != cudaSuccess) return BOS_ERR_CUDA;
        f0 += nb;
    }
    return BOS_OK;
}

}  // namespace

extern "C" {

int bos_analytic_plan_create(int H, int W, int max_frames, bos_analytic_plan** plan, size_t* workspace_bytes) {
    if (plan == nullptr || H < 2 || W < 2 || max_frames < 1) return BOS_ERR_INVALID_ARG;
    *plan = nullptr;
    bos_analytic_plan* pl = new (std::nothrow) bos_analytic_plan;
    if (pl == nullptr) return BOS_ERR_CUDA;
    pl->H = H;
    pl->W = W;
    pl->batch = std::min(max_frames, kChunk);
    size_t w1 = 0, w2 = 0;
    if (make_plan(&pl->full, H, W, pl->batch, &w1) != BOS_OK) {
        delete pl;
        return BOS_ERR_CUDA;
    }
    if (make_plan(&pl->one, H, W, 1, &w2) != BOS_OK) {
        cufftDestroy(pl->full);
        delete pl;
        return BOS_ERR_CUDA;
    }
    pl->work = std::max<size_t>(std::max(w1, w2), 256);
    if (workspace_bytes != nullptr) *workspace_bytes = pl->work;
    *plan = pl;
    return BOS_OK;
}

int bos_analytic_plan_destroy(bos_analytic_plan* plan) {
    if (plan == nullptr) return BOS_OK;
    cufftDestroy(plan->full);
    cufftDestroy(plan->one);
    delete plan;
    return BOS_OK;
}

int bos_analytic_signal_planned(bos_analytic_plan* plan, const uint8_t* frames_u8, int n_frames, double fx,
                                double fy, double radius, int remove_carrier, bos_cf32* out, void* d_workspace,
                                size_t workspace_bytes, void* stream) {
    if (plan == nullptr) return BOS_ERR_INVALID_ARG;
    return run_planned(plan, frames_u8, n_frames, fx, fy, radius, remove_carrier, out, d_workspace, workspace_bytes,
                       static_cast<cudaStream_t>(stream));
}

size_t bos_analytic_signal_workspace_bytes(int H, int W, int n_frames) {
    if (H < 2 || W < 2 || n_frames < 1) return 0;
    bos_analytic_plan* pl = nullptr;
    size_t work = 0;
    if (bos_analytic_plan_create(H, W, n_frames, &pl, &work) != BOS_OK) return 0;
    bos_analytic_plan_destroy(pl);
    return work;
}

int bos_analytic_signal(const uint8_t* frames_u8, int n_frames, int H, int W, double fx, double fy,
                        double radius, int remove, bos_cf32* out, void* d_workspace, size_t workspace_bytes,
                        void* stream) {
    if (frames_u8 == nullptr || out == nullptr || d_workspace == nullptr) return BOS_ERR_INVALID_ARG;
    if (n_frames < 1 || H < 2 || W < 2 || !(radius > 0.0)) return BOS_ERR_INVALID_ARG;
    if (!(fx >= -0.5 && fx <= 0.5 && fy >= -0.5 && fy <= 0.5)) return BOS_ERR_INVALID_ARG;
    if (fx * fx + fy * fy <= radius * radius) return BOS_ERR_INVALID_ARG;   // the disc must exclude DC
    if (!is_dev(frames_u8) || !is_dev(out) || !is_dev(d_workspace)) return BOS_ERR_INVALID_ARG;
    bos_analytic_plan* pl = nullptr;
    if (bos_analytic_plan_create(H, W, n_frames, &pl, nullptr) != BOS_OK) return BOS_ERR_CUDA;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int rc = run_planned(pl, frames_u8, n_frames, fx, fy, radius, remove, out, d_workspace, workspace_bytes, s);
    // cuFFT plans own device resources (twiddles): finish the queued work before destroying them
    if (cudaStreamSynchronize(s) != cudaSuccess && rc == BOS_OK) rc = BOS_ERR_CUDA;
    bos_analytic_plan_destroy(pl);
    return rc;
}

}  // extern "C"
