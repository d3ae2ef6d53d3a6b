// bos_rootmusic.cu — host side of libbosrm.so: argument validation, M-specialised kernel
// dispatch, the time-lapse stack driver and the pipelined host-buffer driver.
// The C ABI is declared (and documented) in include/bos_rootmusic.h.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <cstdint>
#include <mutex>

#include "bos_rootmusic.h"
#include "launch.h"
#include "template_roots.h"

namespace {

using LaunchFn = cudaError_t (*)(const float2*, int, int, int, const float*, float*, uint8_t*, float*, float*,
                                 unsigned long long*, cudaStream_t);

template <bool COUNT, bool FB>
LaunchFn pick(int M) {
    switch (M) {
        case 3: return bos::launch_demod<3, COUNT, FB>;
        case 4: return bos::launch_demod<4, COUNT, FB>;
        case 5: return bos::launch_demod<5, COUNT, FB>;
        case 6: return bos::launch_demod<6, COUNT, FB>;
        case 7: return bos::launch_demod<7, COUNT, FB>;
        case 8: return bos::launch_demod<8, COUNT, FB>;
        case 9: return bos::launch_demod<9, COUNT, FB>;
        case 10: return bos::launch_demod<10, COUNT, FB>;
        case 11: return bos::launch_demod<11, COUNT, FB>;
        case 12: return bos::launch_demod<12, COUNT, FB>;
        case 13: return bos::launch_demod<13, COUNT, FB>;
        case 14: return bos::launch_demod<14, COUNT, FB>;
        case 15: return bos::launch_demod<15, COUNT, FB>;
        case 16: return bos::launch_demod<16, COUNT, FB>;
        case 17: return bos::launch_demod<17, COUNT, FB>;
        case 18: return bos::launch_demod<18, COUNT, FB>;
        case 19: return bos::launch_demod<19, COUNT, FB>;
        case 20: return bos::launch_demod<20, COUNT, FB>;
        case 21: return bos::launch_demod<21, COUNT, FB>;
        case 22: return bos::launch_demod<22, COUNT, FB>;
        case 23: return bos::launch_demod<23, COUNT, FB>;
        case 24: return bos::launch_demod<24, COUNT, FB>;
        case 25: return bos::launch_demod<25, COUNT, FB>;
        case 26: return bos::launch_demod<26, COUNT, FB>;
        case 27: return bos::launch_demod<27, COUNT, FB>;
        case 28: return bos::launch_demod<28, COUNT, FB>;
        case 29: return bos::launch_demod<29, COUNT, FB>;
        case 30: return bos::launch_demod<30, COUNT, FB>;
        case 31: return bos::launch_demod<31, COUNT, FB>;
        case 32: return bos::launch_demod<32, COUNT, FB>;
        default: return nullptr;
    }
}

using LaunchF64 = cudaError_t (*)(const float2*, int, int, int, int, const float*, float*, uint8_t*, float*, float*,
                                  cudaStream_t);

template <bool FB>
LaunchF64 pick_ss(int MS) {
    switch (MS) {
        case 3: return bos::launch_demod_ss<3, FB>;
        case 4: return bos::launch_demod_ss<4, FB>;
        case 5: return bos::launch_demod_ss<5, FB>;
        case 6: return bos::launch_demod_ss<6, FB>;
        case 7: return bos::launch_demod_ss<7, FB>;
        case 8: return bos::launch_demod_ss<8, FB>;
        case 9: return bos::launch_demod_ss<9, FB>;
        case 10: return bos::launch_demod_ss<10, FB>;
        case 11: return bos::launch_demod_ss<11, FB>;
        case 12: return bos::launch_demod_ss<12, FB>;
        case 13: return bos::launch_demod_ss<13, FB>;
        case 14: return bos::launch_demod_ss<14, FB>;
        case 15: return bos::launch_demod_ss<15, FB>;
        case 16: return bos::launch_demod_ss<16, FB>;
        default: return nullptr;
    }
}

template <bool FB>
LaunchF64 pick_f64(int M) {
    switch (M) {
        case 3: return bos::launch_demod_f64<3, FB>;
        case 4: return bos::launch_demod_f64<4, FB>;
        case 5: return bos::launch_demod_f64<5, FB>;
        case 6: return bos::launch_demod_f64<6, FB>;
        case 7: return bos::launch_demod_f64<7, FB>;
        case 8: return bos::launch_demod_f64<8, FB>;
        case 9: return bos::launch_demod_f64<9, FB>;
        case 10: return bos::launch_demod_f64<10, FB>;
        case 11: return bos::launch_demod_f64<11, FB>;
        case 12: return bos::launch_demod_f64<12, FB>;
        case 13: return bos::launch_demod_f64<13, FB>;
        case 14: return bos::launch_demod_f64<14, FB>;
        case 15: return bos::launch_demod_f64<15, FB>;
        case 16: return bos::launch_demod_f64<16, FB>;
        case 17: return bos::launch_demod_f64<17, FB>;
        case 18: return bos::launch_demod_f64<18, FB>;
        case 19: return bos::launch_demod_f64<19, FB>;
        case 20: return bos::launch_demod_f64<20, FB>;
        case 21: return bos::launch_demod_f64<21, FB>;
        case 22: return bos::launch_demod_f64<22, FB>;
        case 23: return bos::launch_demod_f64<23, FB>;
        case 24: return bos::launch_demod_f64<24, FB>;
        case 25: return bos::launch_demod_f64<25, FB>;
        case 26: return bos::launch_demod_f64<26, FB>;
        case 27: return bos::launch_demod_f64<27, FB>;
        case 28: return bos::launch_demod_f64<28, FB>;
        case 29: return bos::launch_demod_f64<29, FB>;
        case 30: return bos::launch_demod_f64<30, FB>;
        case 31: return bos::launch_demod_f64<31, FB>;
        case 32: return bos::launch_demod_f64<32, FB>;
        default: return nullptr;
    }
}
static_assert(BOS_WINDOW_LEN_MAX <= BOS_TEMPLATE_M_MAX, "template table too small");

// 1 if p is a device (or managed) pointer, 0 otherwise.
int is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return 0;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
    const uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    return x < y + nb && y < x + na;
}

int check_common(int n_frames, int H, int W, int window_len, int model_order) {
    if (model_order != BOS_MODEL_ORDER) return BOS_ERR_UNSUPPORTED;
    if (window_len < BOS_WINDOW_LEN_MIN) return BOS_ERR_INVALID_ARG;
    if (window_len > BOS_WINDOW_LEN_MAX) return BOS_ERR_UNSUPPORTED;
    if (n_frames < 1 || H < window_len || W < window_len) return BOS_ERR_INVALID_ARG;
    return BOS_OK;
}

int demod_impl(const bos_cf32* frames, int n_frames, int H, int W, int window_len, int model_order,
               const float* ref_phase, float* out_phase, uint8_t* flags, unsigned long long* counters,
               void* stream, bool check_ptrs, float* omega_x = nullptr, float* omega_y = nullptr,
               int variant = BOS_VARIANT_PAPER, int subarray_len = 0) {
    int rc = check_common(n_frames, H, W, window_len, model_order);
    if (rc != BOS_OK) return rc;
    if (frames == nullptr || out_phase == nullptr) return BOS_ERR_INVALID_ARG;
    const size_t plane = (size_t)H * (size_t)W;
    const size_t n = plane * (size_t)n_frames;
    if (overlaps(frames, n * sizeof(bos_cf32), out_phase, n * sizeof(float))) return BOS_ERR_INVALID_ARG;
    if (ref_phase != nullptr && overlaps(ref_phase, plane * sizeof(float), out_phase, n * sizeof(float)))
        return BOS_ERR_INVALID_ARG;
    if (flags != nullptr && (overlaps(flags, n, out_phase, n * sizeof(float)) ||
                             overlaps(flags, n, frames, n * sizeof(bos_cf32))))
        return BOS_ERR_INVALID_ARG;
    for (float* om : {omega_x, omega_y}) {
        if (om == nullptr) continue;
        if (overlaps(om, n * sizeof(float), out_phase, n * sizeof(float)) ||
            overlaps(om, n * sizeof(float), frames, n * sizeof(bos_cf32)))
            return BOS_ERR_INVALID_ARG;
        if (check_ptrs && !is_device_ptr(om)) return BOS_ERR_INVALID_ARG;
    }
    if (omega_x != nullptr && omega_x == omega_y) return BOS_ERR_INVALID_ARG;
    if (check_ptrs) {
        if (!is_device_ptr(frames) || !is_device_ptr(out_phase)) return BOS_ERR_INVALID_ARG;
        if (ref_phase != nullptr && !is_device_ptr(ref_phase)) return BOS_ERR_INVALID_ARG;
        if (flags != nullptr && !is_device_ptr(flags)) return BOS_ERR_INVALID_ARG;
    }
    if ((variant & ~(BOS_VARIANT_FB | BOS_VARIANT_FP64)) != 0) return BOS_ERR_UNSUPPORTED;
    const int m = (subarray_len == 0) ? window_len : subarray_len;
    if (m < BOS_WINDOW_LEN_MIN || m > window_len) return BOS_ERR_INVALID_ARG;
    if ((variant != BOS_VARIANT_PAPER || m != window_len) && counters != nullptr) return BOS_ERR_UNSUPPORTED;
    const bool fb = (variant & BOS_VARIANT_FB) != 0;
    if (variant & BOS_VARIANT_FP64) {
        LaunchF64 f = fb ? pick_f64<true>(window_len) : pick_f64<false>(window_len);
        if (f == nullptr) return BOS_ERR_UNSUPPORTED;
        const cudaError_t e = f(reinterpret_cast<const float2*>(frames), n_frames, H, W, m, ref_phase, out_phase, flags,
                                omega_x, omega_y, static_cast<cudaStream_t>(stream));
        return e == cudaSuccess ? BOS_OK : BOS_ERR_CUDA;
    }
    if (m != window_len) {                       // FP32 spatial smoothing: order m ≤ 16
        LaunchF64 f = fb ? pick_ss<true>(m) : pick_ss<false>(m);
        if (f == nullptr) return BOS_ERR_UNSUPPORTED;
        const cudaError_t e = f(reinterpret_cast<const float2*>(frames), n_frames, H, W, window_len, ref_phase,
                                out_phase, flags, omega_x, omega_y, static_cast<cudaStream_t>(stream));
        return e == cudaSuccess ? BOS_OK : BOS_ERR_CUDA;
    }
    LaunchFn fn = variant == BOS_VARIANT_FB ? pick<false, true>(window_len)
                                            : (counters ? pick<true, false>(window_len) : pick<false, false>(window_len));
    if (fn == nullptr) return BOS_ERR_UNSUPPORTED;
    const cudaError_t e = fn(reinterpret_cast<const float2*>(frames), n_frames, H, W, ref_phase, out_phase,
                             flags, omega_x, omega_y, counters, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? BOS_OK : BOS_ERR_CUDA;
}

#ifndef BOS_SMALL_STACK_PX
#define BOS_SMALL_STACK_PX (1u << 20)   // ≤ this many pixels in the whole stack: one raw launch + difference
#endif
constexpr size_t kSmallStackPx = BOS_SMALL_STACK_PX;

size_t align_up(size_t v) { return (v + 255) & ~(size_t)255; }

// per-device pipeline objects of bos_rootmusic_demod_stack_host (created on first use, kept
// for the life of the process)
constexpr int kPipeDevices = 64;
struct Pipe {
    bool ready = false;
    cudaStream_t st[2] = {nullptr, nullptr};
    cudaEvent_t ev_start = nullptr, ev_ref = nullptr, ev_end[2] = {nullptr, nullptr};
};
Pipe g_pipe[kPipeDevices];
std::mutex g_pipe_mutex[kPipeDevices];

// out = wrap(a − a): exactly what the demod's fused difference writes for the reference frame
// itself (0, or NaN where a is NaN)
__global__ void self_difference_kernel(const float* __restrict__ a, size_t n, float* __restrict__ out) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = a[i] - a[i];
}

// out[i] = wrap(out[i] − ref[i mod plane]) in place: the fused store's reference difference
// (demod_kernel.cuh a7, same FP32 operations) for the small-stack path of
// bos_rootmusic_demod_stack
__global__ void ref_difference_kernel(float* __restrict__ out, size_t n, size_t plane, const float* __restrict__ ref) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        float a = out[i] - ref[i % plane];
        if (a > CUDART_PI_F) a -= 2.0f * CUDART_PI_F;
        if (a <= -CUDART_PI_F) a += 2.0f * CUDART_PI_F;
        out[i] = a;
    }
}

// Eq.(17): ∂n/∂x = (1/(2 μ f_x)) (n0/L²) φ — a pointwise scale (vectorised, HBM-bound).
__global__ void index_gradient_kernel(const float* __restrict__ phase, size_t n, float k, float* __restrict__ out) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const size_t n4 = n / 4;
    const bool aligned = ((reinterpret_cast<uintptr_t>(phase) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (aligned) {
        const float4* p4 = reinterpret_cast<const float4*>(phase);
        float4* o4 = reinterpret_cast<float4*>(out);
        for (size_t j = i; j < n4; j += stride) {
            float4 v = __ldg(p4 + j);
            v.x *= k; v.y *= k; v.z *= k; v.w *= k;
            o4[j] = v;
        }
        for (size_t j = 4 * n4 + i; j < n; j += stride) out[j] = k * phase[j];
    } else {
        for (size_t j = i; j < n; j += stride) out[j] = k * phase[j];
    }
}

// Row f3, SPEC stack_series: column-averaged phase per row.  One warp per
// (frame, row): coalesced lane-strided loads, FP64 sum and count of the finite pixels,
// shuffle reduction.  HBM-bound (4 B read per pixel).
__global__ void vertical_profile_kernel(const float* __restrict__ phase, size_t rows, int W,
                                        float* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const size_t warps = (size_t)gridDim.x * (blockDim.x >> 5);
    for (size_t r = (size_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
        const float* __restrict__ row = phase + r * (size_t)W;
        double sum = 0.0;
        int cnt = 0;
        for (int x = lane; x < W; x += 32) {
            const float v = __ldg(row + x);
            if (isfinite(v)) {
                sum += (double)v;
                ++cnt;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sum += __shfl_xor_sync(0xffffffffu, sum, o);
            cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        }
        if (lane == 0) out[r] = cnt > 0 ? (float)(sum / (double)cnt) : CUDART_NAN_F;
    }
}

}  // namespace

extern "C" {

int bos_abi_version(void) { return (1 << 16) | 1; }

const char* bos_strerror(int code) {
    switch (code) {
        case BOS_OK: return "ok";
        case BOS_ERR_INVALID_ARG: return "invalid argument (NULL pointer, size, aliasing or host/device pointer)";
        case BOS_ERR_UNSUPPORTED: return "unsupported (model_order must be 3; window_len outside the instantiated range; unknown variant)";
        case BOS_ERR_CUDA: return "CUDA runtime error or kernel launch failure";
        default: return "unknown bos_rootmusic status code";
    }
}

int bos_rootmusic_demod(const bos_cf32* frames, int n_frames, int H, int W, int window_len, int model_order,
                        const float* ref_phase, float* out_phase, uint8_t* flags, void* stream) {
    return demod_impl(frames, n_frames, H, W, window_len, model_order, ref_phase, out_phase, flags, nullptr,
                      stream, true);
}

int bos_rootmusic_demod_ex(const bos_cf32* frames, int n_frames, int H, int W, int window_len, int model_order,
                           const float* ref_phase, float* out_phase, uint8_t* flags, float* omega_x, float* omega_y,
                           void* stream) {
    return demod_impl(frames, n_frames, H, W, window_len, model_order, ref_phase, out_phase, flags, nullptr,
                      stream, true, omega_x, omega_y);
}

int bos_rootmusic_demod_variant(const bos_cf32* frames, int n_frames, int H, int W, int window_len,
                                int subarray_len, int model_order, int variant, const float* ref_phase,
                                float* out_phase, uint8_t* flags, float* omega_x, float* omega_y, void* stream) {
    return demod_impl(frames, n_frames, H, W, window_len, model_order, ref_phase, out_phase, flags, nullptr,
                      stream, true, omega_x, omega_y, variant, subarray_len);
}

int bos_index_gradient(const float* phase, size_t n, double n0, double mu, double f_x, double cell_len,
                       float* out, void* stream) {
    if (phase == nullptr || out == nullptr || n == 0) return BOS_ERR_INVALID_ARG;
    if (!(mu > 0.0) || !(f_x > 0.0) || !(cell_len > 0.0) || !(n0 > 0.0)) return BOS_ERR_INVALID_ARG;
    if (phase != out && overlaps(phase, n * sizeof(float), out, n * sizeof(float))) return BOS_ERR_INVALID_ARG;
    if (!is_device_ptr(phase) || !is_device_ptr(out)) return BOS_ERR_INVALID_ARG;
    const double k = n0 / (2.0 * mu * f_x * cell_len * cell_len);
    const unsigned blocks = (unsigned)std::min<size_t>((n / 4 + 255) / 256 + 1, 148 * 16);
    index_gradient_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(phase, n, (float)k, out);
    return cudaGetLastError() == cudaSuccess ? BOS_OK : BOS_ERR_CUDA;
}

int bos_vertical_profile(const float* phase, int n_frames, int H, int W, float* out, void* stream) {
    if (phase == nullptr || out == nullptr || n_frames < 1 || H < 1 || W < 1) return BOS_ERR_INVALID_ARG;
    const size_t rows = (size_t)n_frames * (size_t)H;
    if (overlaps(phase, rows * (size_t)W * sizeof(float), out, rows * sizeof(float))) return BOS_ERR_INVALID_ARG;
    if (!is_device_ptr(phase) || !is_device_ptr(out)) return BOS_ERR_INVALID_ARG;
    const unsigned blocks = (unsigned)std::min<size_t>((rows + 7) / 8, 148 * 16);
    vertical_profile_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(phase, rows, W, out);
    return cudaGetLastError() == cudaSuccess ? BOS_OK : BOS_ERR_CUDA;
}

int bos_rootmusic_iteration_counts(const bos_cf32* frames, int n_frames, int H, int W, int window_len,
                                   int model_order, const float* ref_phase, float* out_phase,
                                   unsigned long long* d_counters, void* stream) {
    if (d_counters == nullptr || !is_device_ptr(d_counters)) return BOS_ERR_INVALID_ARG;
    return demod_impl(frames, n_frames, H, W, window_len, model_order, ref_phase, out_phase, nullptr,
                      d_counters, stream, true);
}

int bos_rootmusic_demod_stack(const bos_cf32* frames, int n_frames, int H, int W, int window_len,
                              int model_order, int ref_index, float* ref_phase_out, float* out_phase,
                              uint8_t* flags, void* stream) {
    int rc = check_common(n_frames, H, W, window_len, model_order);
    if (rc != BOS_OK) return rc;
    if (ref_index < 0 || ref_index >= n_frames || ref_phase_out == nullptr || frames == nullptr)
        return BOS_ERR_INVALID_ARG;
    const size_t plane = (size_t)H * (size_t)W;
    if (overlaps(ref_phase_out, plane * sizeof(float), frames, plane * (size_t)n_frames * sizeof(bos_cf32)))
        return BOS_ERR_INVALID_ARG;
    if (!is_device_ptr(ref_phase_out)) return BOS_ERR_INVALID_ARG;
    if (out_phase == nullptr || !is_device_ptr(out_phase)) return BOS_ERR_INVALID_ARG;
    if (overlaps(ref_phase_out, plane * sizeof(float), out_phase, plane * (size_t)n_frames * sizeof(float)))
        return BOS_ERR_INVALID_ARG;
    cudaStream_t s0 = static_cast<cudaStream_t>(stream);
    // small stacks (a reference + flow pair of 512² frames, …): every frame raw in ONE launch,
    // then the reference difference by a pointwise kernel — a one-frame launch leaves most of
    // the last wave of the GPU idle, and the flow launch could not start before it ended
    if (n_frames > 1 && plane * (size_t)n_frames <= kSmallStackPx) {
        rc = demod_impl(frames, n_frames, H, W, window_len, model_order, nullptr, out_phase, flags, nullptr, stream,
                        true);
        if (rc != BOS_OK) return rc;
        if (cudaMemcpyAsync(ref_phase_out, out_phase + (size_t)ref_index * plane, plane * sizeof(float),
                            cudaMemcpyDeviceToDevice, s0) != cudaSuccess)
            return BOS_ERR_CUDA;
        const size_t n = plane * (size_t)n_frames;
        const unsigned blocks = (unsigned)std::min<size_t>((n + 255) / 256, 148 * 8);
        ref_difference_kernel<<<blocks, 256, 0, s0>>>(out_phase, n, plane, ref_phase_out);
        return cudaGetLastError() == cudaSuccess ? BOS_OK : BOS_ERR_CUDA;
    }
    // the reference frame once (raw α, and its flags); its own output wrap(α_ref − α_ref) is
    // exactly 0 (NaN where α_ref is) — written by a pointwise kernel instead of demodulating
    // the frame a second time; the other frames in ≤ 2 launches around it
    uint8_t* ref_flags = flags != nullptr ? flags + (size_t)ref_index * plane : nullptr;
    rc = demod_impl(frames + (size_t)ref_index * plane, 1, H, W, window_len, model_order, nullptr, ref_phase_out,
                    ref_flags, nullptr, stream, true);
    if (rc != BOS_OK) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const unsigned blocks = (unsigned)std::min<size_t>((plane + 255) / 256, 148 * 8);
    self_difference_kernel<<<blocks, 256, 0, s>>>(ref_phase_out, plane, out_phase + (size_t)ref_index * plane);
    if (cudaGetLastError() != cudaSuccess) return BOS_ERR_CUDA;
    if (ref_index > 0) {
        rc = demod_impl(frames, ref_index, H, W, window_len, model_order, ref_phase_out, out_phase, flags, nullptr,
                        stream, true);
        if (rc != BOS_OK) return rc;
    }
    const int after = n_frames - ref_index - 1;
    if (after > 0) {
        const size_t o = (size_t)(ref_index + 1) * plane;
        rc = demod_impl(frames + o, after, H, W, window_len, model_order, ref_phase_out, out_phase + o,
                        flags != nullptr ? flags + o : nullptr, nullptr, stream, true);
    }
    return rc;
}

size_t bos_rootmusic_host_workspace_bytes(int H, int W, int chunk_frames, int with_flags) {
    if (H < 1 || W < 1 || chunk_frames < 1) return 0;
    const size_t plane = (size_t)H * (size_t)W;
    const size_t c = (size_t)chunk_frames * plane;
    size_t slot = align_up(c * sizeof(bos_cf32)) + align_up(c * sizeof(float)) + (with_flags ? align_up(c) : 0);
    return align_up(plane * sizeof(float)) + 2 * slot;
}

int bos_rootmusic_demod_stack_host(const bos_cf32* h_frames, int n_frames, int H, int W, int window_len,
                                   int model_order, int ref_index, float* h_out_phase, uint8_t* h_flags,
                                   void* d_workspace, size_t workspace_bytes, int chunk_frames, void* stream) {
    int rc = check_common(n_frames, H, W, window_len, model_order);
    if (rc != BOS_OK) return rc;
    if (h_frames == nullptr || h_out_phase == nullptr || d_workspace == nullptr || chunk_frames < 1 ||
        ref_index < 0 || ref_index >= n_frames)
        return BOS_ERR_INVALID_ARG;
    if (is_device_ptr(h_frames) || is_device_ptr(h_out_phase) || (h_flags && is_device_ptr(h_flags)) ||
        !is_device_ptr(d_workspace))
        return BOS_ERR_INVALID_ARG;
    chunk_frames = std::min(chunk_frames, n_frames);
    const bool wf = h_flags != nullptr;
    if (workspace_bytes < bos_rootmusic_host_workspace_bytes(H, W, chunk_frames, wf)) return BOS_ERR_INVALID_ARG;

    const size_t plane = (size_t)H * (size_t)W;
    const size_t c = (size_t)chunk_frames * plane;
    char* base = static_cast<char*>(d_workspace);
    float* d_ref = reinterpret_cast<float*>(base);
    base += align_up(plane * sizeof(float));
    bos_cf32* d_frames[2];
    float* d_out[2];
    uint8_t* d_flags[2] = {nullptr, nullptr};
    for (int s = 0; s < 2; ++s) {
        d_frames[s] = reinterpret_cast<bos_cf32*>(base);
        base += align_up(c * sizeof(bos_cf32));
        d_out[s] = reinterpret_cast<float*>(base);
        base += align_up(c * sizeof(float));
        if (wf) {
            d_flags[s] = reinterpret_cast<uint8_t*>(base);
            base += align_up(c);
        }
    }

    cudaStream_t user = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaSuccess;
    auto ok = [&](cudaError_t x) {
        if (e == cudaSuccess && x != cudaSuccess) e = x;
        return e == cudaSuccess;
    };
    // The two side streams and four events of the pipeline are created once per device and
    // reused (a call used to create and destroy them: ~tens of µs of driver work per call).
    // One mutex per device serialises the enqueue section of concurrent calls, so an event is
    // never re-recorded by another call between its record and the waits on it.
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kPipeDevices) return BOS_ERR_CUDA;
    std::lock_guard<std::mutex> lock(g_pipe_mutex[dev]);
    Pipe& pp = g_pipe[dev];
    if (!pp.ready) {
        ok(cudaStreamCreateWithFlags(&pp.st[0], cudaStreamNonBlocking));
        ok(cudaStreamCreateWithFlags(&pp.st[1], cudaStreamNonBlocking));
        ok(cudaEventCreateWithFlags(&pp.ev_start, cudaEventDisableTiming));
        ok(cudaEventCreateWithFlags(&pp.ev_ref, cudaEventDisableTiming));
        ok(cudaEventCreateWithFlags(&pp.ev_end[0], cudaEventDisableTiming));
        ok(cudaEventCreateWithFlags(&pp.ev_end[1], cudaEventDisableTiming));
        if (e != cudaSuccess) return BOS_ERR_CUDA;
        pp.ready = true;
    }
    cudaStream_t* st = pp.st;
    cudaEvent_t ev_start = pp.ev_start, ev_ref = pp.ev_ref, *ev_end = pp.ev_end;
    if (e == cudaSuccess) {
        ok(cudaEventRecord(ev_start, user));
        ok(cudaStreamWaitEvent(st[0], ev_start, 0));
        ok(cudaStreamWaitEvent(st[1], ev_start, 0));
        // chunk 0 = the reference frame alone, on stream 0: H2D → raw α → d_ref, its own output
        // wrap(α_ref − α_ref) by the pointwise kernel (as bos_rootmusic_demod_stack), D2H
        ok(cudaMemcpyAsync(d_frames[0], h_frames + (size_t)ref_index * plane, plane * sizeof(bos_cf32),
                           cudaMemcpyHostToDevice, st[0]));
        if (e == cudaSuccess) {
            rc = demod_impl(d_frames[0], 1, H, W, window_len, model_order, nullptr, d_ref, d_flags[0], nullptr,
                            st[0], false);
            if (rc != BOS_OK && e == cudaSuccess) e = cudaErrorLaunchFailure;
        }
        if (e == cudaSuccess) {
            const unsigned blocks = (unsigned)std::min<size_t>((plane + 255) / 256, 148 * 8);
            self_difference_kernel<<<blocks, 256, 0, st[0]>>>(d_ref, plane, d_out[0]);
            ok(cudaGetLastError());
        }
        ok(cudaEventRecord(ev_ref, st[0]));
        ok(cudaMemcpyAsync(h_out_phase + (size_t)ref_index * plane, d_out[0], plane * sizeof(float),
                           cudaMemcpyDeviceToHost, st[0]));
        if (wf) ok(cudaMemcpyAsync(h_flags + (size_t)ref_index * plane, d_flags[0], plane, cudaMemcpyDeviceToHost, st[0]));
        // the other frames, [0, ref) then (ref, n), in chunks ping-ponged over the two streams
        // (H2D(k) ‖ kernel(k−1) ‖ D2H(k−2)).  Chunk sizes ramp up 1, 2, 4, … to chunk_frames and
        // halve again over the tail (never more than half of what is left), so the pipeline
        // fills and drains in about one frame's copy time instead of a whole chunk's.  Stream 1 starts its first copy before
        // it waits for the reference phase.
        bool waited_ref = false;
        int k = 1, ramp = 1;
        for (int part = 0; part < 2 && e == cudaSuccess; ++part) {
            const int lo = part == 0 ? 0 : ref_index + 1, hi = part == 0 ? ref_index : n_frames;
            for (int f0 = lo; f0 < hi && e == cudaSuccess; ++k) {
                const int s = k & 1;
                const int left = hi - f0;
                const int nk = std::min(std::min(ramp, chunk_frames), std::max(1, (left + 1) / 2));
                ramp = std::min(2 * ramp, chunk_frames);
                const size_t cnt = (size_t)nk * plane;
                ok(cudaMemcpyAsync(d_frames[s], h_frames + (size_t)f0 * plane, cnt * sizeof(bos_cf32),
                                   cudaMemcpyHostToDevice, st[s]));
                if (s == 1 && !waited_ref) {
                    ok(cudaStreamWaitEvent(st[1], ev_ref, 0));
                    waited_ref = true;
                }
                if (e != cudaSuccess) break;
                rc = demod_impl(d_frames[s], nk, H, W, window_len, model_order, d_ref, d_out[s], d_flags[s],
                                nullptr, st[s], false);
                if (rc != BOS_OK) {
                    e = cudaErrorLaunchFailure;
                    break;
                }
                ok(cudaMemcpyAsync(h_out_phase + (size_t)f0 * plane, d_out[s], cnt * sizeof(float),
                                   cudaMemcpyDeviceToHost, st[s]));
                if (wf) ok(cudaMemcpyAsync(h_flags + (size_t)f0 * plane, d_flags[s], cnt, cudaMemcpyDeviceToHost, st[s]));
                f0 += nk;
            }
        }
        cudaEventRecord(ev_end[0], st[0]);
        cudaEventRecord(ev_end[1], st[1]);
        cudaStreamWaitEvent(user, ev_end[0], 0);
        cudaStreamWaitEvent(user, ev_end[1], 0);
    }
    return e == cudaSuccess ? BOS_OK : BOS_ERR_CUDA;
}

}  // extern "C"
