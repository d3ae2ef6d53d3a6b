// demod_inst.cu — explicit instantiation of the demod kernel launcher for one window size
// M = BOS_INST_M (the build compiles this file once per M, in parallel).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "demod_f64.cuh"
#include "demod_kernel.cuh"
#include "demod_ss.cuh"
#include "demod_strip.cuh"
#include "demod_wide.cuh"
#include "launch.h"

#ifndef BOS_INST_M
#error "compile with -DBOS_INST_M=<window_len>"
#endif

namespace bos {

// BOS_THREAD_KERNEL=row / =strip forces that kernel on the paper path for M ≤ BOS_STRIP_MAX_M
// (A/B timing and the bitwise test, tests/test_gpu_strip.py); unset = by launch size.  Read per
// launch: a plain getenv.  0 = auto, 1 = row, 2 = strip.
inline int thread_kernel_forced() {
    const char* e = std::getenv("BOS_THREAD_KERNEL");
    if (e == nullptr) return 0;
    return std::strcmp(e, "row") == 0 ? 1 : (std::strcmp(e, "strip") == 0 ? 2 : 0);
}

// Strip kernel launch: one work item (S rows × 32 columns of one frame) per warp (demod_strip.cuh).
// Launches too small for S ≥ BOS_STRIP_MIN_ROWS at ≥ 4 items per resident warp return
// cudaErrorNotReady without launching (a cold start per 2–4 rows costs more than the sliding
// covariance saves: C2 512² pairs ran 9 % slower) and go to the row kernel.
// KIND (strip_kind): 1 = R_y slid in registers (demod_strip_kernel), 2 = no R_y, implicit
// power iteration (demod_strip_im_kernel), 3 = the same for the FB variant (demod_strip_imfb_kernel)
template <int M, bool COUNT, int KIND>
cudaError_t launch_strip(const float2* frames, int n_frames, int H, int W, const float* ref, float* out,
                         uint8_t* flags, float* omega_x, float* omega_y, unsigned long long* counters,
                         cudaStream_t s) {
    constexpr int WARPS = KIND == 1 ? strip_warps<M>() : 1;
    constexpr size_t smem = KIND == 1 ? strip_smem_bytes<M>()
                          : (KIND == 2 ? strip_im_smem_bytes<M>() : strip_imfb_smem_bytes<M>());
    auto kern = [] {
        if constexpr (KIND == 2) return demod_strip_im_kernel<M, COUNT>;
        else if constexpr (KIND == 3) return demod_strip_imfb_kernel<M, COUNT>;
        else return demod_strip_kernel<M, COUNT>;
    }();
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    static int cached[64][2];                  // per device: CTAs/SM, SMs (benign racy cache)
    int nb = (dev >= 0 && dev < 64) ? cached[dev][0] : 0, sms = (dev >= 0 && dev < 64) ? cached[dev][1] : 0;
    if (nb <= 0 || sms <= 0) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, WARPS * 32, smem);
        if (e != cudaSuccess) return e;
        e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return e;
        if (nb < 1) return cudaErrorInvalidConfiguration;
        if (dev >= 0 && dev < 64) { cached[dev][0] = nb; cached[dev][1] = sms; }
    }
    const long long nbx = (W + kBX - 1) / kBX;
    const long long resident = (long long)nb * sms * WARPS;
    const long long row_items = (long long)n_frames * H * nbx;    // (frame, row, 32-column block)
    // S rows per item; small launches use shorter strips so every resident warp gets ≥ 4 items
    int S = BOS_STRIP_ROWS;
    while (S > 2 && row_items / S < 4 * resident) S >>= 1;
    // too small for long strips: the row kernel, except where the row / warp kernels are the
    // weaker choice even then (the implicit kernel from BOS_STRIP_SMALL_MIN_M: a 512² frame at
    // M = 20 runs 359 vs 255 Mpixel/s; up to M = 15 the row kernel's finer work items win)
    constexpr bool kAnySize = (KIND == 2 || KIND == 3) && M >= BOS_STRIP_SMALL_MIN_M;
    if (S < BOS_STRIP_MIN_ROWS && thread_kernel_forced() != 2 && !kAnySize)
        return cudaErrorNotReady;
    const long long items = (long long)n_frames * ((H + S - 1) / S) * nbx;
    const long long grid = std::min<long long>((items + WARPS - 1) / WARPS, 0x7fffffffLL);
    kern<<<(unsigned)grid, WARPS * 32, smem, s>>>(frames, n_frames, H, W, S, ref, out, flags, omega_x, omega_y,
                                                  counters);
    return cudaGetLastError();
}

template <int M, bool COUNT, bool FB>
cudaError_t launch_demod(const float2* frames, int n_frames, int H, int W, const float* ref, float* out,
                         uint8_t* flags, float* omega_x, float* omega_y, unsigned long long* counters,
                         cudaStream_t s) {
    const dim3 block(kBX, kBY, 1);
    constexpr int kKind = FB ? ((M >= kStripFbMinM && M <= kStripFbMaxM) ? 3 : 0) : strip_kind<M>();
    if constexpr (kKind > 0) {
        // paper path: the strip kernels (demod_strip.cuh); small launches fall through.  The
        // counting variant (COUNT) takes the same route, so the iteration counts of the flop
        // model are those of the kernel that runs.
        if (thread_kernel_forced() != 1) {
            const cudaError_t e =
                launch_strip<M, COUNT, kKind>(frames, n_frames, H, W, ref, out, flags, omega_x, omega_y, counters, s);
            if (e != cudaErrorNotReady) return e;
        }
    }
    if constexpr (M >= wide_min_m<FB>()) {
        const dim3 grid((unsigned)((W + kBX - 1) / kBX), (unsigned)((H + kBY - 1) / kBY),
                        (unsigned)std::min(n_frames, 65535));
        demod_wide_kernel<M, COUNT, FB><<<grid, block, 0, s>>>(frames, n_frames, H, W, ref, out, flags, omega_x, omega_y, counters);
    } else {
        // thread kernel: grid.y walks (frame, row block) items, kItemsPerCta per CTA
        const long long items = (long long)n_frames * ((H + kBY - 1) / kBY);
        const long long nbx = (W + kBX - 1) / kBX;
        // several items per CTA (so the next one is prefetched) only with prefetch and for large
        // launches (≥ ~16 waves): small ones keep the finest CTA granularity against the tail;
        // without prefetch (M > 14) 1 item per CTA measured faster (M = 16: 591 vs 550 Mpixel/s)
        const int ipc = (kPrefetch<M>() && nbx * items >= (long long)kItemsPerCta * 148 * 4 * 16) ? kItemsPerCta : 1;
        const long long gy = std::min<long long>((items + ipc - 1) / ipc, 65535);
        const dim3 grid((unsigned)nbx, (unsigned)gy, 1u);
        size_t dyn = 0;
        if constexpr (kRsmem<M, FB>()) {                  // R_y triangles in dynamic shared memory
            dyn = (size_t)kThreads * (M * (M - 1) / 2) * sizeof(unsigned long long);
            const cudaError_t e = cudaFuncSetAttribute(demod_kernel<M, COUNT, FB>,
                                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
            if (e != cudaSuccess) return e;
        }
        demod_kernel<M, COUNT, FB><<<grid, block, dyn, s>>>(frames, n_frames, H, W, ref, out, flags, omega_x, omega_y, counters);
    }
    return cudaGetLastError();
}

template <int M, bool FB>
cudaError_t launch_demod_f64(const float2* frames, int n_frames, int H, int W, int m, const float* ref, float* out,
                             uint8_t* flags, float* omega_x, float* omega_y, cudaStream_t s) {
    const dim3 block(32, 4, 1);
    const dim3 grid((unsigned)((W + 31) / 32), (unsigned)((H + 3) / 4), (unsigned)std::min(n_frames, 65535));
    f64::demod_f64_kernel<M, FB><<<grid, block, 0, s>>>(frames, n_frames, H, W, m, ref, out, flags, omega_x, omega_y);
    return cudaGetLastError();
}
template cudaError_t launch_demod_f64<BOS_INST_M, false>(const float2*, int, int, int, int, const float*, float*,
                                                         uint8_t*, float*, float*, cudaStream_t);
template cudaError_t launch_demod_f64<BOS_INST_M, true>(const float2*, int, int, int, int, const float*, float*,
                                                        uint8_t*, float*, float*, cudaStream_t);

#if BOS_INST_M <= 16
// row f4: spatially smoothed covariance of order MS = BOS_INST_M, runtime window M ≥ MS
template <int MS, bool FB>
cudaError_t launch_demod_ss(const float2* frames, int n_frames, int H, int W, int M, const float* ref, float* out,
                            uint8_t* flags, float* omega_x, float* omega_y, cudaStream_t s) {
    const size_t smem = (size_t)kBY * M * (kBX + M - 1) * sizeof(float2);
    cudaError_t e = cudaFuncSetAttribute(ss::demod_ss_kernel<MS, FB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    const dim3 block(kBX, kBY, 1);
    const dim3 grid((unsigned)((W + kBX - 1) / kBX), (unsigned)((H + kBY - 1) / kBY),
                    (unsigned)std::min(n_frames, 65535));
    ss::demod_ss_kernel<MS, FB><<<grid, block, smem, s>>>(frames, n_frames, H, W, M, ref, out, flags, omega_x, omega_y);
    return cudaGetLastError();
}
template cudaError_t launch_demod_ss<BOS_INST_M, false>(const float2*, int, int, int, int, const float*, float*,
                                                        uint8_t*, float*, float*, cudaStream_t);
template cudaError_t launch_demod_ss<BOS_INST_M, true>(const float2*, int, int, int, int, const float*, float*,
                                                       uint8_t*, float*, float*, cudaStream_t);
#endif

#define BOS_INST(COUNT, FB)                                                                                  \
    template cudaError_t launch_demod<BOS_INST_M, COUNT, FB>(const float2*, int, int, int, const float*, float*, \
                                                             uint8_t*, float*, float*, unsigned long long*,   \
                                                             cudaStream_t);
BOS_INST(false, false)
BOS_INST(true, false)
BOS_INST(false, true)   // variant f4 (forward–backward averaging); no counting instance
#undef BOS_INST
}  // namespace bos
