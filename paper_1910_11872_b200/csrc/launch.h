// launch.h — declarations of the per-M kernel launchers (one object file per window size,
// compiled in parallel from demod_inst.cu with -DBOS_INST_M=<M>).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace bos {
template <int M, bool COUNT, bool FB>
cudaError_t launch_demod(const float2* frames, int n_frames, int H, int W, const float* ref, float* out,
                         uint8_t* flags, float* omega_x, float* omega_y, unsigned long long* counters,
                         cudaStream_t s);
// row f4: the FP64 path (demod_f64.cuh)
template <int M, bool FB>
cudaError_t launch_demod_f64(const float2* frames, int n_frames, int H, int W, int m, const float* ref, float* out,
                             uint8_t* flags, float* omega_x, float* omega_y, cudaStream_t s);
// row f4: spatially smoothed covariance of order MS ≤ 16, runtime window M (demod_ss.cuh)
template <int MS, bool FB>
cudaError_t launch_demod_ss(const float2* frames, int n_frames, int H, int W, int M, const float* ref, float* out,
                            uint8_t* flags, float* omega_x, float* omega_y, cudaStream_t s);
}  // namespace bos
