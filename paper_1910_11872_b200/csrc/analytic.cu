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
#include <cmath>
#include <cstdint>
#include <new>

#include "bos_rootmusic.h"

namespace {

constexpr int kChunk = 8;   // frames per cuFFT batch / fused-path chunk (bounds the work area)
#ifndef BOS_F1_SHIFT_CARRIER
#define BOS_F1_SHIFT_CARRIER 1   // integral carriers removed as a spectral shift (0: always the per-pixel factor)
#endif
#ifndef BOS_F1_FUSED
#define BOS_F1_FUSED 1      // 0: the cuFFT path for every shape (A/B builds)
#endif

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

// ---- Fused path (power-of-two H, W ≤ 4096): the mask keeps only a disc of radius r around the
// carrier, i.e. n_x ≈ 2rW + 1 columns of the spectrum, so the 2-D transform is pruned to them
// and the five full-frame passes above become three, with one 8-byte complex write per output
// pixel and an intermediate of n_x·H values per frame (≈ 0.8 B/px at r = 0.05):
//   A  rows: two real rows packed as one complex W-point FFT, unpacked
//      (X_a = (Z_k + conj Z_{−k})/2, X_b = (Z_k − conj Z_{−k})/2j) at the n_x kept columns only;
//   B  the n_x columns: H-point FFT, the disc mask with its 1/(H·W) scale (the same FP64 bin
//      test as lobe_mask), inverse H-point FFT;
//   C  rows: the n_x values placed at their bins, inverse W-point FFT, carrier removal fused
//      into the store.
// Same transform as FFT → mask → iFFT: every kept bin is summed exactly once per output pixel.
// Each N-point FFT (N = N1·N2) is a four-step transform in shared memory: N2 threads run
// N1-point DFTs in registers over stride-N2 subsequences, twiddle by W_N^{n2·k1}, then N1
// threads run N2-point DFTs over the (padded) rows — two shared-memory round trips per FFT;
// twiddles W_N^m from sincospif of exact m/N.
constexpr int kFusedMaxN = 4096;
#ifndef BOS_F1_THREADS
#define BOS_F1_THREADS 128   // measured per 100 1024² frames: 64 → 1.065, 128 → 1.055, 256 → 1.119, 512 → 1.366 ms
#endif
constexpr int kFusedThreads = BOS_F1_THREADS;
#ifndef BOS_F1_MIN_BLOCKS
#define BOS_F1_MIN_BLOCKS 6     // CTAs/SM the register budget targets for FFTs of ≤ 1024 points (80 registers, no spills)
#endif
template <int N1, int N2>
constexpr int f1_min_blocks() { return N1 * N2 <= 1024 ? BOS_F1_MIN_BLOCKS : 1; }   // threads per CTA (= FFT groups × threads per FFT)

__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ void twiddles(float2* tw, int N) {      // tw[m] = e^{−2πim/N}, m < max(N/2, 1)
    for (int k = threadIdx.x; k < (N > 1 ? N / 2 : 1); k += blockDim.x) {
        float s, c;
        sincospif(2.0f * (float)k / (float)N, &s, &c);
        tw[k] = make_float2(c, -s);
    }
}
// W_N^m (conjugated for the inverse), m < N, from the half table: W^{m+N/2} = −W^m
template <bool INV>
__device__ __forceinline__ float2 twN(const float2* tw, int m, int N) {
    const int h = N >> 1;
    float2 w = tw[m & (h - 1)];
    if (m & h) w = make_float2(-w.x, -w.y);
    if (INV) w.y = -w.y;
    return w;
}
template <int R>
__device__ __forceinline__ constexpr int bitrev_c(int i) {
    int r = 0;
    for (int b = 1; b < R; b <<= 1) r = (r << 1) | ((i & b) ? 1 : 0);
    return r;
}
// R-point DFT (R = 2^k ≤ 64) of a[] in registers, natural order in and out (radix-2 DIT with a
// compile-time bit reversal); the stage twiddles W_R^{j·R/2h} = W_N^{j·N/2h}
template <int R, bool INV>
__device__ __forceinline__ void reg_fft(float2 (&a)[R], const float2* tw, int N) {
    if constexpr (R > 1) {
        float2 b[R];
#pragma unroll
        for (int i = 0; i < R; ++i) b[bitrev_c<R>(i)] = a[i];
#pragma unroll
        for (int h = 1; h < R; h <<= 1) {
#pragma unroll
            for (int j = 0; j < h; ++j) {
                const float2 w = j == 0 ? make_float2(1.0f, 0.0f) : twN<INV>(tw, j * (N / (2 * h)), N);
#pragma unroll
                for (int g = 0; g < R; g += 2 * h) {
                    const float2 u = b[g + j], t = j == 0 ? b[g + j + h] : f2mul(w, b[g + j + h]);
                    b[g + j] = make_float2(u.x + t.x, u.y + t.y);
                    b[g + j + h] = make_float2(u.x - t.x, u.y - t.y);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < R; ++i) a[i] = b[i];
    }
}
template <int N1, int N2>
struct Fft4 {
    static constexpr int N = N1 * N2, T = N1 > N2 ? N1 : N2, LD = N2 + 1, SZ = N1 * LD;
};
// one N-point DFT of S[0..N) (natural order in and out) by the threads t < Fft4::T of its group;
// every thread of the CTA calls it (barriers inside); the caller synchronises before
// (rot: the input read cyclically shifted, x'[n] = S[(n + rot) mod N])
template <int N1, int N2, bool INV>
__device__ __forceinline__ void fft4(float2* S, const float2* tw, int t, int rot = 0) {
    using F = Fft4<N1, N2>;
    {
        float2 a[N1];
        if (t < N2) {
#pragma unroll
            for (int n1 = 0; n1 < N1; ++n1) a[n1] = S[(N2 * n1 + t + rot) & (F::N - 1)];
        }
        __syncthreads();
        if (t < N2) {
            reg_fft<N1, INV>(a, tw, F::N);
#pragma unroll
            for (int k1 = 0; k1 < N1; ++k1) {
                if (k1 > 0 && t > 0) a[k1] = f2mul(twN<INV>(tw, t * k1, F::N), a[k1]);
                S[k1 * F::LD + t] = a[k1];
            }
        }
    }
    __syncthreads();
    float2 b[N2];
    if (t < N1) {
#pragma unroll
        for (int n2 = 0; n2 < N2; ++n2) b[n2] = S[t * F::LD + n2];
        reg_fft<N2, INV>(b, tw, F::N);
    }
    __syncthreads();
    if (t < N1) {
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) S[t + N1 * k2] = b[k2];
    }
    __syncthreads();
}
template <int N1, int N2>
constexpr size_t fused_smem(int G) {
    return (size_t)((Fft4<N1, N2>::N > 1 ? Fft4<N1, N2>::N / 2 : 1) + G * Fft4<N1, N2>::SZ) * sizeof(float2);
}
template <int N1, int N2>
constexpr int fused_groups() { return kFusedThreads / Fft4<N1, N2>::T; }

// A: CTA = G packed row pairs of one frame (W = N1·N2); out X[f][j][y], kx = (kx0 + j) mod W
template <int N1, int N2>
__global__ void __launch_bounds__(kFusedThreads, f1_min_blocks<N1, N2>()) f1_rows_fwd(const uint8_t* __restrict__ in, int H, int G, int kx0,
                                                             int nx, float2* __restrict__ X) {
    using F = Fft4<N1, N2>;
    constexpr int W = F::N;
    extern __shared__ float2 sm[];
    float2* tw = sm;
    float2* S = sm + (W > 1 ? W / 2 : 1);
    const int per = H / (2 * G);
    const int f = blockIdx.x / per, y0 = (blockIdx.x % per) * 2 * G;
    const size_t plane = (size_t)H * W;
    twiddles(tw, W);
    for (int i = threadIdx.x; i < G * W; i += blockDim.x) {
        const int a = i / W, c = i - a * W;
        const uint8_t* r = in + (size_t)f * plane + (size_t)(y0 + 2 * a) * W;
        S[a * F::SZ + c] = make_float2((float)r[c] * (1.0f / 255.0f), (float)r[c + W] * (1.0f / 255.0f));
    }
    __syncthreads();
    const int g = threadIdx.x / F::T;
    fft4<N1, N2, false>(S + (g < G ? g : 0) * F::SZ, tw, g < G ? threadIdx.x % F::T : F::T);
    for (int i = threadIdx.x; i < G * nx; i += blockDim.x) {
        const int j = i / G, a = i - j * G;                      // consecutive threads: consecutive rows
        const int kx = (kx0 + j) & (W - 1), km = (W - kx) & (W - 1);
        const float2 z1 = S[a * F::SZ + kx], z2 = S[a * F::SZ + km];
        float2* o = X + ((size_t)f * nx + j) * H + y0 + 2 * a;
        o[0] = make_float2(0.5f * (z1.x + z2.x), 0.5f * (z1.y - z2.y));    // (Z_k + conj Z_−k)/2
        o[1] = make_float2(0.5f * (z1.y + z2.y), -0.5f * (z1.x - z2.x));   // (Z_k − conj Z_−k)/2j
    }
}

// B: CTA = G kept columns of one frame (H = N1·N2): FFT over y, the disc mask × 1/(H·W), inverse
template <int N1, int N2>
// sy: spectral shift of the kept bins by −sy rows (an integral carrier f_y·H removed in the
// frequency domain, see f1_rows_inv), else 0
__global__ void __launch_bounds__(kFusedThreads, f1_min_blocks<N1, N2>()) f1_cols(int W, int G, int kx0, int nx, double fx, double fy, double r2,
                                                         int sy, float2* __restrict__ X) {
    using F = Fft4<N1, N2>;
    constexpr int H = F::N;
    extern __shared__ float2 sm[];
    float2* tw = sm;
    float2* S = sm + (H > 1 ? H / 2 : 1);
    const int cb = (nx + G - 1) / G;
    const int f = blockIdx.x / cb, j0 = (blockIdx.x % cb) * G;
    twiddles(tw, H);
    for (int i = threadIdx.x; i < G * H; i += blockDim.x) {
        const int a = i / H, y = i - a * H;
        S[a * F::SZ + y] = j0 + a < nx ? X[((size_t)f * nx + j0 + a) * H + y] : make_float2(0.0f, 0.0f);
    }
    __syncthreads();
    const int g = threadIdx.x / F::T;
    const int tf = g < G ? threadIdx.x % F::T : F::T;
    float2* Sg = S + (g < G ? g : 0) * F::SZ;
    fft4<N1, N2, false>(Sg, tw, tf);
    const float scale = 1.0f / (float)((size_t)H * W);
    for (int i = threadIdx.x; i < G * H; i += blockDim.x) {
        const int a = i / H, ky = i - a * H;
        if (j0 + a >= nx) continue;
        const int kx = (kx0 + j0 + a) & (W - 1);
        const double dx = __dadd_rn(bin_freq(kx, W), -fx);
        const double dy = __dadd_rn(bin_freq(ky, H), -fy);
        float2 v = S[a * F::SZ + ky];
        if (__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) <= r2) v = make_float2(v.x * scale, v.y * scale);
        else v = make_float2(0.0f, 0.0f);
        S[a * F::SZ + ky] = v;
    }
    __syncthreads();
    fft4<N1, N2, true>(Sg, tw, tf, sy);
    for (int i = threadIdx.x; i < G * H; i += blockDim.x) {
        const int a = i / H, y = i - a * H;
        if (j0 + a < nx) X[((size_t)f * nx + j0 + a) * H + y] = S[a * F::SZ + y];
    }
}

// C: CTA = G rows of one frame (W = N1·N2): the kept bins → inverse FFT over x → (carrier
// removal).  remove = 1: e^{−2πi f_x x}·e^{−2πi f_y y} from per-CTA tables, each phase reduced
// mod 1 in FP64, multiplied into the store; remove = 2 (integral carrier, f_x·W = sx and
// f_y·H = sy bins): the same factor as a cyclic shift of the spectrum by (−sy, −sx) — exact in
// the DFT, no per-pixel multiply (rows here, columns in f1_cols)
template <int N1, int N2>
__global__ void __launch_bounds__(kFusedThreads, f1_min_blocks<N1, N2>()) f1_rows_inv(const float2* __restrict__ X, int H, int G, int kx0,
                                                             int nx, double fx, double fy, int remove, int sx,
                                                             float2* __restrict__ out) {
    using F = Fft4<N1, N2>;
    constexpr int W = F::N;
    extern __shared__ float2 sm[];
    float2* tw = sm;
    float2* S = sm + (W > 1 ? W / 2 : 1);
    float2* ex = S + G * F::SZ;                       // carrier tables: W + G entries
    const int per = H / G;
    const int f = blockIdx.x / per, y0 = (blockIdx.x % per) * G;
    twiddles(tw, W);
    for (int i = threadIdx.x; i < G * F::SZ; i += blockDim.x) S[i] = make_float2(0.0f, 0.0f);
    if (remove == 1) {
        for (int i = threadIdx.x; i < W + G; i += blockDim.x) {
            double ph = i < W ? fx * (double)i : fy * (double)(y0 + i - W);
            ph -= floor(ph);
            float sn, cs;
            sincospif(-2.0f * (float)ph, &sn, &cs);
            ex[i] = make_float2(cs, sn);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < G * nx; i += blockDim.x) {
        const int j = i / G, a = i - j * G;
        S[a * F::SZ + ((kx0 + j - sx) & (W - 1))] = X[((size_t)f * nx + j) * H + y0 + a];
    }
    __syncthreads();
    const int g = threadIdx.x / F::T;
    fft4<N1, N2, true>(S + (g < G ? g : 0) * F::SZ, tw, g < G ? threadIdx.x % F::T : F::T);
    float2* o = out + ((size_t)f * H + y0) * W;
    for (int i = threadIdx.x; i < G * W; i += blockDim.x) {
        const int a = i / W, c = i - a * W;
        float2 v = S[a * F::SZ + c];
        if (remove == 1) v = f2mul(v, f2mul(ex[c], ex[W + a]));
        o[i] = v;
    }
}

bool pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }
int ilog2(int n) { int l = 0; while ((1 << l) < n) ++l; return l; }
bool fused_shape(int H, int W) { return pow2(H) && pow2(W) && H >= 2 && W >= 2 && H <= kFusedMaxN && W <= kFusedMaxN; }

// the kept columns: the hull, in frequency order, of the kx whose FP64 |f(kx) − f_x|² ≤ r²
// (a superset of every disc bin's column: d² = dx² + dy² ≥ dx² in round-to-nearest); kx0 and
// the count (contiguous mod W)
void kept_columns(int W, double fx, double r2, int* kx0, int* nx) {
    int smin = -1, smax = -1;
    for (int s = 0; s < W; ++s) {                     // shifted order: frequency (s − W/2)/W
        const int kx = (s + W / 2) & (W - 1);
        const int kk = (kx <= (W - 1) / 2) ? kx : kx - W;
        const double freq = (double)kk * (1.0 / (double)W);
        const double dx = freq - fx;
        if (dx * dx <= r2) {
            if (smin < 0) smin = s;
            smax = s;
        }
    }
    *kx0 = smin < 0 ? 0 : (smin + W / 2) & (W - 1);
    *nx = smin < 0 ? 0 : smax - smin + 1;
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
    bool fused;              // power-of-two H, W ≤ 4096: the pruned three-pass path, no cuFFT plans
    cufftHandle full, one;
    size_t work;
};

namespace {

template <int N1, int N2>
int launch_rows(const uint8_t* in, float2* X, float2* out, int nb, int H, int kx0, int nx, double fx, double fy,
                int remove, int sx, cudaStream_t s, bool fwd) {
    using F = Fft4<N1, N2>;
    if (fwd) {
        const int G = std::max(1, std::min(fused_groups<N1, N2>(), H / 2));
        const size_t sm = fused_smem<N1, N2>(G);
        if (cudaFuncSetAttribute(f1_rows_fwd<N1, N2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
            return BOS_ERR_CUDA;
        f1_rows_fwd<N1, N2><<<(unsigned)(nb * (H / (2 * G))), G * F::T, sm, s>>>(in, H, G, kx0, nx, X);
    } else {
        const int G = std::max(1, std::min(fused_groups<N1, N2>(), H));
        const size_t sm = fused_smem<N1, N2>(G) + (remove == 1 ? (size_t)(F::N + G) * sizeof(float2) : 0);   // carrier tables only for the per-pixel factor
        if (cudaFuncSetAttribute(f1_rows_inv<N1, N2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
            return BOS_ERR_CUDA;
        f1_rows_inv<N1, N2><<<(unsigned)(nb * (H / G)), G * F::T, sm, s>>>(X, H, G, kx0, nx, fx, fy, remove, sx, out);
    }
    return cudaGetLastError() == cudaSuccess ? BOS_OK : BOS_ERR_CUDA;
}
template <int N1, int N2>
int launch_cols(float2* X, int nb, int W, int kx0, int nx, double fx, double fy, double r2, int sy, cudaStream_t s) {
    using F = Fft4<N1, N2>;
    const int G = std::max(1, std::min(fused_groups<N1, N2>(), nx));
    const size_t sm = fused_smem<N1, N2>(G);
    if (cudaFuncSetAttribute(f1_cols<N1, N2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
        return BOS_ERR_CUDA;
    f1_cols<N1, N2><<<(unsigned)(nb * ((nx + G - 1) / G)), G * F::T, sm, s>>>(W, G, kx0, nx, fx, fy, r2, sy, X);
    return cudaGetLastError() == cudaSuccess ? BOS_OK : BOS_ERR_CUDA;
}
// N = 2^logN → (N1, N2) = (2^⌈logN/2⌉, 2^⌊logN/2⌋)
#define BOS_F1_SIZES(X) X(1, 2, 1) X(2, 2, 2) X(3, 4, 2) X(4, 4, 4) X(5, 8, 4) X(6, 8, 8) X(7, 16, 8) \
    X(8, 16, 16) X(9, 32, 16) X(10, 32, 32) X(11, 64, 32) X(12, 64, 64)

int run_fused(bos_analytic_plan* pl, const uint8_t* frames_u8, int n_frames, double fx, double fy, double radius,
              int remove, bos_cf32* out, void* d_workspace, cudaStream_t s) {
    const int H = pl->H, W = pl->W, logH = ilog2(H), logW = ilog2(W);
    const size_t plane = (size_t)H * (size_t)W;
    int kx0 = 0, nx = 0;
    kept_columns(W, fx, radius * radius, &kx0, &nx);
    if (nx == 0)                                     // no bin inside the disc: Γ ≡ 0
        return cudaMemsetAsync(out, 0, plane * (size_t)n_frames * sizeof(bos_cf32), s) == cudaSuccess ? BOS_OK
                                                                                                  : BOS_ERR_CUDA;
    // an integral carrier (f_x·W, f_y·H whole bins) is removed as a spectral shift
    const double cxw = fx * (double)W, cyh = fy * (double)H;
    const bool integral = remove && BOS_F1_SHIFT_CARRIER && cxw == std::floor(cxw) && cyh == std::floor(cyh);
    const int rmode = !remove ? 0 : (integral ? 2 : 1);
    const int sx = integral ? (int)(((long long)cxw % W + W) % W) : 0;
    const int sy = integral ? (int)(((long long)cyh % H + H) % H) : 0;
    float2* X = static_cast<float2*>(d_workspace);
    for (int f0 = 0; f0 < n_frames; f0 += pl->batch) {
        const int nb = std::min(pl->batch, n_frames - f0);
        const uint8_t* in = frames_u8 + (size_t)f0 * plane;
        float2* o = reinterpret_cast<float2*>(out) + (size_t)f0 * plane;
        int rc = BOS_ERR_UNSUPPORTED;
        switch (logW) {
#define BOS_F1_ROWS_FWD(L, A, B) case L: rc = launch_rows<A, B>(in, X, o, nb, H, kx0, nx, fx, fy, rmode, sx, s, true); break;
            BOS_F1_SIZES(BOS_F1_ROWS_FWD)
#undef BOS_F1_ROWS_FWD
        }
        if (rc != BOS_OK) return rc;
        rc = BOS_ERR_UNSUPPORTED;
        switch (logH) {
#define BOS_F1_COLS(L, A, B) case L: rc = launch_cols<A, B>(X, nb, W, kx0, nx, fx, fy, radius * radius, sy, s); break;
            BOS_F1_SIZES(BOS_F1_COLS)
#undef BOS_F1_COLS
        }
        if (rc != BOS_OK) return rc;
        rc = BOS_ERR_UNSUPPORTED;
        switch (logW) {
#define BOS_F1_ROWS_INV(L, A, B) case L: rc = launch_rows<A, B>(in, X, o, nb, H, kx0, nx, fx, fy, rmode, sx, s, false); break;
            BOS_F1_SIZES(BOS_F1_ROWS_INV)
#undef BOS_F1_ROWS_INV
        }
        if (rc != BOS_OK) return rc;
    }
    return BOS_OK;
}

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
    if (pl->fused) return run_fused(pl, frames_u8, n_frames, fx, fy, radius, remove, out, d_workspace, s);
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
    pl->fused = fused_shape(H, W) && BOS_F1_FUSED;
    if (pl->fused) {                  // the n_x·H intermediate per frame, n_x ≤ W; no cuFFT plans
        pl->full = pl->one = 0;
        pl->work = (size_t)pl->batch * (size_t)H * (size_t)W * sizeof(float2);
        if (workspace_bytes != nullptr) *workspace_bytes = pl->work;
        *plan = pl;
        return BOS_OK;
    }
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
    if (!plan->fused) {
        cufftDestroy(plan->full);
        cufftDestroy(plan->one);
    }
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
    // (the fused path's plan holds none: no synchronisation)
    if (!pl->fused && cudaStreamSynchronize(s) != cudaSuccess && rc == BOS_OK) rc = BOS_ERR_CUDA;
    bos_analytic_plan_destroy(pl);
    return rc;
}

}  // extern "C"
