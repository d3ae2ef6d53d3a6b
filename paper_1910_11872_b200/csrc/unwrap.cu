// unwrap.cu — SURVEY §8 row f2: 2-D phase unwrapping by reliability sorting (Herráez et al.,
// cited at P:L218 "followed by an unwrapping operation"), the step after the root-MUSIC path.
//
// Herráez processes edges by decreasing reliability and merges pixel groups, shifting the
// smaller group by 2π multiples so that the unwrapped difference across the merging edge is
// the wrapped one.  The merging edges are exactly Kruskal's maximum spanning tree of the
// reliability-ordered edges, and the result is the integral of the wrapped differences along
// that tree (pinned by tests/test_oracle_unwrap.py).  On the GPU the same tree is built by
// Borůvka rounds — every component picks its best edge under the same strict total order
// (reliability desc, edge id asc), so the MST is the same unique tree — with a weighted
// union-find: each node carries its 2π multiple relative to its parent, roots hook onto the
// chosen neighbour's root with the offset that satisfies the edge, and pointer jumping sums
// offsets to the root.  The reliabilities are computed in FP64 with the oracle's operation
// order and IEEE round-to-nearest intrinsics, so the edge order — and hence every 2π multiple —
// is identical to the FP64 oracle (oracle/unwrap.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "bos_rootmusic.h"

namespace {

__device__ __forceinline__ double fin(float v) { return isfinite(v) ? (double)v : 0.0; }

// γ(d) = d − 2π·ceil((d − π)/2π), same operation order as oracle.unwrap.gamma
__device__ __forceinline__ double gam(double d) {
    const double two_pi = 6.283185307179586;   // 2.0 * np.pi
    const double pi = 3.141592653589793;
    const double c = ceil(__ddiv_rn(__dsub_rn(d, pi), two_pi));
    return __dsub_rn(d, __dmul_rn(two_pi, c));
}

__global__ void reliability_kernel(const float* __restrict__ w, int H, int W, int F, double* __restrict__ rel) {
    const size_t plane = (size_t)H * W, n = plane * F;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const size_t f0 = (i / plane) * plane, loc = i - f0;
        const int y = (int)(loc / W), x = (int)(loc % W);
        auto at = [&](int dy, int dx) {
            const int yy = min(max(y + dy, 0), H - 1), xx = min(max(x + dx, 0), W - 1);
            return fin(w[f0 + (size_t)yy * W + xx]);
        };
        const double c = at(0, 0);
        const double h = __dsub_rn(gam(__dsub_rn(at(0, -1), c)), gam(__dsub_rn(c, at(0, 1))));
        const double v = __dsub_rn(gam(__dsub_rn(at(-1, 0), c)), gam(__dsub_rn(c, at(1, 0))));
        const double d1 = __dsub_rn(gam(__dsub_rn(at(-1, -1), c)), gam(__dsub_rn(c, at(1, 1))));
        const double d2 = __dsub_rn(gam(__dsub_rn(at(-1, 1), c)), gam(__dsub_rn(c, at(1, -1))));
        const double s = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(h, h), __dmul_rn(v, v)), __dmul_rn(d1, d1)),
                                   __dmul_rn(d2, d2));
        rel[i] = __ddiv_rn(1.0, __dsqrt_rn(s));
    }
}

__global__ void init_kernel(size_t n, int* parent, int* off) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        parent[i] = (int)i;
        off[i] = 0;
    }
}

__global__ void reset_best(size_t n, unsigned long long* best_rel, unsigned* best_id) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        best_rel[i] = 0ull;
        best_id[i] = 0xffffffffu;
    }
}

// edge id e = 2p (p → p+1) or 2p+1 (p → p+W), p = frame·H·W + y·W + x (a batch of frames is one
// forest of independent grids); returns false for the missing border edges
__device__ __forceinline__ bool edge_ends(unsigned e, int H, int W, int& p, int& q) {
    p = (int)(e >> 1);
    const int loc = p % (H * W);
    const int x = loc % W, y = loc / W;
    if (e & 1u) {
        if (y + 1 >= H) return false;
        q = p + W;
    } else {
        if (x + 1 >= W) return false;
        q = p + 1;
    }
    return true;
}

// pass 1: every component's largest incident cross-edge reliability (positive doubles order as u64)
__global__ void edge_max(int H, int W, int F, const double* __restrict__ rel, const int* __restrict__ parent,
                         unsigned long long* best_rel) {
    const size_t ne = 2 * (size_t)H * W * F;
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += (size_t)gridDim.x * blockDim.x) {
        int p, q;
        if (!edge_ends((unsigned)e, H, W, p, q)) continue;
        const int rp = parent[p], rq = parent[q];
        if (rp == rq) continue;
        const unsigned long long key = (unsigned long long)__double_as_longlong(__dadd_rn(rel[p], rel[q]));
        atomicMax(best_rel + rp, key);
        atomicMax(best_rel + rq, key);
    }
}

// pass 2: among the edges at that reliability, the smallest id
__global__ void edge_argmin(int H, int W, int F, const double* __restrict__ rel, const int* __restrict__ parent,
                            const unsigned long long* __restrict__ best_rel, unsigned* best_id) {
    const size_t ne = 2 * (size_t)H * W * F;
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += (size_t)gridDim.x * blockDim.x) {
        int p, q;
        if (!edge_ends((unsigned)e, H, W, p, q)) continue;
        const int rp = parent[p], rq = parent[q];
        if (rp == rq) continue;
        const unsigned long long key = (unsigned long long)__double_as_longlong(__dadd_rn(rel[p], rel[q]));
        if (key == best_rel[rp]) atomicMin(best_id + rp, (unsigned)e);
        if (key == best_rel[rq]) atomicMin(best_id + rq, (unsigned)e);
    }
}

// e(a→b) = (γ(w_b − w_a) − (w_b − w_a)) / 2π  ∈ {−1, 0, 1}: required k(b) − k(a)
__device__ __forceinline__ int edge_k(const float* __restrict__ w, int a, int b) {
    const double dw = __dsub_rn(fin(w[b]), fin(w[a]));
    return (int)rint(__ddiv_rn(__dsub_rn(gam(dw), dw), 6.283185307179586));
}

// roots hook onto the root across their best edge (reads parent/off, writes parent2/off2)
__global__ void hook(int H, int W, int F, const float* __restrict__ w, const int* __restrict__ parent,
                     const int* __restrict__ off, const unsigned* __restrict__ best_id, int* __restrict__ parent2,
                     int* __restrict__ off2, int* __restrict__ hooked) {
    const size_t n = (size_t)H * W * F;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int c = (int)i;
        int np = parent[c], no = off[c];
        if (np == c && best_id[c] != 0xffffffffu) {
            const unsigned e = best_id[c];
            int p, q;
            edge_ends(e, H, W, p, q);
            const int pc = parent[p] == c ? p : q;
            const int po = pc == p ? q : p;
            const int d = parent[po];
            const bool mutual = best_id[d] == e;
            if (!(mutual && d < c)) {                 // of a mutual pair the smaller id stays root
                np = d;
                no = off[po] - off[pc] - edge_k(w, pc, po);
                *hooked = 1;
            }
        }
        parent2[c] = np;
        off2[c] = no;
    }
}

// pointer jumping: parent ← parent(parent), off ← off + off(parent)
__global__ void jump(size_t n, const int* __restrict__ parent, const int* __restrict__ off, int* __restrict__ parent2,
                     int* __restrict__ off2, int* __restrict__ changed) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int p = parent[i];
        const int pp = parent[p];
        parent2[i] = pp;
        off2[i] = off[i] + off[p];
        if (pp != p) *changed = 1;
    }
}

// Per-frame max reliability (step 4's anchor) and the lowest pixel index attaining it: grid.y
// = frame, grid.x blocks stride over the plane; block-level reduction, then ONE atomic per
// block (a per-pixel atomic on one address per frame serialised: 50 ms for 100 1024² frames).
// Reliabilities are ≥ 0, so their IEEE bit patterns order like the values.
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, v, o);
        v = t > v ? t : v;
    }
    return v;
}
__device__ __forceinline__ unsigned warp_min_u32(unsigned v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__global__ void anchor_max(size_t plane, int f0, const double* __restrict__ rel, unsigned long long* best) {
    __shared__ unsigned long long red[32];
    const int f = f0 + (int)blockIdx.y;
    const double* r = rel + (size_t)f * plane;
    unsigned long long m = 0ull;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < plane; i += (size_t)gridDim.x * blockDim.x) {
        const unsigned long long v = (unsigned long long)__double_as_longlong(r[i]);
        m = v > m ? v : m;
    }
    m = warp_max_u64(m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0ull;
        m = warp_max_u64(m);
        if (threadIdx.x == 0) atomicMax(best + f, m);
    }
}
__global__ void anchor_argmin(size_t plane, int f0, const double* __restrict__ rel, const unsigned long long* best,
                              unsigned* idx) {
    __shared__ unsigned red[32];
    const int f = f0 + (int)blockIdx.y;
    const double* r = rel + (size_t)f * plane;
    const unsigned long long b = best[f];
    unsigned m = 0xffffffffu;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < plane; i += (size_t)gridDim.x * blockDim.x)
        if ((unsigned long long)__double_as_longlong(r[i]) == b) m = min(m, (unsigned)((size_t)f * plane + i));
    m = warp_min_u32(m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0xffffffffu;
        m = warp_min_u32(m);
        if (threadIdx.x == 0 && m != 0xffffffffu) atomicMin(idx + f, m);
    }
}

__global__ void finish(size_t plane, int F, const float* __restrict__ w, const int* __restrict__ off,
                       const unsigned* idx, float* __restrict__ out) {
    const size_t n = plane * F;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int k0 = off[idx[i / plane]];
        const float v = w[i];
        out[i] = isfinite(v) ? (float)((double)v + 6.283185307179586 * (double)(off[i] - k0)) : v;
    }
}

size_t al(size_t v) { return (v + 255) & ~(size_t)255; }

struct Ws {
    double* rel;
    int *parent, *off, *parent2, *off2;
    unsigned long long* best_rel;
    unsigned* best_id;
    int* flags;                  // [0] hooked, [1] changed
    unsigned long long* amax;
    unsigned* aidx;
};

size_t ws_layout(size_t n, int F, char* base, Ws* ws) {
    size_t o = 0;
    auto take = [&](size_t bytes) {
        char* p = base ? base + o : nullptr;
        o += al(bytes);
        return p;
    };
    char* r = take(n * sizeof(double));
    char* p1 = take(n * sizeof(int));
    char* o1 = take(n * sizeof(int));
    char* p2 = take(n * sizeof(int));
    char* o2 = take(n * sizeof(int));
    char* br = take(n * sizeof(unsigned long long));
    char* bi = take(n * sizeof(unsigned));
    char* fl = take(4 * sizeof(int));
    char* am = take(F * sizeof(unsigned long long));
    char* ai = take(F * sizeof(unsigned));
    if (ws) {
        ws->rel = (double*)r;
        ws->parent = (int*)p1;
        ws->off = (int*)o1;
        ws->parent2 = (int*)p2;
        ws->off2 = (int*)o2;
        ws->best_rel = (unsigned long long*)br;
        ws->best_id = (unsigned*)bi;
        ws->flags = (int*)fl;
        ws->amax = (unsigned long long*)am;
        ws->aidx = (unsigned*)ai;
    }
    return o;
}

bool is_dev(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace

extern "C" {

size_t bos_unwrap_workspace_bytes(int H, int W, int n_frames) {
    if (H < 1 || W < 1 || n_frames < 1) return 0;
    const size_t n = (size_t)H * W * n_frames;
    if (n * 2 >= 0xffffffffull) return 0;
    return ws_layout(n, n_frames, nullptr, nullptr);
}

int bos_unwrap(const float* wrapped, int n_frames, int H, int W, float* unwrapped, void* d_workspace,
               size_t workspace_bytes, void* stream) {
    if (wrapped == nullptr || unwrapped == nullptr || d_workspace == nullptr || n_frames < 1 || H < 1 || W < 1)
        return BOS_ERR_INVALID_ARG;
    const size_t plane = (size_t)H * W;
    if (plane * 2 >= 0xffffffffull) return BOS_ERR_INVALID_ARG;       // edge ids are 32-bit
    // as many frames per batch as the workspace (and 32-bit ids) allow
    int F = n_frames;
    while (F > 1 && (bos_unwrap_workspace_bytes(H, W, F) == 0 || bos_unwrap_workspace_bytes(H, W, F) > workspace_bytes))
        F = (F + 1) / 2;
    if (workspace_bytes < bos_unwrap_workspace_bytes(H, W, F)) return BOS_ERR_INVALID_ARG;
    if (!is_dev(wrapped) || !is_dev(unwrapped) || !is_dev(d_workspace)) return BOS_ERR_INVALID_ARG;
    const uintptr_t a = (uintptr_t)wrapped, b = (uintptr_t)unwrapped;
    const size_t tot = plane * (size_t)n_frames * sizeof(float);
    if (a != b && a < b + tot && b < a + tot) return BOS_ERR_INVALID_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int host_flags[2];
    for (int f0 = 0; f0 < n_frames; f0 += F) {
        const int nf = std::min(F, n_frames - f0);
        const size_t n = plane * nf;
        Ws ws;
        ws_layout(n, nf, static_cast<char*>(d_workspace), &ws);
        const unsigned gn = (unsigned)std::min<size_t>((n + 255) / 256, 148 * 16);
        const unsigned ge = (unsigned)std::min<size_t>((2 * n + 255) / 256, 148 * 16);
        const float* w = wrapped + (size_t)f0 * plane;
        float* out = unwrapped + (size_t)f0 * plane;
        reliability_kernel<<<gn, 256, 0, s>>>(w, H, W, nf, ws.rel);
        init_kernel<<<gn, 256, 0, s>>>(n, ws.parent, ws.off);
        for (int round = 0; round < 64; ++round) {                    // Borůvka: ≤ log2(n) rounds
            reset_best<<<gn, 256, 0, s>>>(n, ws.best_rel, ws.best_id);
            edge_max<<<ge, 256, 0, s>>>(H, W, nf, ws.rel, ws.parent, ws.best_rel);
            edge_argmin<<<ge, 256, 0, s>>>(H, W, nf, ws.rel, ws.parent, ws.best_rel, ws.best_id);
            if (cudaMemsetAsync(ws.flags, 0, 2 * sizeof(int), s) != cudaSuccess) return BOS_ERR_CUDA;
            hook<<<gn, 256, 0, s>>>(H, W, nf, w, ws.parent, ws.off, ws.best_id, ws.parent2, ws.off2, ws.flags);
            std::swap(ws.parent, ws.parent2);
            std::swap(ws.off, ws.off2);
            for (int j = 0; j < 64; j += 2) {                             // compress to the roots
                if (cudaMemsetAsync(ws.flags + 1, 0, sizeof(int), s) != cudaSuccess) return BOS_ERR_CUDA;
                for (int t = 0; t < 2; ++t) {                             // two jumps per readback
                    jump<<<gn, 256, 0, s>>>(n, ws.parent, ws.off, ws.parent2, ws.off2, ws.flags + 1);
                    std::swap(ws.parent, ws.parent2);
                    std::swap(ws.off, ws.off2);
                }
                if (cudaMemcpyAsync(host_flags, ws.flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
                    cudaStreamSynchronize(s) != cudaSuccess)
                    return BOS_ERR_CUDA;
                if (!host_flags[1]) break;
            }
            if (!host_flags[0]) break;                                  // nothing hooked: one tree per frame
        }
        if (cudaMemsetAsync(ws.amax, 0, nf * sizeof(unsigned long long), s) != cudaSuccess ||
            cudaMemsetAsync(ws.aidx, 0xff, nf * sizeof(unsigned), s) != cudaSuccess)
            return BOS_ERR_CUDA;
        for (int a0 = 0; a0 < nf; a0 += 65535) {                  // grid.y = frames (≤ 65535 per launch)
            const dim3 ga((unsigned)std::min<size_t>((plane + 255) / 256, 64), (unsigned)std::min(nf - a0, 65535));
            anchor_max<<<ga, 256, 0, s>>>(plane, a0, ws.rel, ws.amax);
            anchor_argmin<<<ga, 256, 0, s>>>(plane, a0, ws.rel, ws.amax, ws.aidx);
        }
        finish<<<gn, 256, 0, s>>>(plane, nf, w, ws.off, ws.aidx, out);
        if (cudaGetLastError() != cudaSuccess) return BOS_ERR_CUDA;
    }
    return cudaStreamSynchronize(s) == cudaSuccess ? BOS_OK : BOS_ERR_CUDA;
}

}  // extern "C"
