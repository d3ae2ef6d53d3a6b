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
// is identical to the FP64 oracle (oracle/unwrap.py).  Phase 1 (tile_boruvka) contracts
// inside 16×16 tiles in shared memory and lists the remaining roots and crossing edges; the
// global rounds then touch only those lists: after every round the still-crossing edges are
// compacted (order-preserving), and only the tile phase's roots are re-linked (every node
// reaches its current root in two hops, find2); one full re-link at the end.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "bos_rootmusic.h"

namespace {

__device__ __forceinline__ double fin(float v) { return isfinite(v) ? (double)v : 0.0; }

// γ(d) = d − 2π·ceil((d − π)/2π), same operation order as oracle.unwrap.gamma.  Only ceil of
// the quotient enters the result, so the correctly rounded division is needed only where the
// product by 1/2π (within 2 ulp of x/2π, same sign) lies within a few ulp of a nonzero integer;
// elsewhere both quotients have the same ceiling (the FP64 divide was 8 of the reliability
// kernel's 9 divisions)
#ifndef BOS_UNWRAP_FAST_GAMMA
#define BOS_UNWRAP_FAST_GAMMA 1
#endif
__device__ __forceinline__ double gam(double d) {
    const double two_pi = 6.283185307179586;   // 2.0 * np.pi
    const double pi = 3.141592653589793;
    const double x = __dsub_rn(d, pi);
    double c;
    if (BOS_UNWRAP_FAST_GAMMA) {
        const double q = __dmul_rn(x, 0.15915494309189535);          // fl(1/2π)
        const double n = rint(q);
        c = (n != 0.0 && fabs(q - n) <= 1e-14 * fabs(q)) ? ceil(__ddiv_rn(x, two_pi)) : ceil(q);
    } else {
        c = ceil(__ddiv_rn(x, two_pi));
    }
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

// union-find node: parent (low 32 bits) and the 2π multiple relative to it (high 32 bits) in
// ONE 64-bit word, so a concurrent reader always sees a consistent (parent, offset) pair and
// pointer jumping can run in place
__device__ __forceinline__ unsigned long long pk(int parent, int off) {
    return (unsigned long long)(unsigned)parent | ((unsigned long long)(unsigned)off << 32);
}
__device__ __forceinline__ int par(unsigned long long w) { return (int)(unsigned)(w & 0xffffffffull); }
__device__ __forceinline__ int ofs(unsigned long long w) { return (int)(unsigned)(w >> 32); }
// (current root, 2π offset to it) of node p.  Invariant of the global rounds: every node points
// at a "former root" (a root when the tile phase ended) or at a current root, and every former
// root's entry is kept pointing at its current root (relink_list) — so two hops reach the root.
__device__ __forceinline__ unsigned long long find2(const unsigned long long* po, int p) {
    const unsigned long long w = po[p];
    const int r = par(w);
    if (r == p) return w;
    const unsigned long long w2 = po[r];
    return pk(par(w2), ofs(w) + ofs(w2));
}


// edge id e = 2p (p → p+1) or 2p+1 (p → p+W), p = frame·H·W + y·W + x (a batch of frames is one
// forest of independent grids).  Every id these kernels see comes from the tile phase's
// crossing-edge lists (or their compactions, or a root's best edge from them), which hold only
// existing edges — so no border test, and no integer divisions, are needed here
__device__ __forceinline__ bool edge_ends(unsigned e, int /*H*/, int W, int& p, int& q) {
    p = (int)(e >> 1);
    q = (e & 1u) ? p + W : p + 1;
    return true;
}

// the global rounds: only the edges that still cross components (the compacted list).  Pass 1
// also stores each edge's (root p, root q, key) in rec[k], so pass 2 reads them sequentially
// instead of repeating the two-hop root lookups and reliability loads (nothing changes the
// roots between the two passes)
__global__ void edge_max_list(const unsigned* __restrict__ list, unsigned n, int H, int W,
                              const double* __restrict__ rel, const unsigned long long* __restrict__ po,
                              unsigned long long* best_rel, uint4* __restrict__ rec) {
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        int p, q;
        edge_ends(list[k], H, W, p, q);
        const int rp = par(find2(po, p)), rq = par(find2(po, q));
        const unsigned long long key = (unsigned long long)__double_as_longlong(__dadd_rn(rel[p], rel[q]));
        rec[k] = make_uint4((unsigned)rp, (unsigned)rq, (unsigned)key, (unsigned)(key >> 32));
        if (rp == rq) continue;
        atomicMax(best_rel + rp, key);
        atomicMax(best_rel + rq, key);
    }
}
__global__ void edge_argmin_list(const unsigned* __restrict__ list, unsigned n, const uint4* __restrict__ rec,
                                 const unsigned long long* __restrict__ best_rel, unsigned* best_id) {
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const uint4 r = rec[k];
        if (r.x == r.y) continue;
        const unsigned long long key = (unsigned long long)r.z | ((unsigned long long)r.w << 32);
        const unsigned e = list[k];
        if (key == best_rel[r.x]) atomicMin(best_id + r.x, e);
        if (key == best_rel[r.y]) atomicMin(best_id + r.y, e);
    }
}

// ---- crossing-edge compaction: after a round's re-link every node points at its final root,
// so an edge is still needed iff its ends have different roots.  Order-preserving stream
// compaction (count → scan → scatter) keeps the list in edge-id order, hence the memory
// locality of the next round's passes (an atomically appended list lost it: 57.7 ms vs 44.6).
constexpr int kFiltThreads = 256;
constexpr int kFiltPerThread = 8;                              // one flag byte per thread
constexpr int kFiltPerBlock = kFiltThreads * kFiltPerThread;

__device__ __forceinline__ unsigned crossing_bits(const unsigned* __restrict__ list, unsigned n_in, int H, int W,
                                                  const unsigned long long* __restrict__ po, unsigned base) {
    unsigned m = 0;
#pragma unroll
    for (int j = 0; j < kFiltPerThread; ++j) {
        const unsigned idx = base + j;
        if (idx >= n_in) break;
        const unsigned e = list[idx];
        int p, q;
        if (edge_ends(e, H, W, p, q) && par(find2(po, p)) != par(find2(po, q))) m |= 1u << j;
    }
    return m;
}
__device__ __forceinline__ unsigned block_excl_scan(unsigned v, unsigned* total) {
    __shared__ unsigned wsum[kFiltThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += t;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        unsigned y = lane < kFiltThreads / 32 ? wsum[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += t;
        }
        if (lane < kFiltThreads / 32) wsum[lane] = y;        // inclusive warp-sum prefix
    }
    __syncthreads();
    const unsigned before = (w > 0 ? wsum[w - 1] : 0u) + x - v;
    if (total != nullptr) *total = wsum[kFiltThreads / 32 - 1];
    return before;
}
__global__ void __launch_bounds__(kFiltThreads) filter_count(const unsigned* __restrict__ list, unsigned n_in, int H,
                                                              int W, const unsigned long long* __restrict__ po,
                                                              uint8_t* __restrict__ bits, unsigned* __restrict__ bcount) {
    const unsigned t = blockIdx.x * kFiltThreads + threadIdx.x;
    const unsigned m = crossing_bits(list, n_in, H, W, po, t * kFiltPerThread);
    bits[t] = (uint8_t)m;
    unsigned tot;
    block_excl_scan((unsigned)__popc(m), &tot);
    if (threadIdx.x == 0) bcount[blockIdx.x] = tot;
}
// exclusive scan of the per-block counts (one CTA; nb ≤ 2^32 / 2048), total → *count
__global__ void __launch_bounds__(kFiltThreads) scan_counts(const unsigned* __restrict__ bcount, unsigned nb,
                                                             unsigned* __restrict__ boff, unsigned* __restrict__ count) {
    const unsigned per = (nb + kFiltThreads - 1) / kFiltThreads;
    const unsigned lo = threadIdx.x * per, hi = min(nb, lo + per);
    unsigned sum = 0;
    for (unsigned i = lo; i < hi; ++i) sum += bcount[i];
    unsigned tot;
    unsigned run = block_excl_scan(sum, &tot);
    for (unsigned i = lo; i < hi; ++i) {
        boff[i] = run;
        run += bcount[i];
    }
    if (threadIdx.x == 0) *count = tot;
}
__global__ void __launch_bounds__(kFiltThreads) filter_scatter(const unsigned* __restrict__ list, unsigned n_in,
                                                                const uint8_t* __restrict__ bits,
                                                                const unsigned* __restrict__ boff,
                                                                unsigned* __restrict__ out) {
    const unsigned t = blockIdx.x * kFiltThreads + threadIdx.x;
    const unsigned m = bits[t];
    unsigned pos = boff[blockIdx.x] + block_excl_scan((unsigned)__popc(m), nullptr);
    const unsigned base = t * kFiltPerThread;
#pragma unroll
    for (int j = 0; j < kFiltPerThread; ++j)
        if ((m >> j) & 1u) out[pos++] = list[base + j];
}

// e(a→b) = (γ(w_b − w_a) − (w_b − w_a)) / 2π  ∈ {−1, 0, 1}: required k(b) − k(a)
__device__ __forceinline__ int edge_k(const float* __restrict__ w, int a, int b) {
    const double dw = __dsub_rn(fin(w[b]), fin(w[a]));
    return (int)rint(__ddiv_rn(__dsub_rn(gam(dw), dw), 6.283185307179586));
}

// ---- Phase 1: Borůvka inside kTile×kTile tiles, in shared memory.  A component may contract along
// its best incident edge only if that edge is the best among ALL its incident edges (cut
// property of the unique maximum spanning tree), so every node also sees its cross-tile edges
// (reliabilities of the 1-pixel halo) — a component whose best edge leaves the tile stops
// growing here and is finished by the global rounds.  Every contracted edge is therefore a
// global MST edge, and the 2π offsets integrate along the same tree: the result is identical.
// In smooth regions most best edges are local, so the global rounds start from ~tile-sized
// components instead of single pixels (their pointer-jumping and re-link passes over all
// nodes dominated: 13.5 of 38.8 ms per 100 1024² frames in jump_list alone).
#ifndef BOS_UNWRAP_TILE
#define BOS_UNWRAP_TILE 16
#endif
constexpr int kTile = BOS_UNWRAP_TILE;
#ifndef BOS_UNWRAP_CHASE
#define BOS_UNWRAP_CHASE 1     // 1: root chains compressed by one chase_list launch; 0: jump_list pairs + readbacks
#endif
#ifndef BOS_UNWRAP_TILE_ROUNDS
#define BOS_UNWRAP_TILE_ROUNDS 32   // local Borůvka rounds (the global rounds finish whatever is left)
#endif       // 16: 256-thread CTAs, 8 per SM (32: one 1024-thread CTA per SM — its barriers stall the SM — 14.2 ms of 23.8 per 100 1024² frames)
__device__ __forceinline__ unsigned tpk(int parent, int off) { return (unsigned)(parent & 0xffff) | ((unsigned)off << 16); }
__device__ __forceinline__ int tpar(unsigned v) { return (int)(v & 0xffffu); }
__device__ __forceinline__ int tofs(unsigned v) { return (int)v >> 16; }

#ifndef BOS_UNWRAP_TILE_MIN_BLOCKS
#define BOS_UNWRAP_TILE_MIN_BLOCKS (2048 / (kTile * kTile))
#endif
__global__ void __launch_bounds__(kTile * kTile, BOS_UNWRAP_TILE_MIN_BLOCKS) tile_boruvka(const float* __restrict__ w, const double* __restrict__ rel,
                                                              int H, int W, int F, unsigned long long* __restrict__ po,
                                                              unsigned* __restrict__ roots, unsigned* __restrict__ roots0,
                                                              unsigned* __restrict__ nroots, unsigned* __restrict__ edges,
                                                              unsigned* __restrict__ nedges) {
    __shared__ unsigned node[kTile * kTile];                 // (local parent, 2π offset to it)
    __shared__ unsigned long long bkey[kTile * kTile];       // best incident key per component root
    __shared__ unsigned bid[kTile * kTile];                  // best incident edge id per component root
    __shared__ unsigned staged[kTile * kTile];
    // this node's 4 incident edges in fixed slots (right, down, left, up): the keys in shared
    // memory (registers bound the CTAs per SM: 62 registers with them in registers, 4 CTAs);
    // edge id and local index of the other end (−1: outside the tile) recomputed from p, l
    __shared__ unsigned long long skey[4][kTile * kTile];
    const int tilesx = (W + kTile - 1) / kTile, tilesy = (H + kTile - 1) / kTile;
    const int f = blockIdx.x / (tilesx * tilesy);
    const int t = blockIdx.x % (tilesx * tilesy);
    const int x0 = (t % tilesx) * kTile, y0 = (t / tilesx) * kTile;
    const int l = threadIdx.x, lx = l % kTile, ly = l / kTile;
    const int x = x0 + lx, y = y0 + ly;
    const bool valid = x < W && y < H;
    const size_t plane = (size_t)H * W;
    const int p = (int)((size_t)f * plane + (size_t)y * W + x);
    node[l] = tpk(l, 0);
    auto eid = [&](int k) -> unsigned {
        return k == 0 ? 2u * (unsigned)p : k == 1 ? 2u * (unsigned)p + 1u : k == 2 ? 2u * (unsigned)(p - 1)
                                                                                    : 2u * (unsigned)(p - W) + 1u;
    };
    auto ol = [&](int k) -> int {
        return k == 0 ? (lx + 1 < kTile ? l + 1 : -1) : k == 1 ? (ly + 1 < kTile ? l + kTile : -1)
                                                              : k == 2 ? (lx > 0 ? l - 1 : -1) : (ly > 0 ? l - kTile : -1);
    };
    unsigned has = 0;
    if (valid) {
        const double rp = rel[p];
        if (x + 1 < W) { has |= 1u; skey[0][l] = (unsigned long long)__double_as_longlong(__dadd_rn(rp, rel[p + 1])); }
        if (y + 1 < H) { has |= 2u; skey[1][l] = (unsigned long long)__double_as_longlong(__dadd_rn(rp, rel[p + W])); }
        if (x > 0)     { has |= 4u; skey[2][l] = (unsigned long long)__double_as_longlong(__dadd_rn(rel[p - 1], rp)); }
        if (y > 0)     { has |= 8u; skey[3][l] = (unsigned long long)__double_as_longlong(__dadd_rn(rel[p - W], rp)); }
    }
    __syncthreads();
    for (int round = 0; round < BOS_UNWRAP_TILE_ROUNDS; ++round) {
        const int r = tpar(node[l]);                        // fully compressed: the root
        bkey[l] = 0ull;
        bid[l] = 0xffffffffu;
        __syncthreads();
        // the incident edges that still leave the component; an edge that became internal stays
        // internal, so it leaves `has` for good
        unsigned cross = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (((has >> k) & 1u) && (ol(k) < 0 || tpar(node[ol(k)]) != r)) cross |= 1u << k;
        has = cross;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if ((cross >> k) & 1u) atomicMax(bkey + r, skey[k][l]);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (((cross >> k) & 1u) && skey[k][l] == bkey[r]) atomicMin(bid + r, eid(k));
        __syncthreads();
        // roots hook across their best edge when it stays inside the tile; the edge's tile-side
        // end that belongs to this component is p_in, the other end q_out
        unsigned out = node[l];
        if (valid && r == l && bid[l] != 0xffffffffu) {
            const unsigned e = bid[l];
            const int a = (int)(e >> 1), b = (e & 1u) ? a + W : a + 1;   // global ends
            const int la = (a - (int)((size_t)f * plane)) / W - y0, ca = (a - (int)((size_t)f * plane)) % W - x0;
            const int lb = (b - (int)((size_t)f * plane)) / W - y0, cb = (b - (int)((size_t)f * plane)) % W - x0;
            const bool ain = la >= 0 && la < kTile && ca >= 0 && ca < kTile;
            const bool bin = lb >= 0 && lb < kTile && cb >= 0 && cb < kTile;
            if (ain && bin) {
                const int lA = la * kTile + ca, lB = lb * kTile + cb;
                const bool aMine = tpar(node[lA]) == l;
                const int lin = aMine ? lA : lB, lot = aMine ? lB : lA;
                const int gin = aMine ? a : b, got = aMine ? b : a;
                const unsigned wo = node[lot], wc = node[lin];
                const int d = tpar(wo);
                const bool mutual = bid[d] == e;
                if (!(mutual && d < l)) {
                    out = tpk(d, tofs(wo) - tofs(wc) - edge_k(w, gin, got));
                }
            }
        }
        staged[l] = out;
        const bool hooked = __syncthreads_or(out != node[l]);
        if (r == l) node[l] = staged[l];
        __syncthreads();
        if (!hooked) break;
        // pointer jumping to full compression (in place, packed words stay consistent); ends
        // after a pass in which nothing changed
        for (int j = 0; j < 12; ++j) {
            const unsigned v = node[l];
            const unsigned vp = node[tpar(v)];
            const bool ch = tpar(vp) != tpar(v);
            if (ch) node[l] = tpk(tpar(vp), tofs(v) + tofs(vp));
            if (!__syncthreads_or(ch)) break;
        }
    }
    // outputs: the node entries, the list of the remaining roots (twice: the global rounds'
    // working list and the former-root list of find2), and the edges that still cross
    // components (this node's right and down edges), appended block by block
    __shared__ unsigned cnt_r, cnt_e, base_r, base_e;
    if (l == 0) cnt_r = cnt_e = 0u;
    __syncthreads();
    const unsigned v = node[l];
    const bool is_root = valid && tpar(v) == l;
    const bool cr = ((has & 1u) != 0) && (ol(0) < 0 || tpar(node[ol(0)]) != tpar(v));
    const bool cd = ((has & 2u) != 0) && (ol(1) < 0 || tpar(node[ol(1)]) != tpar(v));
    const unsigned my_r = is_root ? atomicAdd(&cnt_r, 1u) : 0u;
    const unsigned my_e = (cr || cd) ? atomicAdd(&cnt_e, (unsigned)cr + (unsigned)cd) : 0u;
    __syncthreads();
    if (l == 0) {
        base_r = atomicAdd(nroots, cnt_r);
        base_e = atomicAdd(nedges, cnt_e);
    }
    __syncthreads();
    if (is_root) {
        roots[base_r + my_r] = (unsigned)p;
        roots0[base_r + my_r] = (unsigned)p;
    }
    if (cr) edges[base_e + my_e] = eid(0);
    if (cd) edges[base_e + my_e + (cr ? 1u : 0u)] = eid(1);
    if (valid) {
        const int rl = tpar(v);
        const int gr = (int)((size_t)f * plane + (size_t)(y0 + rl / kTile) * W + (x0 + rl % kTile));
        po[p] = pk(gr, tofs(v));
    }
}

// ---- root lists: after the first rounds most nodes are not roots, so the per-round work that
// only concerns roots (reset, hook, compression of the root chains) runs over a compact list
// of the current roots; one full pass then re-links every node to its new root.
__global__ void reset_best_list(const unsigned* __restrict__ list, const unsigned* __restrict__ count,
                                unsigned long long* best_rel, unsigned* best_id) {
    const unsigned n = *count;
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const unsigned r = list[k];
        best_rel[r] = 0ull;
        best_id[r] = 0xffffffffu;
    }
}
// roots hook onto the root across their best edge; the new entry goes to staged[c] (the
// best_rel slot of root c, no longer needed) so that roots read each other's old entries
__global__ void hook_list(int H, int W, const float* __restrict__ w, const unsigned* __restrict__ list,
                          const unsigned* __restrict__ count, const unsigned long long* __restrict__ po,
                          const unsigned* __restrict__ best_id, unsigned long long* staged, int* hooked) {
    const unsigned n = *count;
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int c = (int)list[k];
        unsigned long long out = po[c];
        if (best_id[c] != 0xffffffffu) {
            const unsigned e = best_id[c];
            int p, q;
            edge_ends(e, H, W, p, q);
            const unsigned long long wp = find2(po, p), wq = find2(po, q);
            const bool pin = par(wp) == c;
            const int pc = pin ? p : q, oth = pin ? q : p;
            const unsigned long long wc = pin ? wp : wq, wo = pin ? wq : wp;
            const int d = par(wo);
            const bool mutual = best_id[d] == e;
            if (!(mutual && d < c)) {                 // of a mutual pair the smaller id stays root
                out = pk(d, ofs(wo) - ofs(wc) - edge_k(w, pc, oth));
                *hooked = 1;
            }
        }
        staged[c] = out;
    }
}
__global__ void apply_list(const unsigned* __restrict__ list, const unsigned* __restrict__ count,
                           const unsigned long long* __restrict__ staged, unsigned long long* po) {
    const unsigned n = *count;
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const unsigned c = list[k];
        po[c] = staged[c];
    }
}
#if !BOS_UNWRAP_CHASE
__global__ void jump_list(const unsigned* __restrict__ list, const unsigned* __restrict__ count,
                          unsigned long long* po, int* __restrict__ changed) {
    const unsigned n = *count;
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const unsigned i = list[k];
        const unsigned long long wi = po[i];
        const int p = par(wi);
        const unsigned long long wp = __ldcg(po + p);
        const int pp = par(wp);
        if (pp != p) {
            po[i] = pk(pp, ofs(wi) + ofs(wp));
            *changed = 1;
        }
    }
}
#endif
// compress the root chains after a round's hooks in ONE launch: every listed node follows its
// parent pointers to the root (a hooked root's chain may be several components long) and
// stores (root, Σ offsets).  Entries other threads rewrite meanwhile are ancestors with the
// matching offset sums (packed 64-bit words: a reader sees the old or the new pair, both
// consistent), so every walk ends at the same root with the same sum; the hooks leave no
// cycle (of a mutual pair the smaller id stays root).  Replaces 2·k jump_list launches and a
// host readback per two of them.
__global__ void chase_list(const unsigned* __restrict__ list, const unsigned* __restrict__ count,
                           unsigned long long* po) {
    const unsigned n = *count;
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const unsigned i = list[k];
        const unsigned long long wi = __ldcg(po + i);
        int p = par(wi);
        if (p == (int)i) continue;
        int off = ofs(wi);
        for (;;) {
            const unsigned long long wp = __ldcg(po + p);
            const int pp = par(wp);
            if (pp == p) break;
            off += ofs(wp);
            p = pp;
        }
        po[i] = pk(p, off);
    }
}
// every node: (old root r, off) → (root(r), off + off(r)); roots' entries already point at
// their final roots (after jump_list), and only roots' entries are read, so one pass suffices
__global__ void relink_all(size_t n, unsigned long long* po) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const unsigned long long wi = po[i];
        const int p = par(wi);
        const unsigned long long wp = po[p];
        const int pp = par(wp);
        if (pp != p) po[i] = pk(pp, ofs(wi) + ofs(wp));
    }
}
// the former roots (the tile phase's roots, `list0`) re-pointed at their current roots after a
// round's hooks and jumps — the only entries the two-hop lookup (find2) reads through
__global__ void relink_list(const unsigned* __restrict__ list, unsigned n, unsigned long long* po) {
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const unsigned i = list[k];
        const unsigned long long wi = po[i];
        const int p = par(wi);
        const unsigned long long wp = po[p];
        const int pp = par(wp);
        if (pp != p) po[i] = pk(pp, ofs(wi) + ofs(wp));
    }
}
__global__ void compact_roots(const unsigned* __restrict__ list, const unsigned* __restrict__ count,
                              const unsigned long long* __restrict__ po, unsigned* out, unsigned* out_count) {
    const unsigned n = *count;
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const unsigned c = list[k];
        if (par(po[c]) == (int)c) out[atomicAdd(out_count, 1u)] = c;
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

__global__ void finish(size_t plane, int F, const float* __restrict__ w, const unsigned long long* __restrict__ po,
                       const unsigned* idx, float* __restrict__ out) {
    const size_t n = plane * F;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int k0 = ofs(po[idx[i / plane]]);
        const float v = w[i];
        out[i] = isfinite(v) ? (float)((double)v + 6.283185307179586 * (double)(ofs(po[i]) - k0)) : v;
    }
}

size_t al(size_t v) { return (v + 255) & ~(size_t)255; }

struct Ws {
    double* rel;
    unsigned long long* po;           // packed (parent, 2π offset) nodes
    unsigned *list, *list2;           // current roots / next round's roots
    unsigned* list0;                  // former roots (the tile phase's), relinked every round
    unsigned long long* best_rel;
    unsigned* best_id;
    int* flags;                  // [0] hooked, [1] changed, [2] scratch, [4] / [5] list counts, [6] edge count
    unsigned long long* amax;
    unsigned* aidx;
    unsigned *edges, *edges2;    // crossing-edge lists (ping-pong), ≤ 2n ids each
    uint8_t* ebits;              // filter flags, one byte per 8 edges
    unsigned *bcount, *boff;     // filter per-block counts / offsets
    uint4* rec;                  // per listed edge: (root p, root q, key) from pass 1 for pass 2
};

size_t ws_layout(size_t n, int F, char* base, Ws* ws) {
    size_t o = 0;
    auto take = [&](size_t bytes) {
        char* p = base ? base + o : nullptr;
        o += al(bytes);
        return p;
    };
    char* r = take(n * sizeof(double));
    char* p1 = take(n * sizeof(unsigned long long));
    char* l1 = take(n * sizeof(unsigned));
    char* l2 = take(n * sizeof(unsigned));
    char* l0 = take(n * sizeof(unsigned));
    char* br = take(n * sizeof(unsigned long long));
    char* bi = take(n * sizeof(unsigned));
    char* fl = take(8 * sizeof(int));
    char* am = take(F * sizeof(unsigned long long));
    char* ai = take(F * sizeof(unsigned));
    const size_t nblk = (2 * n + kFiltPerBlock - 1) / kFiltPerBlock;
    char* e1 = take(2 * n * sizeof(unsigned));
    char* e2 = take(2 * n * sizeof(unsigned));
    char* eb = take(nblk * kFiltThreads);
    char* bc = take(nblk * sizeof(unsigned));
    char* bo = take(nblk * sizeof(unsigned));
    char* rc = take(2 * n * sizeof(uint4));
    if (ws) {
        ws->rec = (uint4*)rc;
        ws->rel = (double*)r;
        ws->po = (unsigned long long*)p1;
        ws->list = (unsigned*)l1;
        ws->list2 = (unsigned*)l2;
        ws->list0 = (unsigned*)l0;
        ws->best_rel = (unsigned long long*)br;
        ws->best_id = (unsigned*)bi;
        ws->flags = (int*)fl;
        ws->amax = (unsigned long long*)am;
        ws->aidx = (unsigned*)ai;
        ws->edges = (unsigned*)e1;
        ws->edges2 = (unsigned*)e2;
        ws->ebits = (uint8_t*)eb;
        ws->bcount = (unsigned*)bc;
        ws->boff = (unsigned*)bo;
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
#if !BOS_UNWRAP_CHASE
    int host_flags[2];
#endif
    for (int f0 = 0; f0 < n_frames; f0 += F) {
        const int nf = std::min(F, n_frames - f0);
        const size_t n = plane * nf;
        Ws ws;
        ws_layout(n, nf, static_cast<char*>(d_workspace), &ws);
        const unsigned gn = (unsigned)std::min<size_t>((n + 255) / 256, 148 * 16);
        const float* w = wrapped + (size_t)f0 * plane;
        float* out = unwrapped + (size_t)f0 * plane;
        reliability_kernel<<<gn, 256, 0, s>>>(w, H, W, nf, ws.rel);
        unsigned* cnt = reinterpret_cast<unsigned*>(ws.flags + 4);
        unsigned* cnt2 = reinterpret_cast<unsigned*>(ws.flags + 5);
        unsigned* ecount = reinterpret_cast<unsigned*>(ws.flags + 6);
        unsigned* E = ws.edges;
        unsigned* E2 = ws.edges2;
        // phase 1: tile-local Borůvka; it also emits the remaining roots and crossing edges
        if (cudaMemsetAsync(ws.flags + 4, 0, 3 * sizeof(int), s) != cudaSuccess) return BOS_ERR_CUDA;
        {
            const unsigned tiles = (unsigned)(((W + kTile - 1) / kTile) * ((H + kTile - 1) / kTile) * nf);
            tile_boruvka<<<tiles, kTile * kTile, 0, s>>>(w, ws.rel, H, W, nf, ws.po, ws.list, ws.list0, cnt, E, ecount);
        }
        unsigned host_counts[3];
        if (cudaMemcpyAsync(host_counts, ws.flags + 4, 3 * sizeof(unsigned), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return BOS_ERR_CUDA;
        const unsigned n_former = host_counts[0];
        unsigned n_edges = host_counts[2];
        for (int round = 0; round < 64; ++round) {                    // Borůvka: ≤ log2(n) rounds
            reset_best_list<<<gn, 256, 0, s>>>(ws.list, cnt, ws.best_rel, ws.best_id);
            if (n_edges == 0) break;                                    // no crossing edge: done
            {
                const unsigned gl = (unsigned)std::min<size_t>(((size_t)n_edges + 255) / 256, 148 * 16);
                edge_max_list<<<gl, 256, 0, s>>>(E, n_edges, H, W, ws.rel, ws.po, ws.best_rel, ws.rec);
                edge_argmin_list<<<gl, 256, 0, s>>>(E, n_edges, ws.rec, ws.best_rel, ws.best_id);
            }
            if (cudaMemsetAsync(ws.flags, 0, 2 * sizeof(int), s) != cudaSuccess) return BOS_ERR_CUDA;
            hook_list<<<gn, 256, 0, s>>>(H, W, w, ws.list, cnt, ws.po, ws.best_id, ws.best_rel, ws.flags);
            apply_list<<<gn, 256, 0, s>>>(ws.list, cnt, ws.best_rel, ws.po);
#if BOS_UNWRAP_CHASE
            // compress the root chains in one launch; no readback: with a crossing edge left
            // some component always hooks (Borůvka), so the edge count alone ends the loop
            chase_list<<<gn, 256, 0, s>>>(ws.list, cnt, ws.po);
#else
            for (int j = 0; j < 64; j += 2) {                             // compress the root chains
                // two in-place jumps per readback; the flag records only the second, so a pass
                // that changed nothing ends the compression
                jump_list<<<gn, 256, 0, s>>>(ws.list, cnt, ws.po, ws.flags + 2);
                if (cudaMemsetAsync(ws.flags + 1, 0, sizeof(int), s) != cudaSuccess) return BOS_ERR_CUDA;
                jump_list<<<gn, 256, 0, s>>>(ws.list, cnt, ws.po, ws.flags + 1);
                if (cudaMemcpyAsync(host_flags, ws.flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
                    cudaStreamSynchronize(s) != cudaSuccess)
                    return BOS_ERR_CUDA;
                if (!host_flags[1]) break;
            }
            if (!host_flags[0]) break;                                  // nothing hooked: one tree per frame
#endif
            {
                const unsigned gf = (unsigned)std::min<size_t>(((size_t)n_former + 255) / 256, 148 * 16);
                if (n_former > 0) relink_list<<<gf, 256, 0, s>>>(ws.list0, n_former, ws.po);
            }
            if (cudaMemsetAsync(cnt2, 0, sizeof(unsigned), s) != cudaSuccess) return BOS_ERR_CUDA;
            compact_roots<<<gn, 256, 0, s>>>(ws.list, cnt, ws.po, ws.list2, cnt2);
            std::swap(ws.list, ws.list2);
            std::swap(cnt, cnt2);
            // keep only the edges that still cross components (every node now points at its root)
            const unsigned nb = (unsigned)(((size_t)n_edges + kFiltPerBlock - 1) / kFiltPerBlock);
            filter_count<<<nb, kFiltThreads, 0, s>>>(E, n_edges, H, W, ws.po, ws.ebits, ws.bcount);
            scan_counts<<<1, kFiltThreads, 0, s>>>(ws.bcount, nb, ws.boff, ecount);
            filter_scatter<<<nb, kFiltThreads, 0, s>>>(E, n_edges, ws.ebits, ws.boff, E2);
            if (cudaMemcpyAsync(&n_edges, ecount, sizeof(unsigned), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
                cudaStreamSynchronize(s) != cudaSuccess)
                return BOS_ERR_CUDA;
            std::swap(E, E2);
        }
        relink_all<<<gn, 256, 0, s>>>(n, ws.po);                        // every node → its final root
        if (cudaMemsetAsync(ws.amax, 0, nf * sizeof(unsigned long long), s) != cudaSuccess ||
            cudaMemsetAsync(ws.aidx, 0xff, nf * sizeof(unsigned), s) != cudaSuccess)
            return BOS_ERR_CUDA;
        for (int a0 = 0; a0 < nf; a0 += 65535) {                  // grid.y = frames (≤ 65535 per launch)
            const dim3 ga((unsigned)std::min<size_t>((plane + 255) / 256, 64), (unsigned)std::min(nf - a0, 65535));
            anchor_max<<<ga, 256, 0, s>>>(plane, a0, ws.rel, ws.amax);
            anchor_argmin<<<ga, 256, 0, s>>>(plane, a0, ws.rel, ws.amax, ws.aidx);
        }
        finish<<<gn, 256, 0, s>>>(plane, nf, w, ws.po, ws.aidx, out);
        if (cudaGetLastError() != cudaSuccess) return BOS_ERR_CUDA;
    }
    return cudaStreamSynchronize(s) == cudaSuccess ? BOS_OK : BOS_ERR_CUDA;
}

}  // extern "C"
