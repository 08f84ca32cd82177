// nbk_kbw.cuh -- K_B in warp-stream form (k_dssum_w): the fused dssum + shared-
// node pap of the CG step (gslib gs_op; glsc3 part of T1 line 6) with
// no shared memory and no block barriers.  Every warp walks its own tiles of
// the dssum plan (grid-stride by warp; the tile order keeps the w sectors of
// a tile in L2 while the warp is on it) as a stream of batches of 256 copies:
// a batch is 32 lanes x 8 plan entries of one multiplicity group -- 4 nodes of
// m = 2, 2 of m = 4 or 1 of m = 8 per lane -- so the group (and m) is warp-
// uniform and the per-lane chains compile with constant m.  The plan entries
// of the next batch are loaded while the current batch's copies are in flight
// (software pipelining), so one global round trip is exposed per batch, with
// no barriers.  The block-barrier form k_dssum (nbk_kernels.cuh: TMA-staged
// plan rows, cp.async gather into shared memory, then the chains) spends ~28 %
// of its stall samples at the barrier after the gather (ncu, C5 FP32).
//
// Same chains (rule C4: ascending local index, written back to every copy) and
// the same pap terms (add_node_pap, rule C6) as k_dssum -- bitwise identical.
#pragma once
#include "nbk_kernels.cuh"

namespace nbk {

// Experiment (off by default): same-box C5 FP32 K_B 0.845 vs 0.570 ms for the
// block-barrier k_dssum, FP64 1.11 vs 0.78 -- half the instructions, but 24
// resident warps holding their copies in registers keep too few loads in
// flight (long-scoreboard 22.7 per issue, 37 % warps active; ncu C5 FP32).
#ifndef NBK_KBW
#define NBK_KBW 0   // 1: the fused CG step uses k_dssum_w
#endif
#ifndef NBK_KBW_MINB32
#define NBK_KBW_MINB32 3   // 256-thread blocks per SM (launch bounds; registers), FP32
#endif
#ifndef NBK_KBW_MINB64
#define NBK_KBW_MINB64 2   // ... FP64
#endif

template <typename T, bool FUSED, int PM>
__host__ __device__ constexpr bool kbw_on()
{
    return NBK_KBW && FUSED && PM == PM_NONE;
}

// Chains of one batch with multiplicity M (H = 8 / M nodes per lane): v holds
// the lane's 8 copies (node h: v[h M .. h M + M)), ix their SL positions.
template <typename T, int M>
__device__ __forceinline__ void kbw_batch(const DssumArgs<T>& a, acc_t& acc, const int32_t (&ix)[8], int nv)
{
    constexpr int H = 8 / M;
    T v[8], p0[H];
#pragma unroll
    for (int c = 0; c < 8; ++c)
        if (c < nv) {
            NBK_ASSERT(ix[c] >= 0 && (int64_t)ix[c] < a.mesh.E * a.mesh.N * a.mesh.N * a.mesh.N);
            v[c] = a.w[ix[c]];
        }
#pragma unroll
    for (int h = 0; h < H; ++h)
        if (h * M < nv) p0[h] = __ldg(a.p + ix[h * M]);
#pragma unroll
    for (int h = 0; h < H; ++h) {
        if (h * M >= nv) break;
        T sum = v[h * M];   // C4: ascending local index
#pragma unroll
        for (int c = 1; c < M; ++c) sum = add_t<T>(sum, v[h * M + c]);
#pragma unroll
        for (int c = 0; c < M; ++c) a.w[ix[h * M + c]] = sum;
        add_node_pap<T, PM_NONE>(acc, sum, p0[h], M, a.single, a.pm);
    }
}

// Position of a warp in its stream of batches.
struct KbwPos {
    int ti;          // ordinal of the warp's current tile (tile index gw + ti * TW)
    int g;           // group 0/1/2 (m = 2/4/8)
    int q0;          // first node of the batch within the group's segment of the tile
    int s0, s1, s2, n0, n1, n2;   // the tile's segments of g2 / g4 / g8 (scalars: no local memory)
    bool live;
    __device__ __forceinline__ int seg_s() const { return g == 0 ? s0 : (g == 1 ? s1 : s2); }
    __device__ __forceinline__ int seg_n() const { return g == 0 ? n0 : (g == 1 ? n1 : n2); }
};

__device__ __forceinline__ bool kbw_tile(const int32_t* toff, int ntiles, int rev, int gw, int tw, int ti,
                                         KbwPos& ps)
{
    const int i = gw + ti * tw;
    if (i >= ntiles) return false;
    const int t = rev ? ntiles - 1 - i : i;
    tile_range(toff, t, ps.s0, ps.n0, ps.s1, ps.n1, ps.s2, ps.n2);
    return true;
}
// advance to the first non-empty batch at or after (ti, g, q0)
__device__ __forceinline__ void kbw_settle(const int32_t* toff, int ntiles, int rev, int gw, int tw, KbwPos& ps)
{
    while (ps.live) {
        while (ps.g < 3 && ps.q0 >= ps.seg_n()) {
            ++ps.g;
            ps.q0 = 0;
        }
        if (ps.g < 3) return;
        ++ps.ti;
        ps.g = 0;
        ps.q0 = 0;
        ps.live = kbw_tile(toff, ntiles, rev, gw, tw, ps.ti, ps);
    }
}
// this lane's 8 plan entries of the batch at ps (nv valid), 8-byte loads
__device__ __forceinline__ void kbw_load_ix(const int32_t* g2, const int32_t* g4,
                                            const int32_t* g8, const KbwPos& ps, int lane, int32_t (&ix)[8], int& nv)
{
    const int m = 2 << ps.g;
    const int32_t* G = ps.g == 0 ? g2 : (ps.g == 1 ? g4 : g8);
    const int64_t base = (int64_t)m * (ps.seg_s() + ps.q0) + 8 * lane;   // first entry of this lane
    const int64_t end = (int64_t)m * (ps.seg_s() + ps.seg_n());
    nv = (int)(end - base < 0 ? 0 : (end - base > 8 ? 8 : end - base));
    const int2* src = reinterpret_cast<const int2*>(G + base);
#pragma unroll
    for (int c = 0; c < 4; ++c)
        if (2 * c < nv) {
            const int2 q = __ldcs(src + c);   // the plan is read once per iteration: streaming
            ix[2 * c] = q.x;
            ix[2 * c + 1] = q.y;
        }
}

template <typename T, bool FUSED, int PM = PM_NONE>
__global__ void __launch_bounds__(256, sizeof(T) == 4 ? NBK_KBW_MINB32 : NBK_KBW_MINB64) k_dssum_w(DssumArgs<T> a)
{
    acc_t acc;
    const int lane = threadIdx.x & 31;
    const int gw = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
    const int tw = (int)(gridDim.x * (blockDim.x >> 5));
    pdl_wait();
    KbwPos ps{};
    ps.live = kbw_tile(a.toff, a.ntiles, a.rev, gw, tw, 0, ps);
    kbw_settle(a.toff, a.ntiles, a.rev, gw, tw, ps);
    int32_t ix[8];
    int nv = 0;
    if (ps.live) kbw_load_ix(a.g2, a.g4, a.g8, ps, lane, ix, nv);
    while (ps.live) {
        // advance to the next batch and put its plan entries in flight with
        // this batch's copies
        const int g = ps.g;
        ps.q0 += 256 >> (g + 1);   // 32 lanes x 8 / m nodes
        kbw_settle(a.toff, a.ntiles, a.rev, gw, tw, ps);
        int32_t ixn[8];
        int nvn = 0;
        if (ps.live) kbw_load_ix(a.g2, a.g4, a.g8, ps, lane, ixn, nvn);
        if (g == 0) kbw_batch<T, 2>(a, acc, ix, nv);
        else if (g == 1) kbw_batch<T, 4>(a, acc, ix, nv);
        else kbw_batch<T, 8>(a, acc, ix, nv);
#pragma unroll
        for (int c = 0; c < 8; ++c) ix[c] = ixn[c];
        nv = nvn;
    }
    pdl_launch_dependents();
    dssum_fused_epilogue<T, PM_NONE>(a, acc);
}

}  // namespace nbk
