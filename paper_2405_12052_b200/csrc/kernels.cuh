// kernels.cuh -- sm_100a kernels of one Lloyd iteration (arXiv 2405.12052).
//
// Step map (DESIGN.md section 1 / section 5):
//   k_prep / k_input_bbox / k_morton / k_gather_sorted / k_chunk_bbox
//                   create: input -> padded AoSoA fp32 tiles (Hilbert- or
//                   Z-curve-sorted by default), non-finite check, per-chunk /
//                   super-box boxes
//   k_init_gather   mu^0_k = (double) x[init_idx[k]]
//   k_assign_pruned sorted shard (default): one warp per 1024-point chunk fed by
//                   TMA bulk copies; exact box and bisector bounds keep only the
//                   centroids that can be a point's argmin; form-D distances (packed
//                   f32x2), strict-< argmin (lowest index on ties), fused fp64
//                   sums / counts / inertia -> one sparse row per chunk
//                                                                        PAPER.md:45-52
//   k_prune / k_assign_heavy_tiles   K > 16: super-box candidate lists; chunks
//                   with more than 64 candidates, one 8-warp block per 128-point
//                   tile (k_assign_heavy: one block per chunk, KM_HEAVY_TILES=0)
//   k_assign_chunk  full scan (small shards, KMEANS_FLAG_NO_SORT), K <= 16:
//                   one warp per 2048-point chunk, centroids in registers,
//                   exact argmin via FMNMX3 + select, per-lane fp64 columns
//   k_assign_large  full scan, 16 < K <= 1024: centroids in smem
//   k_fused_iterate small full-scan shards on one GPU: many whole iterations in
//                   one cooperative launch (one grid barrier per iteration)
//   k_merge_sparse16 / k_merge_rows / k_merge_sparse   chunk rows -> groups
//   k_merge         groups -> one vector, fixed order (the OpenMP "global
//                   variable" merge of PAPER.md:97, without the critical section)
//   k_merge_update / k_update / k_p2p_update   mu^{t+1} = S/n (empty cluster
//                   keeps mu^t), E, J, stop flag (k_p2p_update: after the sum
//                   over ranks through peer memory)
//   k_generate      the synthetic mixture on the device
// No global float atomics anywhere; every reduction has a fixed order, so results
// are bit-reproducible run to run for a fixed grid.
#pragma once
#include <cooperative_groups.h>
#include <cstdio>
#include <type_traits>
#include <cuda_runtime.h>
#include <stdint.h>

namespace km {

// KM_CHECKS=1 (the "checked" test build, tools/build_variants.py): device-side
// bounds and protocol checks that trap on violation -- the stand-in for
// compute-sanitizer, which this GPU pool does not allow.  Compiled out by
// default.
#ifndef KM_CHECKS
#define KM_CHECKS 0
#endif
#if KM_CHECKS
#define KM_CHECK(c)                                                                 \
    do {                                                                            \
        if (!(c)) {                                                                 \
            printf("KM_CHECK failed: %s at %s:%d (block %d thread %d)\n", #c, __FILE__, \
                   __LINE__, (int)blockIdx.x, (int)threadIdx.x);                     \
            __trap();                                                               \
        }                                                                           \
    } while (0)
#else
#define KM_CHECK(c) \
    do {            \
    } while (0)
#endif

// Device-resident loop state (E compared with tol "at the end of each
// iteration").  t = completed iterations; mu^t lives in mu_buf[t & 1].
struct DevState {
    int t;
    int done;
    int max_iter;
    int gen;        // kmeans_start generation (P2P exchange epochs)
    double tol;
    double E;
    double J;
    int err;        // kErrExchangeTimeout: a peer never published (the run stopped)
    int pad;
};
enum : int { kErrExchangeTimeout = 1, kErrIterationTimeout = 2 };

// Global nanosecond timer (bounded waits on peers).
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Programmatic dependent launch (PDL): a kernel launched with programmatic
// stream serialization may start before its predecessor finishes; it must not
// read the predecessor's results before pdl_wait() (griddepcontrol.wait: the
// predecessor grid has completed and its writes are visible), and pdl_trigger()
// lets its own successor launch early.  Both are no-ops without the attribute.
#ifndef KM_PDL_ASSIGN_TRIGGER
#define KM_PDL_ASSIGN_TRIGGER 0   // measured: an early trigger in the assign kernel costs ~7 us
#endif
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

constexpr int kLargeTPBMax = 256;  // threads per block (max), large-K path

__device__ __forceinline__ float pos_inf() { return __int_as_float(0x7f800000); }

// Read of 2 consecutive fp32 coordinates (8-byte aligned), read-only path.
__device__ __forceinline__ float2 ld_stream2(const float* p) {
    return __ldg(reinterpret_cast<const float2*>(p));
}

// ---------------------------------------------------------------------------
// Internal point layout: AoSoA tiles of 64 points:
//   tile t = points [64t, 64t+64): x[64] | y[64] | (z[64])     (D*256 bytes)
// so one warp-tile is one contiguous TMA bulk copy, and a lane's 2 consecutive
// points of one coordinate are one 8-byte float2.
// ---------------------------------------------------------------------------
constexpr int kWarpTile = 64;

template <int D>
__device__ __forceinline__ const float* tile_coord(const float* X, int64_t p, int j) {
    return X + (p >> 6) * (D * kWarpTile) + j * kWarpTile + (p & 63);
}

// k_prep: tiled[p] <- in[p * si + j * sj] for p < N, 0 for N <= p < ldx.
// Any non-finite coordinate sets *flag (integer atomic, order-free).
__global__ void k_prep(const float* __restrict__ in, int64_t N, int d, int64_t si, int64_t sj,
                       float* __restrict__ out, int64_t ldx, int* __restrict__ flag) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ldx; i += stride) {
        for (int j = 0; j < d; ++j) {
            float v = 0.0f;
            if (i < N) {
                v = in[i * si + (int64_t)j * sj];
                bad |= !isfinite(v);
            }
            out[(i >> 6) * (d * kWarpTile) + j * kWarpTile + (i & 63)] = v;
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// mu^0_k = (double) x_{idx_k} for the indices this rank owns, 0 elsewhere (the
// allreduce over ranks then assembles mu^0 exactly: one x plus zeros).
__global__ void k_init_gather(const float* __restrict__ X, int d, int K,
                              const int64_t* __restrict__ idx, int64_t offset, int64_t n_local,
                              const int32_t* __restrict__ pos, double* __restrict__ mu0) {
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= K * d) return;
    int k = q / d, j = q % d;
    int64_t i = idx[k] - offset;
    if (pos) i = pos[k];   // sorted layout: position found by k_find_pos (-1: not local)
    KM_CHECK(i < n_local);
    KM_CHECK(!pos || i >= 0 || idx[k] < offset || idx[k] - offset >= n_local);   // local -> found
    mu0[q] = (i >= 0 && i < n_local)
                 ? (double)X[(i >> 6) * (d * kWarpTile) + j * kWarpTile + (i & 63)]
                 : 0.0;
}

// Sorted layout: the sorted positions of the local initial indices.  pairs =
// (local index, k) sorted by index (host-built, npairs <= K <= 1024, staged in
// shared memory); every sorted position p looks its perm[p] up by binary
// search and, on a hit, writes pos[k] = p.  (Replaces a full inverse
// permutation: one coalesced pass over perm per kmeans_start.)
__global__ void k_find_pos(const int32_t* __restrict__ perm, int64_t n, const int2* __restrict__ pairs,
                           int npairs, int32_t* __restrict__ pos) {
    __shared__ int2 sp[1024];
    for (int t = threadIdx.x; t < npairs; t += blockDim.x) sp[t] = pairs[t];
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
        const int i = perm[p];
        int lo = 0, hi = npairs;   // first pair with index >= i
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sp[mid].x < i) lo = mid + 1;
            else hi = mid;
        }
        if (lo < npairs && sp[lo].x == i) pos[sp[lo].y] = (int32_t)p;
    }
}

// Per-block partial layout: part[e * G + b], e in [0, K*D + K + 1):
//   e <  K*D          : S_k,j  (k-major)
//   K*D <= e < K*D+K  : n_k    (exact integer in fp64)
//   e == K*D + K      : J
// Merged / allreduced vector red[e] has the same e order.

enum : int { kModeReduce = 1, kModeLabels = 2 };

// ---------------------------------------------------------------------------
// Exact argmin used by the small-K path.  KP = compile-time padded K (4, 8 or
// 16); padded slots have c = +inf so their distance is +inf and never wins.
//
// Argmin (exact, lowest index on ties): m = min_k d_k by a 3-input FMNMX tree
// (min is exact and order-free for non-NaN values), then the lowest k with
// d_k == m by short descending select chains and an integer min.  This is the same (value, index) the
// ascending strict-< scan of the oracle returns.
// ---------------------------------------------------------------------------
template <int KP>
__device__ __forceinline__ void exact_argmin(const float (&d)[KP], float& m, int& lab) {
    float t[KP];
#pragma unroll
    for (int k = 0; k < KP; ++k) t[k] = d[k];
    int n = KP;
#pragma unroll
    for (int level = 0; level < 4; ++level) {
        if (n > 1) {
            int w = 0;
#pragma unroll
            for (int k = 0; k < KP; k += 3) {
                if (k < n) {
                    float v = t[k];
                    if (k + 1 < n) v = fminf(v, t[k + 1]);
                    if (k + 2 < n) v = fminf(v, t[k + 2]);
                    t[w++] = v;
                }
            }
            n = w;
        }
    }
    m = t[0];
    // lowest k with d_k == m: descending select chains over groups of 4 (each
    // yields its lowest match or KP), then the minimum over the groups.
    int g[KP / 4];
#pragma unroll
    for (int q = 0; q < KP / 4; ++q) {
        int l = KP;
#pragma unroll
        for (int k = 4 * q + 3; k >= 4 * q; --k) l = (d[k] == m) ? k : l;
        g[q] = l;
    }
    int l = g[0];
#pragma unroll
    for (int q = 1; q < KP / 4; ++q) l = min(l, g[q]);
    lab = l;
}

// ---------------------------------------------------------------------------
// Small-K path (K <= 16): k_assign_chunk.
//
// Work unit = one 2048-point chunk processed by a one-warp block.  Blocks are
// scheduled by the hardware as SMs free up, so warps the issue arbiter starves
// do not hold up the grid, and the result stays deterministic: a chunk's
// partial row depends only on its own points, summed in a fixed order.  The
// point stream is fed by TMA bulk copies (cp.async.bulk, one per 128-point
// warp-tile) into a kStages-deep shared-memory ring completed on mbarriers.
//
// Per lane: 4 points per warp-tile (2 float2 groups), packed f32x2 form-D math,
// centroids (negated fp32) in registers, exact argmin, private fp64 column.
// Partials: one coalesced row per chunk; k_merge_rows sums each group of
// kDenseGroup rows in ascending order, k_merge sums the groups.  No atomics.
// ---------------------------------------------------------------------------
constexpr int kLaneTile = 2 * kWarpTile;                 // 128 points per warp-tile
#ifndef KM_CHUNK_TILES
#define KM_CHUNK_TILES 16
#endif
#ifndef KM_SORTED_STAGES
#define KM_SORTED_STAGES 2
#endif
#ifndef KM_SORTED_CHUNK_TILES
#define KM_SORTED_CHUNK_TILES 8
#endif
#ifndef KM_TWO_CAND
#define KM_TWO_CAND 1   // register path for two-candidate chunks (K <= 16)
#endif
#ifndef KM_TWO_CAND_PRED
#define KM_TWO_CAND_PRED 1   // two-candidate chunks: predicated adds instead of +0.0 selects
#endif
#ifndef KM_REFINE_UNROLL
#define KM_REFINE_UNROLL 4   // heavy kernel's refinement loops: entries in flight per lane
#endif
constexpr int kRefineUnroll = KM_REFINE_UNROLL;
#ifndef KM_LARGE_REVERSE
#define KM_LARGE_REVERSE 1   // large-K pruned kernel: chunks in reverse order
#endif
#ifndef KM_HEAVY_PROF
#define KM_HEAVY_PROF 0   // tuning aid: per-chunk phase times of k_assign_heavy (printf)
#endif
#ifndef KM_AGG_UNIT
#define KM_AGG_UNIT 1   // large K: slot sums per TMA unit (8 points per lane), not per warp-tile
#endif
#ifndef KM_AGG_TRANSPOSE
#define KM_AGG_TRANSPOSE 1   // slot sums by a transposing butterfly (see pruned_body's agg)
#endif
#ifndef KM_CAND_UNROLL2
#define KM_CAND_UNROLL2 1   // multi-candidate argmin: two candidates per loop step
#endif
#ifndef KM_LARGE_CAP
#define KM_LARGE_CAP 64
#endif
constexpr int kChunkTiles = KM_CHUNK_TILES;
constexpr int kChunkPoints = kLaneTile * kChunkTiles;    // 2048
constexpr int kStages = 3;
#ifndef KM_SPARSE_GROUP
#define KM_SPARSE_GROUP 128   // measured at C5: 64 -> 128 saves ~5 us per iteration (k_merge reads half the groups); 256 is slower
#endif
constexpr int kGroupChunks = KM_SPARSE_GROUP;   // chunks per group, large-K sparse rows (<= 256)
#ifndef KM_ROW_GROUP
#define KM_ROW_GROUP 256
#endif
constexpr int kRowGroup = KM_ROW_GROUP;   // chunks per group, sorted small-K rows (k_merge_sparse16)
constexpr int kMergeWarps = kRowGroup / 32;
constexpr int kDenseGroup = 256;   // chunks per group, dense rows (k_merge_rows)
constexpr int kRowDoubles = 16 * 4 + 2;                  // [k][Sx Sy Sz n] + J + pad

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
#ifndef KM_EVICT_FIRST
#define KM_EVICT_FIRST 1   // the point stream (read once per iteration, >> L2) marked evict-first
#endif
// TMA bulk copy global -> shared completing on `bar`.  evict_first: an L2 hint
// for streams read once per iteration (measured: NS assign 196 -> 187 us, C3
// 121 -> 112 us); not for the large-K pruned kernel, whose multi-pass chunks
// and heavy chunks re-read their points from L2, nor for the FP32-bound full
// scan (no gain measured).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         bool evict_first = true) {
#if KM_EVICT_FIRST
    if (!evict_first) {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
            : "memory");
        return;
    }
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
#else
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
#endif
}

// L2 cache policies for the point stream (createpolicy): evict_first for the
// part of the shard streamed from HBM every iteration, evict_last for the part
// kept resident in the 126 MB L2 across iterations (the "keep" prefix).
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s_pol(void* dst, const void* src, unsigned bytes,
                                             uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

template <int D, int KP>
struct ChunkSmem {
    double2 A[KP][32];                  // {Sx, Sy} per (k, lane)
    double2 B[KP][32];                  // {Sz, n|pad} per (k, lane)
    float ring[kStages][D * kLaneTile]; // two AoSoA tiles (one warp-tile) per stage
    uint64_t bar[kStages];
    float cst[KP * D];                  // staged negated fp32 centroids
};

template <int D, int KP>
__device__ __forceinline__ void form_d_pair(const float (&nc)[KP][D], float2 x, float2 y, float2 z,
                                            float (&d0)[KP], float (&d1)[KP]) {
#pragma unroll
    for (int k = 0; k < KP; ++k) {
        float2 e0 = __fadd2_rn(x, make_float2(nc[k][0], nc[k][0]));
        float2 e1 = __fadd2_rn(y, make_float2(nc[k][1], nc[k][1]));
        float2 sq = __fmul2_rn(e0, e0);
        sq = __ffma2_rn(e1, e1, sq);
        if (D == 3) {
            float2 e2 = __fadd2_rn(z, make_float2(nc[k][2], nc[k][2]));
            sq = __ffma2_rn(e2, e2, sq);
        }
        d0[k] = sq.x;
        d1[k] = sq.y;
    }
}

__device__ __forceinline__ void mbar_inval(uint64_t* bar) {
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Start chunk `chunk`'s point stream: (re)initialise the stage barriers and
// issue the first kStages tiles (lane 0).  `reinit`: the barriers were used by
// an earlier chunk of this warp (all their copies consumed).
template <int D, int KP>
__device__ __forceinline__ void chunk_prologue(ChunkSmem<D, KP>& S, const float* __restrict__ X,
                                               int64_t n, int chunk, int lane, bool reinit) {
    constexpr int kTileFloats = D * kLaneTile;
    constexpr unsigned kTileBytes = kTileFloats * 4;
    const int64_t base = (int64_t)chunk * kChunkPoints;
    const int64_t rem = n - base;
    const int64_t ntile64 = (rem + kLaneTile - 1) / kLaneTile;
    const int ntile = ntile64 < kChunkTiles ? (int)ntile64 : kChunkTiles;
    const float* src = X + (base >> 6) * (D * kWarpTile);   // first AoSoA tile of the chunk
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < kStages; ++s) {
            if (reinit) mbar_inval(&S.bar[s]);
            mbar_init(&S.bar[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
        for (int s = 0; s < kStages; ++s) {
            if (s < ntile) {
                mbar_expect_tx(&S.bar[s], kTileBytes);
                bulk_g2s(S.ring[s], src + s * kTileFloats, kTileBytes, &S.bar[s], false);
            }
        }
    }
}

// One chunk of the full scan (after chunk_prologue): reassignment (PAPER.md:
// 45-49, form D, exact argmin) of its points, 4 per lane per warp-tile, and
// the fused numerator / denominator of the mean added to the
// lane's private fp64 columns S.A / S.B and to J, points in the fixed order
// a0, a1, b0, b1 of each tile, tiles ascending.
template <int D, int KP, int MODE>
__device__ __forceinline__ void chunk_body(ChunkSmem<D, KP>& S, const float* __restrict__ X,
                                           int64_t n, int chunk, const float (&nc)[KP][D],
                                           double& J, int32_t* __restrict__ labels, int lane) {
    constexpr int kTileFloats = D * kLaneTile;
    constexpr unsigned kTileBytes = kTileFloats * 4;
    const int64_t base = (int64_t)chunk * kChunkPoints;
    const int64_t rem = n - base;
    const int64_t ntile64 = (rem + kLaneTile - 1) / kLaneTile;
    const int ntile = ntile64 < kChunkTiles ? (int)ntile64 : kChunkTiles;
    const int nfull = rem >= kChunkPoints ? kChunkTiles : (int)(rem / kLaneTile);
    const float* src = X + (base >> 6) * (D * kWarpTile);

    auto accumulate = [&](int l, float px, float py, float pz) {
        double2 a = S.A[l][lane], b = S.B[l][lane];
        a.x += (double)px;
        a.y += (double)py;
        if (D == 3) b.x += (double)pz;
        int2 c = *reinterpret_cast<int2*>(&b.y);
        c.x += 1;
        b.y = *reinterpret_cast<double*>(&c);
        S.A[l][lane] = a;
        S.B[l][lane] = b;
    };

    // Points of one warp-tile held by a lane: a = (2L, 2L+1), b = (64+2L, 64+2L+1).
    struct Pts {
        float2 xa, ya, za, xb, yb, zb;
    };
    // Wait for tile i's stage, read this lane's points, refill the stage that
    // tile i-1 used (its values are in registers and consumed by then).
    auto fetch = [&](int i) {
        const int s = i % kStages;
        mbar_wait(&S.bar[s], (unsigned)(i / kStages) & 1u);
        const float* rg = S.ring[s];
        const float* rb = rg + D * kWarpTile;
        Pts P;
        P.xa = reinterpret_cast<const float2*>(rg)[lane];
        P.ya = reinterpret_cast<const float2*>(rg + kWarpTile)[lane];
        P.za = (D == 3) ? reinterpret_cast<const float2*>(rg + 2 * kWarpTile)[lane]
                        : make_float2(0.f, 0.f);
        P.xb = reinterpret_cast<const float2*>(rb)[lane];
        P.yb = reinterpret_cast<const float2*>(rb + kWarpTile)[lane];
        P.zb = (D == 3) ? reinterpret_cast<const float2*>(rb + 2 * kWarpTile)[lane]
                        : make_float2(0.f, 0.f);
        __syncwarp();
        const int r = i - 1 + kStages;   // tile refilled into stage (i-1) % kStages
        if (lane == 0 && i >= 1 && r < ntile) {
            const int sr = (i - 1) % kStages;
            mbar_expect_tx(&S.bar[sr], kTileBytes);
            bulk_g2s(S.ring[sr], src + (int64_t)r * kTileFloats, kTileBytes, &S.bar[sr], false);
        }
        return P;
    };
    // Reassignment, form D, 4 points per lane.
    auto assign = [&](int i, const Pts& P, float (&m)[4], int (&l)[4]) {
        float da0[KP], da1[KP], db0[KP], db1[KP];
        form_d_pair<D, KP>(nc, P.xa, P.ya, P.za, da0, da1);
        form_d_pair<D, KP>(nc, P.xb, P.yb, P.zb, db0, db1);
        exact_argmin<KP>(da0, m[0], l[0]);
        exact_argmin<KP>(da1, m[1], l[1]);
        exact_argmin<KP>(db0, m[2], l[2]);
        exact_argmin<KP>(db1, m[3], l[3]);
        if (MODE & kModeLabels) {
            const int64_t pa = base + (int64_t)i * kLaneTile + 2 * lane;
            *reinterpret_cast<int2*>(labels + pa) = make_int2(l[0], l[1]);
            *reinterpret_cast<int2*>(labels + pa + kWarpTile) = make_int2(l[2], l[3]);
        }
    };
    auto reduce_full = [&](const Pts& P, const float (&m)[4], const int (&l)[4]) {
        if (!(MODE & kModeReduce)) return;
        accumulate(l[0], P.xa.x, P.ya.x, P.za.x);
        accumulate(l[1], P.xa.y, P.ya.y, P.za.y);
        accumulate(l[2], P.xb.x, P.yb.x, P.zb.x);
        accumulate(l[3], P.xb.y, P.yb.y, P.zb.y);
        J += (double)m[0];
        J += (double)m[1];
        J += (double)m[2];
        J += (double)m[3];
    };
    auto reduce_checked = [&](int i, const Pts& P, const float (&m)[4], const int (&l)[4]) {
        if (!(MODE & kModeReduce)) return;
        const int64_t pa = base + (int64_t)i * kLaneTile + 2 * lane, pb = pa + kWarpTile;
        if (pa < n) { accumulate(l[0], P.xa.x, P.ya.x, P.za.x); J += (double)m[0]; }
        if (pa + 1 < n) { accumulate(l[1], P.xa.y, P.ya.y, P.za.y); J += (double)m[1]; }
        if (pb < n) { accumulate(l[2], P.xb.x, P.yb.x, P.zb.x); J += (double)m[2]; }
        if (pb + 1 < n) { accumulate(l[3], P.xb.y, P.yb.y, P.zb.y); J += (double)m[3]; }
    };

    if (nfull == kChunkTiles) {
        // Full chunk: software pipeline unrolled by 2 -- the smem reduction of
        // one tile sits in the same basic block as the distance math of the next,
        // so the scheduler interleaves them.
        float mA[4], mB[4];
        int lA[4], lB[4];
        Pts A = fetch(0);
        assign(0, A, mA, lA);
#pragma unroll 1
        for (int i = 1; i < kChunkTiles - 1; i += 2) {
            const Pts B = fetch(i);
            reduce_full(A, mA, lA);
            assign(i, B, mB, lB);
            A = fetch(i + 1);
            reduce_full(B, mB, lB);
            assign(i + 1, A, mA, lA);
        }
        const Pts B = fetch(kChunkTiles - 1);
        reduce_full(A, mA, lA);
        assign(kChunkTiles - 1, B, mB, lB);
        reduce_full(B, mB, lB);
    } else {
        // the last chunk: plain loop with per-point bounds
#pragma unroll 1
        for (int i = 0; i < ntile; ++i) {
            const Pts P = fetch(i);
            float m[4];
            int l[4];
            assign(i, P, m, l);
            reduce_checked(i, P, m, l);
        }
    }
}

// Lane L's entry of the warp row: the sum over the 32 lanes' private columns of
// (k = L >> 1, half = L & 1), in a rotated (bank-conflict-free) fixed order.
template <int KP, class SM>
__device__ __forceinline__ double2 columns_to_row(const SM& S, int lane) {
    const int k = lane >> 1;
    const double2* col = (lane & 1) ? &S.B[0][0] : &S.A[0][0];
    double v0 = 0.0, v1 = 0.0;
    long long cnt = 0;
    if (k < KP) {
#pragma unroll 8
        for (int r = 0; r < 32; ++r) {
            const int t = (r + lane) & 31;
            const double2 w = col[k * 32 + t];
            v0 += w.x;
            if (lane & 1) cnt += reinterpret_cast<const int2*>(&w.y)->x;
            else v1 += w.y;
        }
    }
    return (k < KP) ? ((lane & 1) ? make_double2(v0, (double)cnt) : make_double2(v0, v1))
                    : make_double2(0.0, 0.0);
}

template <int KP, class SM>
__device__ __forceinline__ void zero_columns(SM& S, int lane) {
#pragma unroll
    for (int k = 0; k < KP; ++k) {
        S.A[k][lane] = make_double2(0.0, 0.0);
        S.B[k][lane] = make_double2(0.0, 0.0);
    }
}

#ifndef KM_CHUNK_MINB
#define KM_CHUNK_MINB (D == 2 ? 16 : 10)   // measured: 2D 463 -> 442 us at C3 size; 3D unchanged
#endif
template <int D, int KP, int MODE>
__global__ void __launch_bounds__(32, KM_CHUNK_MINB)
k_assign_chunk(const float* __restrict__ X, int64_t n, int K,
               const double* __restrict__ mu_buf, const DevState* __restrict__ st,
               int mu_sel, int ignore_done, double* __restrict__ cpart,
               int32_t* __restrict__ labels) {
    if (!ignore_done && st->done) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ChunkSmem<D, KP>& S = *reinterpret_cast<ChunkSmem<D, KP>*>(smem_raw);
    const int lane = threadIdx.x;
    const int chunk = blockIdx.x;
    // kick off the point stream first (its latency overlaps the staging below)
    chunk_prologue<D, KP>(S, X, n, chunk, lane, false);

    const int t_it = st->t;
    const double* mu = mu_buf + (size_t)((t_it - mu_sel) & 1) * K * D;
    // Stage: c_k = fl32(mu_k^t) (RN), negated so that x + (-c) == x - c; each
    // lane converts <= 2 entries, the warp shares them through smem.
    for (int q = lane; q < KP * D; q += 32)
        S.cst[q] = (q < K * D) ? -__double2float_rn(__ldg(&mu[q])) : -pos_inf();
    if (MODE & kModeReduce) zero_columns<KP>(S, lane);
    __syncwarp();
    float nc[KP][D];
#pragma unroll
    for (int k = 0; k < KP; ++k) {
#pragma unroll
        for (int j = 0; j < D; ++j) nc[k][j] = S.cst[k * D + j];
    }
    double J = 0.0;
    chunk_body<D, KP, MODE>(S, X, n, chunk, nc, J, labels, lane);
    if (!(MODE & kModeReduce)) return;

    // ---- chunk partial: row[4k + j] = sum over lanes, fixed rotation order ----
    __syncwarp();
    const double2 out = columns_to_row<KP>(S, lane);
    double jj = J;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) jj += __shfl_xor_sync(0xffffffffu, jj, o);
    double* row = cpart + (size_t)chunk * kRowDoubles;
    // row layout [k][Sx, Sy, Sz, n] (k < KP), then J at 64
    reinterpret_cast<double2*>(row)[lane] = out;
    if (lane == 0) row[64] = jj;
}

// ---------------------------------------------------------------------------
// Spatially sorted path (default for K <= 16): preprocessing kernels.
//
// At kmeans_create the shard's points are put in Hilbert-curve order (3D, and
// 2D below KM_BIG_CHUNK_MIN_N) or Morton (Z-curve) order once (CUB radix sort of up to 64-bit keys; stable, so deterministic), and each
// 1024-point chunk gets its bounding box.  The order is an internal layout:
// labels are scattered back to the caller's order, and every result of the
// iteration is unchanged (sums are accumulated in a different fixed order).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned ord_f32(float f) {   // order-preserving float -> uint
    unsigned u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unord_f32(unsigned u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// Global bounding box of the input (ordered-int min/max atomics: order-free)
// plus the non-finite check.  box[0..d) = min, box[d..2d) = max (ordered ints).
// d is a template argument: the per-axis registers stay registers (a runtime d
// put them on the stack: 3x slower at create).
template <int d>
__global__ void k_input_bbox(const float* __restrict__ in, int64_t N, int64_t si, int64_t sj,
                             unsigned* __restrict__ box, int* __restrict__ flag) {
    unsigned mn[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, mx[3] = {0u, 0u, 0u};
    int bad = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) {
#pragma unroll
        for (int j = 0; j < d; ++j) {
            const float v = in[i * si + (int64_t)j * sj];
            bad |= !isfinite(v);
            const unsigned o = ord_f32(v);
            mn[j] = min(mn[j], o);
            mx[j] = max(mx[j], o);
        }
    }
#pragma unroll
    for (int j = 0; j < d; ++j) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn[j] = min(mn[j], __shfl_xor_sync(0xffffffffu, mn[j], o));
            mx[j] = max(mx[j], __shfl_xor_sync(0xffffffffu, mx[j], o));
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(&box[j], mn[j]);
            atomicMax(&box[d + j], mx[j]);
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

__device__ __forceinline__ unsigned long long part1by1_64(unsigned long long x) {   // 32 -> even bits
    x &= 0x00000000ffffffffull;
    x = (x | (x << 16)) & 0x0000ffff0000ffffull;
    x = (x | (x << 8)) & 0x00ff00ff00ff00ffull;
    x = (x | (x << 4)) & 0x0f0f0f0f0f0f0f0full;
    x = (x | (x << 2)) & 0x3333333333333333ull;
    x = (x | (x << 1)) & 0x5555555555555555ull;
    return x;
}
__device__ __forceinline__ unsigned long long part1by2_64(unsigned long long x) {  // 21 -> every 3rd
    x &= 0x1fffffull;
    x = (x | (x << 32)) & 0x1f00000000ffffull;
    x = (x | (x << 16)) & 0x1f0000ff0000ffull;
    x = (x | (x << 8)) & 0x100f00f00f00f00full;
    x = (x | (x << 4)) & 0x10c30c30c30c30c3ull;
    x = (x | (x << 2)) & 0x1249249249249249ull;
    return x;
}

// Hilbert index of a grid cell (d = 2 or 3 axes of `bits` bits each): J.
// Skilling's transform ("Programming the Hilbert curve", AIP Conf. Proc. 707,
// 2004) turns the coordinates into the curve's "transposed" index in place;
// interleaving their bits (axis 0 most significant) gives the index.  Unlike
// the Z-curve, consecutive cells are always adjacent, so a run of consecutive
// points never jumps across the box: chunk boxes stay compact and the pruning
// keeps fewer candidates.
__device__ __forceinline__ void hilbert_transpose(unsigned (&x)[3], int d, int bits) {
    const unsigned M = 1u << (bits - 1);
    for (unsigned Q = M; Q > 1; Q >>= 1) {   // inverse undo excess work (branch-free)
        const unsigned P = Q - 1;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            if (i >= d) break;
            const unsigned hit = 0u - ((x[i] & Q) != 0u);   // all ones: invert, else exchange
            x[0] ^= P & hit;
            const unsigned t = (x[0] ^ x[i]) & P & ~hit;
            x[0] ^= t;
            x[i] ^= t;
        }
    }
    for (int i = 1; i < d; ++i) x[i] ^= x[i - 1];   // Gray encode
    unsigned t = 0;
    for (unsigned Q = M; Q > 1; Q >>= 1)
        if (x[d - 1] & Q) t ^= Q - 1;
    for (int i = 0; i < d; ++i) x[i] ^= t;
}

// 64-bit Morton key of every point (qbits <= 21 bits per axis in 3D, <= 32 in 2D) on an
// isotropic grid over the global box -- cubic cells keep chunk boxes compact
// even when the box is very elongated (C5's far outliers), and the fine grid
// keeps the dense regions resolved -- with the identity permutation as values.
template <typename KeyT, int d>   // uint32 (d * qbits <= 32) or uint64 keys; d = 2 or 3
__global__ void k_morton(const float* __restrict__ in, int64_t N, int64_t si, int64_t sj,
                         const unsigned* __restrict__ box, int qbits, int hilbert,
                         KeyT* __restrict__ keys, int32_t* __restrict__ iota) {
    const double qmax = (double)((1ull << qbits) - 1ull);   // qbits <= 32 (2D), <= 21 (3D)
    double lo[3], sc[3], ext = 0.0;
#pragma unroll
    for (int j = 0; j < d; ++j) {
        lo[j] = (double)unord_f32(box[j]);
        ext = fmax(ext, (double)unord_f32(box[d + j]) - lo[j]);
    }
#pragma unroll
    for (int j = 0; j < d; ++j) sc[j] = (ext > 0.0) ? qmax / ext : 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) {
        unsigned long long q[3] = {0ull, 0ull, 0ull};
#pragma unroll
        for (int j = 0; j < d; ++j) {
            double t = ((double)in[i * si + (int64_t)j * sj] - lo[j]) * sc[j];
            t = fmin(fmax(t, 0.0), qmax);
            q[j] = (unsigned long long)t;
        }
        if (hilbert) {   // transposed Hilbert index; axis 0 the most significant
            unsigned x[3] = {(unsigned)q[0], (unsigned)q[1], (unsigned)q[2]};
            hilbert_transpose(x, d, qbits);
            q[0] = x[d - 1];
            q[1] = x[d - 2];
            q[2] = d == 3 ? x[0] : 0ull;
        }
        keys[i] = (KeyT)((d == 2) ? (part1by1_64(q[0]) | (part1by1_64(q[1]) << 1))
                                  : (part1by2_64(q[0]) | (part1by2_64(q[1]) << 1) |
                                     (part1by2_64(q[2]) << 2)));
        iota[i] = (int32_t)i;
    }
}

// Sorted AoSoA layout: point p (sorted position) = input point perm[p].
// Padding points (p >= N) are zeros.
__global__ void k_gather_sorted(const float* __restrict__ in, int64_t N, int d, int64_t si,
                                int64_t sj, const int32_t* __restrict__ perm,
                                float* __restrict__ out, int64_t ldx) {
    // U points per thread per pass, all their (random) loads in flight at once
    constexpr int U = 8;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p0 < ldx; p0 += U * stride) {
        int64_t i[U];
        float v[U][3];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t p = p0 + u * stride;
            i[u] = (p < N) ? perm[p] : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < 3; ++j)
                v[u][j] = (i[u] >= 0 && j < d) ? __ldg(in + i[u] * si + (int64_t)j * sj) : 0.0f;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t p = p0 + u * stride;
            if (p >= ldx) break;
#pragma unroll
            for (int j = 0; j < 3; ++j)
                if (j < d) out[(p >> 6) * (d * kWarpTile) + j * kWarpTile + (p & 63)] = v[u][j];
        }
    }
}

// Per-chunk bounding box of the (sorted) points: cbox[c] = {lo[D], hi[D]}.
// One warp per chunk; only valid points (p < n) count.
__global__ void k_chunk_bbox(const float* __restrict__ X, int64_t n, int d, int chunk_points,
                             int n_chunks, float* __restrict__ cbox) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= n_chunks) return;
    const int64_t p0 = (int64_t)warp * chunk_points;
    const int64_t p1 = (n < p0 + chunk_points) ? n : p0 + chunk_points;
    for (int j = 0; j < d; ++j) {
        float lo = pos_inf(), hi = -pos_inf();
        for (int64_t p = p0 + lane; p < p1; p += 32) {
            const float v = X[(p >> 6) * (d * kWarpTile) + j * kWarpTile + (p & 63)];
            lo = fminf(lo, v);
            hi = fmaxf(hi, v);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) {
            cbox[(size_t)warp * 2 * d + j] = lo;
            cbox[(size_t)warp * 2 * d + d + j] = hi;
        }
    }
}

// labels_out[perm[p]] = labels_sorted[p] for p < n (back to the caller's order).
__global__ void k_scatter_labels(const int32_t* __restrict__ lab_sorted,
                                 const int32_t* __restrict__ perm, int64_t n,
                                 int32_t* __restrict__ lab_out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
        KM_CHECK(perm[p] >= 0 && perm[p] < n);
        lab_out[perm[p]] = lab_sorted[p];
    }
}

// ---------------------------------------------------------------------------
// k_assign_pruned (sorted points): exact per-chunk pruning, any K <= 1024.
//
// For the chunk's box B and the staged fp32 centroids c_k, a lane computes in
// fp64  dmin2_k = min_{x in B} ||x - c_k||^2  and  dmax2_k = max_{x in B} ||x - c_k||^2.
// With M = min_k dmax2_k, centroid b is excluded when
//     dmin2_b > M (1 + 1e-5) + 2^-100.
// Then for every x in B the exact squared distances satisfy
// E_b > E_a (1 + 1e-5) + 2^-100 for the a attaining M, and since form D is
// within (d+2) 2^-24 relative (+ a few subnormal ulps absolute) of the exact
// value (pinned in tests/test_oracle_pins.py), D(x, c_b) > D(x, c_a) strictly
// in fp32: b can neither win nor tie.  So the exact argmin over the remaining
// candidates, scanned in ascending k with strict <, equals the full scan's
// (value, lowest index).  If M could overflow fp32 (> 1e37) nothing is pruned.
//
// Small K (<= 16): lane k evaluates centroid k.  Large K: k_prune first keeps,
// per super-chunk of kSuperChunks chunks, the candidates of the super box (the
// same test); the chunk then refines that list (a centroid excluded for the
// super box is excluded for every sub-box, and the chunk's M is attained inside
// the super list, so the refined set is exact).  More than kPCap refined
// candidates ("big" chunks, rare): the unrefined super list is used (a superset,
// still exact).
//
// One candidate: every label is known; distances are still computed (form D)
// for the inertia; sums accumulate in registers.  Several: running strict-<
// argmin over the candidates; the winning slot of each point is cached in
// shared memory; per-lane private fp64 columns hold kPSlots slots per pass and
// passes > 0 re-read the chunk's points from L2.
//
// Output: a sparse row per chunk: [J, count, entries...], entry = {Sx, Sy, Sz,
// (k, n) as int2 bits}; k_merge_sparse sums the rows of each group in fixed
// chunk order.  No float atomics.
// ---------------------------------------------------------------------------
#ifndef KM_SORTED_UNIT_SUB
#define KM_SORTED_UNIT_SUB 2
#endif
constexpr int kUnitSub = KM_SORTED_UNIT_SUB;           // 128-point sub-tiles per stage
constexpr int kSortedUnit = kUnitSub * kLaneTile;      // points per TMA stage
// Sorted path chunk: the pruning box and the partial row cover kSChunkPoints
// points (a one-warp block each).  Measured on NS (tools/sweep.py): 1024
// points beats 512 (per-block overhead) and 2048 (more multi-candidate boxes).
constexpr int kSChunkPoints = KM_SORTED_CHUNK_TILES * kLaneTile;   // 1024
constexpr int kSortedUnits = kSChunkPoints / kSortedUnit;          // 4 per chunk
constexpr int kSortedStages = KM_SORTED_STAGES;
#ifndef KM_SUPER_CHUNKS
#define KM_SUPER_CHUNKS 64
#endif
constexpr int kSuperChunks = KM_SUPER_CHUNKS;           // chunks per prune super-box
constexpr int kRowHead = 2;                             // J, count

template <bool LARGE>
struct PCfg {
    static constexpr int kCap = LARGE ? KM_LARGE_CAP : 16;   // refined candidates kept (<= 64)
};
static_assert(KM_LARGE_CAP <= 64, "pruned_body: slot masks are 64-bit");

// Large K: up to kCap refined candidates per chunk, a kCap-slot table T
// (chunks with more go to k_assign_heavy).
template <int D, bool LARGE>
struct PrunedSmem {
    float ring[kSortedStages][D * kSortedUnit];
    uint64_t bar[kSortedStages];
    float4 cand[PCfg<LARGE>::kCap];     // negated fp32 centroid of each candidate slot
    int candk[PCfg<LARGE>::kCap];       // centroid index of each slot (ascending)
    double T[PCfg<LARGE>::kCap * 4];    // per slot {Sx, Sy, Sz, n}
    __device__ __forceinline__ float* ring_at(int s) { return ring[s]; }
};

// Small K: no per-lane columns.  The rare >= 3-candidate chunks add each
// point set into a 16-slot table T with one fixed butterfly per slot present
// in the warp, so a CTA needs ~6.9 KB (3D) and more CTAs (more bytes in
// flight) fit on an SM.
template <int D>
struct PrunedSmem<D, false> {
    float ring[kSortedStages][D * kSortedUnit];
    uint64_t bar[kSortedStages];
    float4 cand[PCfg<false>::kCap];
    int candk[PCfg<false>::kCap];
    double T[PCfg<false>::kCap * 4];   // per slot {Sx, Sy, Sz, n}
    __device__ __forceinline__ float* ring_at(int s) { return ring[s]; }
};

// {k, n} in one double's bits: k in the low word, n in the high word
__device__ __forceinline__ double pack_kn(int k, int n) {
    KM_CHECK(k >= 0 && k < 1024 && n >= 0 && n <= 2048);
    return __hiloint2double(n, k);
}

// A lane's 4 points of one 128-point warp-tile: a = (2L, 2L+1), b = (64+2L, 64+2L+1).
struct LanePts {
    float2 xa, ya, za, xb, yb, zb;
};

// Form D for two points at once (packed f32x2): e_j = x_j + (-c_j), s = e_0 e_0,
// s = fma(e_j, e_j, s) -- reading R6.  cc = negated staged centroid.
template <int D>
__device__ __forceinline__ float2 form_d2(float2 x, float2 y, float2 z, const float4& cc) {
    float2 e0 = __fadd2_rn(x, make_float2(cc.x, cc.x));
    float2 e1 = __fadd2_rn(y, make_float2(cc.y, cc.y));
    float2 sq = __fmul2_rn(e0, e0);
    sq = __ffma2_rn(e1, e1, sq);
    if (D == 3) {
        float2 e2 = __fadd2_rn(z, make_float2(cc.z, cc.z));
        sq = __ffma2_rn(e2, e2, sq);
    }
    return sq;
}

// Exact box bound of one centroid c against the box [lo, hi] (fp64): the min
// and max squared distance from the box to c.
template <int D>
__device__ __forceinline__ void box_bounds(const float (&c)[3], const double (&lo)[3],
                                           const double (&hi)[3], double& dmin2, double& dmax2) {
    dmin2 = 0.0;
    dmax2 = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        const double cj = (double)c[j];
        const double dm = fmax(fmax(lo[j] - cj, cj - hi[j]), 0.0);
        dmin2 += dm * dm;
        const double dx = fmax(fabs(cj - lo[j]), fabs(hi[j] - cj));
        dmax2 += dx * dx;
    }
}

// Exclusion threshold from M = min_k dmax2_k: b is excluded when dmin2_b > thr.
__device__ __forceinline__ double prune_threshold(double M) {
    return (M > 1e37) ? (double)pos_inf() : M * (1.0 + 1e-5) + 0x1p-100;
}

#ifndef KM_BISECTOR
#define KM_BISECTOR 1   // the bisector test on top of the box test
#endif
// Bisector test (the "filtering" test of Kanungo et al.'s kd-tree k-means):
// centroid b can neither win nor tie anywhere in the box if the whole box
// lies on a's side of the bisector of a and b, with margin.  For x in the box
//   ||x - b||^2 - ||x - a||^2 = sum_j (a_j - b_j)(2 x_j - a_j - b_j)
// is linear in x, so its minimum over the box is the sum over axes of the
// smaller of the two corner values (fp64, from fp32 inputs: no cancellation
// of large squares).  b is excluded when that minimum exceeds
// 1e-5 (dmax2_a + dmax2_b) + 2^-100: form D's fp32 results are within
// (d+2) 2^-24 relative (plus a few subnormal ulps) of the exact squares,
// each at most its dmax2 over the box, so D(x, b) > D(x, a) strictly.  a is
// the centroid attaining M = min dmax2 (any centroid would be sound).
// Never when M could overflow fp32 (then nothing is pruned).
template <int D>
__device__ __forceinline__ bool bisector_excludes(const float (&b)[3], const float (&a)[3],
                                                  const double (&lo)[3], const double (&hi)[3],
                                                  double dmax2_b, double M) {
    if (!KM_BISECTOR || M > 1e37) return false;
    double f = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        const double aj = (double)a[j], bj = (double)b[j];
        const double dj = aj - bj;
        f += fmin(dj * (2.0 * lo[j] - aj - bj), dj * (2.0 * hi[j] - aj - bj));
    }
    return f > 1e-5 * (M + dmax2_b) + 0x1p-100;
}

// ---------------------------------------------------------------------------
// small_chunk (sorted path, K <= 16): one warp, one chunk of points
// [base, base + npts) streamed as nunit 256-point units by `fetch` (which waits
// for unit u's TMA stage, loads the lane's points and refills the ring).  Lane
// k tests centroid k against the chunk box (bx: lane j < 2D holds lo/hi of
// axis j): the candidates; then the exact strict-< argmin over them (lowest k
// on ties), form-D distances, and the fused fp64 sums / counts / inertia ->
// the chunk's sparse row [J, count, entries {Sx, Sy, Sz, (k, n)}] (ascending
// k).  Used by k_assign_pruned (one chunk per CTA) and k_persist_iterate.
// ACC: instead of the row, lane 0 adds the chunk's entries to the warp's
// dense table acc[4 k + {0, 1, 2, 3}] = {Sx, Sy, Sz, n}, acc[64] = J (shared
// memory; chunks in the warp's fixed order) -- k_persist_iterate.
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// pruned_body: the points of one chunk segment given its candidates cand[0..nc)
// (negated staged centroids, ascending k in candk): nc == 1 and nc == 2 keep
// the sums in registers; more (up to SLOTS) run the strict-< argmin over the
// list (two candidates per step, ascending, lowest k on ties) and add each
// warp-tile's points into T[slot] = {Sx, Sy, Sz, n} by one fixed butterfly
// per slot present in the warp.  Output: the sparse row (non-empty slots,
// ascending k), or with ACC the warp's dense table.  Shared by the small-K
// and large-K pruned kernels and k_persist_iterate.
// ---------------------------------------------------------------------------
template <int D, int MODE, int SLOTS, bool ACC, class Fetch>
__device__ __forceinline__ void pruned_body(const float4* cand, const int* candk, double* T, int lane,
                                           int K, int nc, int64_t base, int64_t n, int nunit,
                                           int npts, double* __restrict__ row,
                                           int32_t* __restrict__ labels, Fetch&& fetch,
                                           double* acc) {
    const int64_t rem = n - base;
    const int remc = rem < (int64_t)0x7fffffff ? (int)rem : 0x7fffffff;   // valid: offset < remc
    auto cand_at = [&](int j, float4& cc) -> int {   // candidate j: negated centroid, index
        cc = cand[j];
        return candk[j];
    };

    if (nc == 1) {
        // ---- one candidate: labels known, sums in registers (four chains) ----
        float4 cc;
        const int k0 = cand_at(0, cc);
        KM_CHECK(k0 >= 0 && k0 < K);
        double sx[4] = {0.0, 0.0, 0.0, 0.0}, sy[4] = {0.0, 0.0, 0.0, 0.0};
        double sz[4] = {0.0, 0.0, 0.0, 0.0}, Jc[4] = {0.0, 0.0, 0.0, 0.0};
        auto add4 = [&](const LanePts& Q, float2 da, float2 db, int m) {
            // m: bit mask of the valid points (a0, a1, b0, b1)
            if (m & 1) { sx[0] += (double)Q.xa.x; sy[0] += (double)Q.ya.x; sz[0] += (double)Q.za.x; Jc[0] += (double)da.x; }
            if (m & 2) { sx[1] += (double)Q.xa.y; sy[1] += (double)Q.ya.y; sz[1] += (double)Q.za.y; Jc[1] += (double)da.y; }
            if (m & 4) { sx[2] += (double)Q.xb.x; sy[2] += (double)Q.yb.x; sz[2] += (double)Q.zb.x; Jc[2] += (double)db.x; }
            if (m & 8) { sx[3] += (double)Q.xb.y; sy[3] += (double)Q.yb.y; sz[3] += (double)Q.zb.y; Jc[3] += (double)db.y; }
        };
#pragma unroll 1
        for (int u = 0; u < nunit; ++u) {
            LanePts P[kUnitSub];
            fetch(u, P);
#pragma unroll
            for (int h = 0; h < kUnitSub; ++h) {
                const float2 da = form_d2<D>(P[h].xa, P[h].ya, P[h].za, cc);
                const float2 db = form_d2<D>(P[h].xb, P[h].yb, P[h].zb, cc);
                const int64_t pa = base + (int64_t)u * kSortedUnit + h * kLaneTile + 2 * lane;
                const int64_t pb = pa + kWarpTile;
                if (MODE & kModeLabels) {
                    *reinterpret_cast<int2*>(labels + pa) = make_int2(k0, k0);
                    *reinterpret_cast<int2*>(labels + pb) = make_int2(k0, k0);
                }
                if (MODE & kModeReduce) {
                    if ((int64_t)u * kSortedUnit + (h + 1) * kLaneTile <= rem)
                        add4(P[h], da, db, 15);
                    else
                        add4(P[h], da, db, (pa < n ? 1 : 0) | (pa + 1 < n ? 2 : 0) |
                                               (pb < n ? 4 : 0) | (pb + 1 < n ? 8 : 0));
                }
            }
        }
        if (!(MODE & kModeReduce)) return;
        double sxt = (sx[0] + sx[1]) + (sx[2] + sx[3]);
        double syt = (sy[0] + sy[1]) + (sy[2] + sy[3]);
        double szt = (sz[0] + sz[1]) + (sz[2] + sz[3]);
        double J = (Jc[0] + Jc[1]) + (Jc[2] + Jc[3]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sxt += __shfl_xor_sync(0xffffffffu, sxt, o);
            syt += __shfl_xor_sync(0xffffffffu, syt, o);
            szt += __shfl_xor_sync(0xffffffffu, szt, o);
            J += __shfl_xor_sync(0xffffffffu, J, o);
        }
        if (ACC) {
            if (lane == 0) {
                double* a = acc + 4 * k0;
                a[0] += sxt;
                a[1] += syt;
                a[2] += szt;
                a[3] += (double)npts;
                acc[64] += J;
            }
        } else if (lane == 0) {   // sparse row: J, 1 entry {Sx, Sy, Sz, (k, n)}
            row[0] = J;
            row[1] = 1.0;
            reinterpret_cast<double2*>(row + kRowHead)[0] = make_double2(sxt, syt);
            reinterpret_cast<double2*>(row + kRowHead)[1] = make_double2(szt, pack_kn(k0, npts));
        }
        return;
    }

#if KM_TWO_CAND
    if (nc == 2) {
        // ---- two candidates (nearly every multi-candidate chunk at NS): the
        // strict-< argmin of the pair (lowest k on ties: the list ascends in k),
        // sums of both candidates in registers (selects; adding +0.0 leaves a
        // sum unchanged), two chains (a- and b-points) ----
        float4 c0, c1;
        const int k0 = cand_at(0, c0), k1 = cand_at(1, c1);
        double s0[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
        double s1[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
        double Jc[2] = {0.0, 0.0};
        int n1[2] = {0, 0}, nv[2] = {0, 0};
        auto add = [&](int ch, float px, float py, float pz, float d0, float d1) {
            const bool w1 = d1 < d0;
            const double x = (double)px, y = (double)py, z = (double)pz;
#if KM_TWO_CAND_PRED
            if (w1) {   // predicated adds: half the instructions of the selects
                s1[ch][0] += x;
                s1[ch][1] += y;
                if (D == 3) s1[ch][2] += z;
            } else {
                s0[ch][0] += x;
                s0[ch][1] += y;
                if (D == 3) s0[ch][2] += z;
            }
#else
            s0[ch][0] += w1 ? 0.0 : x;
            s0[ch][1] += w1 ? 0.0 : y;
            s1[ch][0] += w1 ? x : 0.0;
            s1[ch][1] += w1 ? y : 0.0;
            if (D == 3) {
                s0[ch][2] += w1 ? 0.0 : z;
                s1[ch][2] += w1 ? z : 0.0;
            }
#endif
            Jc[ch] += (double)(w1 ? d1 : d0);
            n1[ch] += w1 ? 1 : 0;
            nv[ch] += 1;
        };
#pragma unroll 1
        for (int u = 0; u < nunit; ++u) {
            LanePts P[kUnitSub];
            fetch(u, P);
#pragma unroll
            for (int h = 0; h < kUnitSub; ++h) {
                const float2 a0 = form_d2<D>(P[h].xa, P[h].ya, P[h].za, c0);
                const float2 a1 = form_d2<D>(P[h].xa, P[h].ya, P[h].za, c1);
                const float2 b0 = form_d2<D>(P[h].xb, P[h].yb, P[h].zb, c0);
                const float2 b1 = form_d2<D>(P[h].xb, P[h].yb, P[h].zb, c1);
                const int64_t pa = base + (int64_t)u * kSortedUnit + h * kLaneTile + 2 * lane;
                const int64_t pb = pa + kWarpTile;
                if (MODE & kModeLabels) {
                    *reinterpret_cast<int2*>(labels + pa) =
                        make_int2(a1.x < a0.x ? k1 : k0, a1.y < a0.y ? k1 : k0);
                    *reinterpret_cast<int2*>(labels + pb) =
                        make_int2(b1.x < b0.x ? k1 : k0, b1.y < b0.y ? k1 : k0);
                }
                if (MODE & kModeReduce) {
                    // validity from the in-chunk offset (32-bit compares)
                    const int off = u * kSortedUnit + h * kLaneTile + 2 * lane;
                    if (off < remc) add(0, P[h].xa.x, P[h].ya.x, P[h].za.x, a0.x, a1.x);
                    if (off + 1 < remc) add(0, P[h].xa.y, P[h].ya.y, P[h].za.y, a0.y, a1.y);
                    if (off + kWarpTile < remc) add(1, P[h].xb.x, P[h].yb.x, P[h].zb.x, b0.x, b1.x);
                    if (off + kWarpTile + 1 < remc)
                        add(1, P[h].xb.y, P[h].yb.y, P[h].zb.y, b0.y, b1.y);
                }
            }
        }
        if (!(MODE & kModeReduce)) return;
        double v[7] = {s0[0][0] + s0[1][0], s0[0][1] + s0[1][1], s0[0][2] + s0[1][2],
                       s1[0][0] + s1[1][0], s1[0][1] + s1[1][1], s1[0][2] + s1[1][2],
                       Jc[0] + Jc[1]};
        int c1n = n1[0] + n1[1], cvn = nv[0] + nv[1];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
            for (int q = 0; q < 7; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
            c1n += __shfl_xor_sync(0xffffffffu, c1n, o);
            cvn += __shfl_xor_sync(0xffffffffu, cvn, o);
        }
        if (ACC) {
            if (lane == 0) {
                double* a = acc + 4 * k0;
                a[0] += v[0];
                a[1] += v[1];
                a[2] += v[2];
                a[3] += (double)(cvn - c1n);
                double* b = acc + 4 * k1;
                b[0] += v[3];
                b[1] += v[4];
                b[2] += v[5];
                b[3] += (double)c1n;
                acc[64] += v[6];
            }
        } else if (lane == 0) {   // sparse row: J, 2 entries (ascending k)
            row[0] = v[6];
            row[1] = 2.0;
            double2* e = reinterpret_cast<double2*>(row + kRowHead);
            e[0] = make_double2(v[0], v[1]);
            e[1] = make_double2(v[2], pack_kn(k0, cvn - c1n));
            e[2] = make_double2(v[3], v[4]);
            e[3] = make_double2(v[5], pack_kn(k1, c1n));
        }
        return;
    }
#endif

    // ---- several candidates ----
    const int ncand = nc;
    // >= 3 candidates: one pass over the TMA ring; the points of a
    // warp-tile are added to T[slot] by one fixed butterfly per slot
    // present in the warp, counts by ballot
    for (int q = lane; q < 4 * ncand; q += 32) T[q] = 0.0;
    __syncwarp();
    double J = 0.0;
    // the 4 points of a lane (a0, a1, b0, b1) at once: per slot present in
    // the warp, each lane sums its points of that slot in that order, then
    // one fixed butterfly over the lanes; counts by ballot
    // the NP points of a lane at once (a warp-tile: 4 -- a whole TMA unit, 8,
    // measured no faster): per slot present in the warp, each lane sums its
    // points of that slot in point order, then one fixed butterfly over the lanes
    auto agg = [&](auto np_tag, const bool* v, const int* sl, const float* px, const float* py,
                   const float* pz) {
        constexpr int NP = decltype(np_tag)::value;
        unsigned long long mine_bits = 0ull;
#pragma unroll
        for (int i = 0; i < NP; ++i)
            if (v[i]) mine_bits |= 1ull << sl[i];
        unsigned long long pres = __reduce_or_sync(0xffffffffu, (unsigned)mine_bits);
        if (SLOTS > 32)
            pres |= (unsigned long long)__reduce_or_sync(0xffffffffu, (unsigned)(mine_bits >> 32))
                    << 32;
        while (pres) {
            const int q = __ffsll((long long)pres) - 1;
            pres &= pres - 1;
            double sx = 0.0, sy = 0.0, sz = 0.0;
            unsigned c = 0u;
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                if (v[i] && sl[i] == q) {   // predicated adds (no selects)
                    sx += (double)px[i];
                    sy += (double)py[i];
                    sz += (double)pz[i];
                    ++c;
                }
            }
#if KM_AGG_TRANSPOSE
            // (Sx, Sy, Sz, n) over the 32 lanes by a transposing butterfly:
            // the offset-16 step trades half the values (each half-warp keeps
            // a pair), the offset-8 step half again, then three plain steps
            // on one value -- 7 fp64 shuffles and 6 adds instead of 15 and 15
            // plus a REDUX; lane 8 j ends with value j (fixed order).
            const bool up16 = lane & 16, up8 = lane & 8;
            double k0 = up16 ? sz : sx, k1 = up16 ? (double)c : sy;
            const double o0 = up16 ? sx : sz, o1 = up16 ? sy : (double)c;
            k0 += __shfl_xor_sync(0xffffffffu, o0, 16);
            k1 += __shfl_xor_sync(0xffffffffu, o1, 16);
            double kv = up8 ? k1 : k0;
            kv += __shfl_xor_sync(0xffffffffu, up8 ? k0 : k1, 8);
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) kv += __shfl_xor_sync(0xffffffffu, kv, o);
            if ((lane & 7) == 0) T[4 * q + (lane >> 3)] += kv;
#else
            const unsigned cnt = __reduce_add_sync(0xffffffffu, c);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                sx += __shfl_xor_sync(0xffffffffu, sx, o);
                sy += __shfl_xor_sync(0xffffffffu, sy, o);
                if (D == 3) sz += __shfl_xor_sync(0xffffffffu, sz, o);
            }
            if (lane == 0) {
                double* t = T + 4 * q;
                t[0] += sx;
                t[1] += sy;
                t[2] += sz;
                t[3] += (double)cnt;
            }
#endif
        }
        __syncwarp();
    };
    // large K: one slot aggregation per 256-point TMA unit (8 points per lane;
    // fewer butterflies: C5 assign 0.276 -> 0.265 ms); small K (where >= 3
    // candidates are rare) per warp-tile (the unit form measured slower there)
    constexpr bool kUnitAgg = KM_AGG_UNIT && SLOTS > 16;
#pragma unroll 1
    for (int u = 0; u < nunit; ++u) {
        LanePts P[kUnitSub];
        fetch(u, P);
        bool uv[4 * kUnitSub];   // the unit's points of this lane: valid, slot
        int us[4 * kUnitSub];
#pragma unroll
        for (int h = 0; h < kUnitSub; ++h) {
            const int off = u * kSortedUnit + h * kLaneTile + 2 * lane;   // in-chunk index
            const int64_t pa = base + off, pb = pa + kWarpTile;
            float4 cc;
            cand_at(0, cc);
            float2 ba = form_d2<D>(P[h].xa, P[h].ya, P[h].za, cc);
            float2 bb = form_d2<D>(P[h].xb, P[h].yb, P[h].zb, cc);
            int s0 = 0, s1 = 0, s2 = 0, s3 = 0;
            int j = 1;
#pragma unroll 1
            for (; j + 1 < ncand; j += 2) {   // two candidates per step, ascending
                float4 c2;
                cand_at(j, cc);
                cand_at(j + 1, c2);
                const float2 da = form_d2<D>(P[h].xa, P[h].ya, P[h].za, cc);
                const float2 db = form_d2<D>(P[h].xb, P[h].yb, P[h].zb, cc);
                const float2 ea = form_d2<D>(P[h].xa, P[h].ya, P[h].za, c2);
                const float2 eb = form_d2<D>(P[h].xb, P[h].yb, P[h].zb, c2);
                if (da.x < ba.x) { ba.x = da.x; s0 = j; }
                if (da.y < ba.y) { ba.y = da.y; s1 = j; }
                if (db.x < bb.x) { bb.x = db.x; s2 = j; }
                if (db.y < bb.y) { bb.y = db.y; s3 = j; }
                if (ea.x < ba.x) { ba.x = ea.x; s0 = j + 1; }
                if (ea.y < ba.y) { ba.y = ea.y; s1 = j + 1; }
                if (eb.x < bb.x) { bb.x = eb.x; s2 = j + 1; }
                if (eb.y < bb.y) { bb.y = eb.y; s3 = j + 1; }
            }
            if (j < ncand) {
                cand_at(j, cc);
                const float2 da = form_d2<D>(P[h].xa, P[h].ya, P[h].za, cc);
                const float2 db = form_d2<D>(P[h].xb, P[h].yb, P[h].zb, cc);
                if (da.x < ba.x) { ba.x = da.x; s0 = j; }
                if (da.y < ba.y) { ba.y = da.y; s1 = j; }
                if (db.x < bb.x) { bb.x = db.x; s2 = j; }
                if (db.y < bb.y) { bb.y = db.y; s3 = j; }
            }
            if (MODE & kModeLabels) {
                float4 t;
                *reinterpret_cast<int2*>(labels + pa) = make_int2(cand_at(s0, t), cand_at(s1, t));
                *reinterpret_cast<int2*>(labels + pb) = make_int2(cand_at(s2, t), cand_at(s3, t));
            }
            if (MODE & kModeReduce) {
                // validity from the in-chunk offset (32-bit compares; every
                // point of all but the shard's last chunk is valid)
                const bool v0 = off < remc, v1 = off + 1 < remc;
                const bool v2 = off + kWarpTile < remc, v3 = off + kWarpTile + 1 < remc;
                if (v0) J += (double)ba.x;
                if (v1) J += (double)ba.y;
                if (v2) J += (double)bb.x;
                if (v3) J += (double)bb.y;
                uv[4 * h + 0] = v0;
                uv[4 * h + 1] = v1;
                uv[4 * h + 2] = v2;
                uv[4 * h + 3] = v3;
                us[4 * h + 0] = s0;
                us[4 * h + 1] = s1;
                us[4 * h + 2] = s2;
                us[4 * h + 3] = s3;
                if constexpr (!kUnitAgg) {
                    const float xx[4] = {P[h].xa.x, P[h].xa.y, P[h].xb.x, P[h].xb.y};
                    const float yy[4] = {P[h].ya.x, P[h].ya.y, P[h].yb.x, P[h].yb.y};
                    const float zz[4] = {P[h].za.x, P[h].za.y, P[h].zb.x, P[h].zb.y};
                    agg(std::integral_constant<int, 4>{}, uv + 4 * h, us + 4 * h, xx, yy, zz);
                }
            }
        }
        if constexpr (kUnitAgg && (MODE & kModeReduce)) {   // the whole unit's points at once
            float xx[4 * kUnitSub], yy[4 * kUnitSub], zz[4 * kUnitSub];
#pragma unroll
            for (int h = 0; h < kUnitSub; ++h) {
                xx[4 * h + 0] = P[h].xa.x; xx[4 * h + 1] = P[h].xa.y;
                xx[4 * h + 2] = P[h].xb.x; xx[4 * h + 3] = P[h].xb.y;
                yy[4 * h + 0] = P[h].ya.x; yy[4 * h + 1] = P[h].ya.y;
                yy[4 * h + 2] = P[h].yb.x; yy[4 * h + 3] = P[h].yb.y;
                zz[4 * h + 0] = P[h].za.x; zz[4 * h + 1] = P[h].za.y;
                zz[4 * h + 2] = P[h].zb.x; zz[4 * h + 3] = P[h].zb.y;
            }
            agg(std::integral_constant<int, 4 * kUnitSub>{}, uv, us, xx, yy, zz);
        }
    }
    if (!(MODE & kModeReduce)) return;
    if constexpr (ACC) {   // slots in ascending k order
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) J += __shfl_xor_sync(0xffffffffu, J, o);
        if (lane == 0) {
            for (int sl = 0; sl < ncand; ++sl) {
                double* a = acc + 4 * candk[sl];
                const double* t = T + 4 * sl;
                a[0] += t[0];
                a[1] += t[1];
                a[2] += t[2];
                a[3] += t[3];
            }
            acc[64] += J;
        }
    } else {
        // the non-empty slots, compacted in ascending slot (= ascending k) order
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) J += __shfl_xor_sync(0xffffffffu, J, o);
        int outc = 0;
        for (int s0 = 0; s0 < ncand; s0 += 32) {
            const int sl = s0 + lane;
            const bool nz = sl < ncand && T[4 * sl + 3] > 0.0;
            const unsigned m = __ballot_sync(0xffffffffu, nz);
            if (nz) {
                const int o = outc + __popc(m & ((1u << lane) - 1u));
                const double* t = T + 4 * sl;
                double2* e = reinterpret_cast<double2*>(row + kRowHead) + 2 * o;
                e[0] = make_double2(t[0], t[1]);
                e[1] = make_double2(t[2], pack_kn(candk[sl], (int)t[3]));
            }
            outc += __popc(m);
        }
        if (lane == 0) {
            row[0] = J;
            row[1] = (double)outc;
        }
    }
}

template <int D, int MODE, bool ACC = false, class Fetch>
__device__ __forceinline__ void small_chunk(PrunedSmem<D, false>& S, int lane, int K, float4 cl,
                                            float bx, int64_t base, int64_t n, int nunit,
                                            int npts, double* __restrict__ row,
                                            int32_t* __restrict__ labels, int* cand_slot,
                                            Fetch&& fetch, double* acc = nullptr) {
    double lo[3], hi[3];
#pragma unroll
    for (int j = 0; j < D; ++j) {
        lo[j] = (double)__shfl_sync(0xffffffffu, bx, j);
        hi[j] = (double)__shfl_sync(0xffffffffu, bx, D + j);
    }
    int nc = 0;   // candidates
    {
        float c[3] = {0.f, 0.f, 0.f};
        double dmin2 = 0.0, dmax2 = 0.0;
        const bool is_k = lane < K;
        if (is_k) {
            c[0] = -cl.x;
            c[1] = -cl.y;
            c[2] = -cl.z;
            box_bounds<D>(c, lo, hi, dmin2, dmax2);
        }
        double M = is_k ? dmax2 : (double)pos_inf();
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) M = fmin(M, __shfl_xor_sync(0xffffffffu, M, o));
        // a = the centroid attaining M (lowest such lane)
        const int al = __ffs(__ballot_sync(0xffffffffu, is_k && dmax2 == M)) - 1;
        float a[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) a[j] = __shfl_sync(0xffffffffu, c[j], al & 31);
        const bool cand = is_k && dmin2 <= prune_threshold(M) &&
                          !bisector_excludes<D>(c, a, lo, hi, dmax2, M);
        const unsigned mask = __ballot_sync(0xffffffffu, cand);
        nc = __popc(mask);
        if (cand) {
            const int sl = __popc(mask & ((1u << lane) - 1u));
            S.cand[sl] = make_float4(-c[0], -c[1], D == 3 ? -c[2] : 0.0f, 0.0f);
            S.candk[sl] = lane;
        }
    }
    KM_CHECK(nc >= 1 && nc <= K);
    if (lane == 0 && cand_slot) *cand_slot = nc;
    __syncwarp();
    pruned_body<D, MODE, PCfg<false>::kCap, ACC>(S.cand, S.candk, S.T, lane, K, nc, base, n,
                                                 nunit, npts, row, labels, fetch, acc);
}

// Small K: resident CTAs per SM the register budget is cut for (more CTAs =
// more bytes in flight; measured: 28 best in 3D, 32 -- the per-SM block limit --
// in 2D; a 64-register 3D kernel loses more to its two-candidate path)
#ifndef KM_PRUNED_MINB
#define KM_PRUNED_MINB (D == 2 ? 32 : 28)
#endif
#ifndef KM_PRUNED_MINB_LARGE
#define KM_PRUNED_MINB_LARGE 22   // 9.5 KB of shared memory per CTA: 22 fit an SM
#endif
template <int D, int MODE, bool LARGE, int CHT = KM_SORTED_CHUNK_TILES>
__global__ void __launch_bounds__(32, LARGE ? KM_PRUNED_MINB_LARGE : KM_PRUNED_MINB)
k_assign_pruned(const float* __restrict__ X, int64_t n, int K,
                const float4* __restrict__ cneg_buf, const DevState* __restrict__ st,
                int mu_sel, int ignore_done, const float* __restrict__ cbox,
                const int* __restrict__ slist, const float4* __restrict__ scl,
                const int* __restrict__ scount,
                double* __restrict__ rows, int row_stride, int32_t* __restrict__ labels,
                int* __restrict__ cand_count, int* __restrict__ heavy,
                int* __restrict__ heavy_count, int64_t keep_n) {
    using C = PCfg<LARGE>;
    // Prologue before pdl_wait() touches only what no predecessor writes: the
    // chunk box and the points (the TMA ring is filled here, so with PDL the
    // first units stream in while the previous update finishes).
    const int lane = threadIdx.x;
    // large K: chunks in reverse curve order -- the far end of the curve
    // (outlier sites) makes the widest super boxes and the longest chunk
    // prologues, which then start first instead of stretching the tail
    const int chunk = (LARGE && KM_LARGE_REVERSE) ? (int)gridDim.x - 1 - (int)blockIdx.x
                                                  : (int)blockIdx.x;
    const float4* cneg = cneg_buf + (size_t)mu_sel * K;   // -fl32(mu^t) (or mu^{t-1})
    const float bx = (lane < 2 * D) ? __ldg(&cbox[(size_t)chunk * 2 * D + lane]) : 0.0f;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PrunedSmem<D, LARGE>& S = *reinterpret_cast<PrunedSmem<D, LARGE>*>(smem_raw);
    constexpr int kUnitFloats = D * kSortedUnit;
    constexpr unsigned kUnitBytes = kUnitFloats * 4;
    constexpr int SS = kSortedStages;
    // chunk of CHT warp-tiles (1024 points by default; 2048 for large small-K
    // shards, chosen at create -- the large-K kernels assume 1024)
    constexpr int CHP = CHT * kLaneTile, CHU = CHP / kSortedUnit;
    static_assert(!LARGE || CHP == kSChunkPoints, "large K: 1024-point chunks");
    const int64_t base = (int64_t)chunk * CHP;
    const int64_t rem = n - base;
    const int64_t nu64 = (rem + kSortedUnit - 1) / kSortedUnit;
    const int nunit = nu64 < CHU ? (int)nu64 : CHU;
    const int npts = rem < CHP ? (int)rem : CHP;
    const float* src = X + (base >> 6) * (D * kWarpTile);

    // point stream: units 0..nunit-1 through the TMA ring (unit q in stage q % SS).
    // Small K: points below keep_n stay resident in L2 across iterations
    // (evict_last), the rest stream from HBM (evict_first).
    unsigned issued = 0;   // lane 0
    const bool keep = !LARGE && base < keep_n;
    const uint64_t pol = LARGE ? 0ull : (keep ? l2_policy_evict_last() : l2_policy_evict_first());
    auto issue_upto = [&](unsigned limit) {
        if (lane != 0) return;
        while (issued < limit && (int)issued < nunit) {
            const int s = issued % SS;
            mbar_expect_tx(&S.bar[s], kUnitBytes);
            if (LARGE)
                bulk_g2s(S.ring_at(s), src + (int64_t)issued * kUnitFloats, kUnitBytes, &S.bar[s],
                         false);
            else
                bulk_g2s_pol(S.ring_at(s), src + (int64_t)issued * kUnitFloats, kUnitBytes,
                             &S.bar[s], pol);
            ++issued;
        }
    };
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < SS; ++s) mbar_init(&S.bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    issue_upto(SS);
#if KM_PDL_ASSIGN_TRIGGER
    pdl_trigger();
#endif
    pdl_wait();   // the centroids, the stop flag and (large K) the super lists are ready
    const float4 cl = (!LARGE && lane < K) ? __ldg(&cneg[lane]) : make_float4(0.f, 0.f, 0.f, 0.f);
    const int sup_count = LARGE ? __ldg(&scount[chunk / kSuperChunks]) : 0;
    const int done_flag = ignore_done ? 0 : *(volatile const int*)&st->done;
    if (done_flag) {   // stop rule already met: drain the issued copies, then leave
        for (unsigned q = 0; q < (unsigned)min(SS, nunit); ++q) mbar_wait(&S.bar[q % SS], 0u);
        return;
    }
    // a lane's points of unit q (waits for its stage, then refills the ring)
    auto fetch = [&](unsigned q, LanePts (&P)[kUnitSub]) {
        const int s = q % SS;
        mbar_wait(&S.bar[s], (q / SS) & 1u);
#pragma unroll
        for (int h = 0; h < kUnitSub; ++h) {
            const float* rg = S.ring_at(s) + h * (D * kLaneTile);
            const float* rb = rg + D * kWarpTile;
            P[h].xa = reinterpret_cast<const float2*>(rg)[lane];
            P[h].ya = reinterpret_cast<const float2*>(rg + kWarpTile)[lane];
            P[h].za = (D == 3) ? reinterpret_cast<const float2*>(rg + 2 * kWarpTile)[lane]
                               : make_float2(0.f, 0.f);
            P[h].xb = reinterpret_cast<const float2*>(rb)[lane];
            P[h].yb = reinterpret_cast<const float2*>(rb + kWarpTile)[lane];
            P[h].zb = (D == 3) ? reinterpret_cast<const float2*>(rb + 2 * kWarpTile)[lane]
                               : make_float2(0.f, 0.f);
        }
        __syncwarp();
        issue_upto(q + SS);
    };
    if constexpr (!LARGE) {
        small_chunk<D, MODE>(S, lane, K, cl, bx, base, n, nunit, npts,
                             rows + (size_t)chunk * row_stride, labels,
                             cand_count ? cand_count + chunk : nullptr, fetch);
        return;
    } else {

        // ---- candidates of this chunk ----
        double lo[3], hi[3];
#pragma unroll
        for (int j = 0; j < D; ++j) {
            lo[j] = (double)__shfl_sync(0xffffffffu, bx, j);
            hi[j] = (double)__shfl_sync(0xffffffffu, bx, D + j);
        }
        auto bounds = [&](const float (&c)[3], double& dmin2, double& dmax2) {
            dmin2 = 0.0;
            dmax2 = 0.0;
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const double cj = (double)c[j];
                const double dm = fmax(fmax(lo[j] - cj, cj - hi[j]), 0.0);
                dmin2 += dm * dm;
                const double dx = fmax(fabs(cj - lo[j]), fabs(hi[j] - cj));
                dmax2 += dx * dx;
            }
        };
        auto warp_min = [&](double v) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
            return v;
        };
        auto threshold = [&](double M) {
            return (M > 1e37) ? (double)pos_inf() : M * (1.0 + 1e-5) + 0x1p-100;
        };
        int nc = 0;          // refined candidates
        bool big = false;    // candidates = the unrefined super list (global)
        const int* glist = nullptr;
        const float4* gcl = nullptr;   // the super list's staged centroids, k in .w
        int gcount = 0;
        {
            const int sup = chunk / kSuperChunks;
            glist = slist + (size_t)sup * K;
            gcl = scl + (size_t)sup * K;
            gcount = sup_count;
            double Ml = (double)pos_inf();   // this lane's min dmax2 and its position
            int Mil = 0x7fffffff;
            for (int i = lane; i < gcount; i += 32) {
                const float4 v = __ldg(&gcl[i]);
                const float c[3] = {-v.x, -v.y, -v.z};
                double a, b;
                bounds(c, a, b);
                if (b < Ml) {
                    Ml = b;
                    Mil = i;
                }
            }
            const double M = warp_min(Ml);
            int Mi = (Ml == M) ? Mil : 0x7fffffff;   // the lowest position attaining M
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) Mi = min(Mi, __shfl_xor_sync(0xffffffffu, Mi, o));
            const float4 av = __ldg(&gcl[Mi]);   // a = the centroid attaining M
            const float ca[3] = {-av.x, -av.y, -av.z};
            const double thr = threshold(M);
            for (int i0 = 0; i0 < gcount; i0 += 32) {
                const int i = i0 + lane;
                float c[3] = {0.f, 0.f, 0.f};
                int k = 0;
                bool cand = false;
                if (i < gcount) {
                    const float4 v = __ldg(&gcl[i]);
                    k = __float_as_int(v.w);
                    c[0] = -v.x;
                    c[1] = -v.y;
                    c[2] = -v.z;
                    double a, b;
                    bounds(c, a, b);
                    cand = a <= thr && !bisector_excludes<D>(c, ca, lo, hi, b, M);
                }
                const unsigned mask = __ballot_sync(0xffffffffu, cand);
                const int sl = nc + __popc(mask & ((1u << lane) - 1u));
                if (cand && sl < C::kCap) {
                    S.cand[sl] = make_float4(-c[0], -c[1], D == 3 ? -c[2] : 0.0f, 0.0f);
                    S.candk[sl] = k;
                }
                nc += __popc(mask);
            }
            big = nc > C::kCap;
        }
        KM_CHECK(nc >= 1 && (LARGE || nc <= K) && (!LARGE || nc <= gcount));
        if (lane == 0 && cand_count) cand_count[chunk] = nc;
        if (LARGE && big) {
            // more than kCap candidates: k_assign_heavy takes this chunk with a whole
            // block.  Drain the units already in flight, then leave.
            if (lane == 0) {
                const int h = atomicAdd(heavy_count, 1);
                KM_CHECK(h >= 0 && (int64_t)h * CHP < n);   // h < n_chunks
                heavy[h] = chunk;
            }
            const unsigned nq = __shfl_sync(0xffffffffu, issued, 0);
            for (unsigned q = 0; q < nq; ++q) mbar_wait(&S.bar[q % SS], (q / SS) & 1u);
            return;
        }
        __syncwarp();
        pruned_body<D, MODE, C::kCap, false>(S.cand, S.candk, S.T, lane, K, nc, base, n, nunit,
                                             npts, rows + (size_t)chunk * row_stride, labels,
                                             fetch, nullptr);
    }   // LARGE
}

// ---------------------------------------------------------------------------
// k_assign_heavy (large K): the chunks with more than kCap refined candidates
// (boxes spanning sparse or far regions), one 8-warp block each.  Warp w
// takes the chunk's 128-point sub-tile w on its own -- no block barrier until
// the row is assembled:
//   * its points (LDG) and their box; the super-box list refined against
//     that box (the same exact test as k_assign_pruned: the tile's minimiser
//     of dmax2 is in the super list, so the tile's M and exclusions are exact);
//   * the strict-< argmin over the tile list (ascending k: lowest k on ties);
//   * the tile's sums into a 64-slot table by one fixed butterfly per slot
//     present in the warp (slots in windows of 64 when the list is longer),
//     compacted to (k, Sx, Sy, Sz, n) entries in ascending k.
// After one barrier warp 0 writes the chunk's row: the 8 tiles' entries in
// tile order (a k may appear once per tile; k_merge_sparse adds entries in
// row order) and J summed in tile order.
// ---------------------------------------------------------------------------
constexpr int kHeavyWarps = kSChunkPoints / kLaneTile;   // 8 sub-tiles of 128 points
constexpr int kHeavySlots = 64;                          // slot window of the tile table

// row capacity (entries) of the large-K path: pruned rows hold <= kCap
// entries, heavy rows up to 8 tiles x min(K, 128) (a k once per tile)
__host__ __device__ constexpr int large_row_entries(int K) {
    return K < 128 ? (8 * K < kSChunkPoints ? 8 * K : kSChunkPoints) : kSChunkPoints;
}

constexpr int kHeavySplit = 64;   // tile lists longer than this are walked by all 8 warps

template <int D>
struct HeavySmem {
    double4 ent[kHeavyWarps][kLaneTile];      // per warp: {Sx, Sy, Sz, (k, n)} entries
    float2 part[kHeavyWarps][kHeavyWarps][4][32];   // split walks: (distance, slot) per
                                                    // tile, warp, point, lane
    float2 pts[kHeavyWarps][6][32];           // each tile's points (xa ya za xb yb zb per lane)
    double wJ[kHeavyWarps];
    int went[kHeavyWarps];
    int wnt[kHeavyWarps];
    // followed by the super list's staged centroids float4 cl[K] and the tile
    // lists unsigned short list[kHeavyWarps][K] (super-list positions)
};

// Strict-< argmin of a lane's 4 points over list positions [t0, t1) of a
// tile list (slots ascending), two candidates per step (independent chains;
// the updates stay in ascending slot order).  t0 < t1.
template <int D>
__device__ __forceinline__ void argmin_walk(const unsigned short* list, const float4* cl, int t0,
                                            int t1, float2 xa, float2 ya, float2 za, float2 xb,
                                            float2 yb, float2 zb, float (&best)[4], int (&sl)[4]) {
    {
        const float4 cc = cl[list[t0]];
        const float2 da = form_d2<D>(xa, ya, za, cc), db = form_d2<D>(xb, yb, zb, cc);
        best[0] = da.x; best[1] = da.y; best[2] = db.x; best[3] = db.y;
        sl[0] = sl[1] = sl[2] = sl[3] = t0;
    }
    int t = t0 + 1;
    for (; t + 1 < t1; t += 2) {
        const float4 c0 = cl[list[t]], c1 = cl[list[t + 1]];
        const float2 da = form_d2<D>(xa, ya, za, c0), db = form_d2<D>(xb, yb, zb, c0);
        const float2 ea = form_d2<D>(xa, ya, za, c1), eb = form_d2<D>(xb, yb, zb, c1);
        if (da.x < best[0]) { best[0] = da.x; sl[0] = t; }
        if (da.y < best[1]) { best[1] = da.y; sl[1] = t; }
        if (db.x < best[2]) { best[2] = db.x; sl[2] = t; }
        if (db.y < best[3]) { best[3] = db.y; sl[3] = t; }
        if (ea.x < best[0]) { best[0] = ea.x; sl[0] = t + 1; }
        if (ea.y < best[1]) { best[1] = ea.y; sl[1] = t + 1; }
        if (eb.x < best[2]) { best[2] = eb.x; sl[2] = t + 1; }
        if (eb.y < best[3]) { best[3] = eb.y; sl[3] = t + 1; }
    }
    if (t < t1) {
        const float4 cc = cl[list[t]];
        const float2 da = form_d2<D>(xa, ya, za, cc), db = form_d2<D>(xb, yb, zb, cc);
        if (da.x < best[0]) { best[0] = da.x; sl[0] = t; }
        if (da.y < best[1]) { best[1] = da.y; sl[1] = t; }
        if (db.x < best[2]) { best[2] = db.x; sl[2] = t; }
        if (db.y < best[3]) { best[3] = db.y; sl[3] = t; }
    }
}

template <int D, int MODE>
__global__ void __launch_bounds__(kHeavyWarps * 32)
k_assign_heavy(const float* __restrict__ X, int64_t n, int K, const float4* __restrict__ cneg_buf,
               const DevState* __restrict__ st, int mu_sel, int ignore_done,
               const float* __restrict__ cbox, const int* __restrict__ slist,
               const float4* __restrict__ scl,
               const int* __restrict__ scount, const int* __restrict__ heavy,
               const int* __restrict__ heavy_count, double* __restrict__ rows, int row_stride,
               int32_t* __restrict__ labels) {
    (void)cbox;
    if (!ignore_done && st->done) return;
    static_assert(kSChunkPoints == kHeavyWarps * kLaneTile, "one 128-point sub-tile per warp");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    HeavySmem<D>& S = *reinterpret_cast<HeavySmem<D>*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float4* cl = reinterpret_cast<float4*>(smem_raw + sizeof(HeavySmem<D>));   // [K]
    unsigned short* my = reinterpret_cast<unsigned short*>(cl + K) + (size_t)warp * K;
    (void)cneg_buf;   // the super lists carry the staged centroids (scl)
    (void)mu_sel;
    const int nh = *heavy_count;
    for (int h = blockIdx.x; h < nh; h += gridDim.x) {
        const int chunk = heavy[h];
#if KM_HEAVY_PROF
        const unsigned long long tp0 = (unsigned long long)global_ns();
#endif
        const int* list = slist + (size_t)(chunk / kSuperChunks) * K;
        const int gc = scount[chunk / kSuperChunks];
        // ---- this warp's sub-tile: points (loads issued before the staging) ----
        const int64_t pa = (int64_t)chunk * kSChunkPoints + warp * kLaneTile + 2 * lane;
        const int64_t pb = pa + kWarpTile;
        const float2 xa = ld_stream2(tile_coord<D>(X, pa, 0));
        const float2 ya = ld_stream2(tile_coord<D>(X, pa, 1));
        const float2 za = (D == 3) ? ld_stream2(tile_coord<D>(X, pa, 2)) : make_float2(0.f, 0.f);
        const float2 xb = ld_stream2(tile_coord<D>(X, pb, 0));
        const float2 yb = ld_stream2(tile_coord<D>(X, pb, 1));
        const float2 zb = (D == 3) ? ld_stream2(tile_coord<D>(X, pb, 2)) : make_float2(0.f, 0.f);
        const float4* lcl = scl + (size_t)(chunk / kSuperChunks) * K;
        for (int i = tid; i < gc; i += blockDim.x) cl[i] = __ldg(&lcl[i]);
        // the tile's points for the split walks of the other warps
        S.pts[warp][0][lane] = xa;
        S.pts[warp][1][lane] = ya;
        S.pts[warp][2][lane] = za;
        S.pts[warp][3][lane] = xb;
        S.pts[warp][4][lane] = yb;
        S.pts[warp][5][lane] = zb;
        __syncthreads();   // the super list's centroids (and the tiles' points) are staged
#if KM_HEAVY_PROF
        const unsigned long long tp1 = (unsigned long long)global_ns();
#endif
        const bool v[4] = {pa < n, pa + 1 < n, pb < n, pb + 1 < n};
        const float px[4] = {xa.x, xa.y, xb.x, xb.y}, py[4] = {ya.x, ya.y, yb.x, yb.y};
        const float pz[4] = {za.x, za.y, zb.x, zb.y};
        double tlo[3] = {0, 0, 0}, thi[3] = {0, 0, 0};
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const float* pj = j == 0 ? px : (j == 1 ? py : pz);
            float l_ = pos_inf(), h_ = -pos_inf();
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (v[i]) {
                    l_ = fminf(l_, pj[i]);
                    h_ = fmaxf(h_, pj[i]);
                }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                l_ = fminf(l_, __shfl_xor_sync(0xffffffffu, l_, o));
                h_ = fmaxf(h_, __shfl_xor_sync(0xffffffffu, h_, o));
            }
            tlo[j] = (double)l_;
            thi[j] = (double)h_;
        }
        const bool any_valid = tlo[0] <= thi[0];   // false for an all-padding tile
        // ---- the super list refined against the tile box (ascending k) ----
        int nt = 0;
        if (any_valid) {
            double Ml = (double)pos_inf();   // this lane's min dmax2 and its position
            int Mil = 0x7fffffff;
#pragma unroll kRefineUnroll
            for (int i = lane; i < gc; i += 32) {
                const float4 c4 = cl[i];
                const float c[3] = {-c4.x, -c4.y, -c4.z};
                double a, b;
                box_bounds<D>(c, tlo, thi, a, b);
                if (b < Ml) {
                    Ml = b;
                    Mil = i;
                }
            }
            double M = Ml;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) M = fmin(M, __shfl_xor_sync(0xffffffffu, M, o));
            int Mi = (Ml == M) ? Mil : 0x7fffffff;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) Mi = min(Mi, __shfl_xor_sync(0xffffffffu, Mi, o));
            const float4 a4 = cl[Mi];   // a = the centroid attaining M
            const float ca[3] = {-a4.x, -a4.y, -a4.z};
            const double thr = prune_threshold(M);
#pragma unroll kRefineUnroll
            for (int i0 = 0; i0 < gc; i0 += 32) {
                const int i = i0 + lane;
                bool cand = false;
                if (i < gc) {
                    const float4 c4 = cl[i];
                    const float c[3] = {-c4.x, -c4.y, -c4.z};
                    double a, b;
                    box_bounds<D>(c, tlo, thi, a, b);
                    cand = a <= thr && !bisector_excludes<D>(c, ca, tlo, thi, b, M);
                }
                const unsigned m = __ballot_sync(0xffffffffu, cand);
                if (cand) my[nt + __popc(m & ((1u << lane) - 1u))] = (unsigned short)i;
                nt += __popc(m);
            }
        } else {
            if (lane == 0) my[0] = 0;
            nt = 1;
        }
        KM_CHECK(nt >= 1 && nt <= gc);
        __syncwarp();
        // ---- exact argmin over the tile list (ascending k; strict <) ----
        // A long list (a tile spanning a sparse gap, e.g. to a far site) is
        // walked by all 8 warps, each over a contiguous eighth; the partial
        // (distance, slot) pairs are combined in ascending eighths with
        // strict <, which is the serial walk's result (lowest slot on ties).
        if (lane == 0) S.wnt[warp] = nt;
        __syncthreads();   // every tile's list length
#if KM_HEAVY_PROF
        const unsigned long long tp2 = (unsigned long long)global_ns();
#endif
        float best[4];
        int sl[4];
        if (nt <= kHeavySplit) argmin_walk<D>(my, cl, 0, nt, xa, ya, za, xb, yb, zb, best, sl);
        // every long tile in one round: warp w walks the w-th eighth of each
        // (the tile's points from shared memory), one barrier, then the tile's
        // own warp combines the eighths in ascending order (strict <)
        bool any_long = false;
        for (int T = 0; T < kHeavyWarps; ++T) {   // block-uniform
            const int ntT = S.wnt[T];
            if (ntT <= kHeavySplit) continue;
            any_long = true;
            const float2* tp = &S.pts[T][0][0];
            const unsigned short* listT = my - (size_t)warp * K + (size_t)T * K;
            const int t0 = (int)((int64_t)ntT * warp / kHeavyWarps);
            const int t1 = (int)((int64_t)ntT * (warp + 1) / kHeavyWarps);
            float pb_[4];
            int ps_[4];
            argmin_walk<D>(listT, cl, t0, t1, tp[0 * 32 + lane], tp[1 * 32 + lane],
                           tp[2 * 32 + lane], tp[3 * 32 + lane], tp[4 * 32 + lane],
                           tp[5 * 32 + lane], pb_, ps_);
#pragma unroll
            for (int i = 0; i < 4; ++i)
                S.part[T][warp][i][lane] = make_float2(pb_[i], __int_as_float(ps_[i]));
        }
        if (any_long) {
            __syncthreads();   // every eighth of every long tile
            if (nt > kHeavySplit) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    float2 b2 = S.part[warp][0][i][lane];
                    best[i] = b2.x;
                    sl[i] = __float_as_int(b2.y);
                    for (int w = 1; w < kHeavyWarps; ++w) {
                        const float2 c2 = S.part[warp][w][i][lane];
                        if (c2.x < best[i]) {
                            best[i] = c2.x;
                            sl[i] = __float_as_int(c2.y);
                        }
                    }
                }
            }
        }
        if (MODE & kModeLabels) {
            *reinterpret_cast<int2*>(labels + pa) =
                make_int2(__ldg(&list[my[sl[0]]]), __ldg(&list[my[sl[1]]]));
            *reinterpret_cast<int2*>(labels + pb) =
                make_int2(__ldg(&list[my[sl[2]]]), __ldg(&list[my[sl[3]]]));
        }
        if (MODE & kModeReduce) {
            double j4 = 0.0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (v[i]) j4 += (double)best[i];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) j4 += __shfl_xor_sync(0xffffffffu, j4, o);
            // ---- sums: slot windows of 64, one butterfly per slot present ----
            int ne = 0;   // entries of this tile
            for (int w0 = 0; w0 < nt; w0 += kHeavySlots) {
                unsigned long long mine = 0ull;
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (v[i] && sl[i] >= w0 && sl[i] < w0 + kHeavySlots) mine |= 1ull << (sl[i] - w0);
                unsigned long long pres = __reduce_or_sync(0xffffffffu, (unsigned)mine);
                pres |= (unsigned long long)__reduce_or_sync(0xffffffffu, (unsigned)(mine >> 32)) << 32;
                while (pres) {   // ascending slots = ascending k
                    const int q = __ffsll((long long)pres) - 1;
                    pres &= pres - 1;
                    double sx = 0.0, sy = 0.0, sz = 0.0;
                    unsigned cnt = 0u;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const bool m = v[i] && sl[i] == w0 + q;
                        sx += m ? (double)px[i] : 0.0;
                        sy += m ? (double)py[i] : 0.0;
                        sz += m ? (double)pz[i] : 0.0;
                        cnt += __popc(__ballot_sync(0xffffffffu, m));
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        sx += __shfl_xor_sync(0xffffffffu, sx, o);
                        sy += __shfl_xor_sync(0xffffffffu, sy, o);
                        if (D == 3) sz += __shfl_xor_sync(0xffffffffu, sz, o);
                    }
                    if (lane == 0) {
                        KM_CHECK(ne < kLaneTile);
                        S.ent[warp][ne] = make_double4(sx, sy, sz,
                                                       pack_kn(__ldg(&list[my[w0 + q]]), (int)cnt));
                    }
                    ++ne;
                }
            }
            if (lane == 0) {
                S.wJ[warp] = j4;
                S.went[warp] = ne;
            }
        }
        __syncthreads();   // every tile's entries are in shared memory
#if KM_HEAVY_PROF
        const unsigned long long tp3 = (unsigned long long)global_ns();
#endif
        if ((MODE & kModeReduce) && warp == 0) {
            // the chunk row: tiles in order, each tile's entries in ascending k
            double* row = rows + (size_t)chunk * row_stride;
            int off = 0;
            double J = 0.0;
            for (int w = 0; w < kHeavyWarps; ++w) {
                const int ne = S.went[w];
                KM_CHECK(kRowHead + 4 * (off + ne) <= row_stride);
                for (int e = lane; e < ne; e += 32) {
                    const double4 x = S.ent[w][e];
                    double2* d2 = reinterpret_cast<double2*>(row + kRowHead) + 2 * (off + e);
                    d2[0] = make_double2(x.x, x.y);
                    d2[1] = make_double2(x.z, x.w);
                }
                off += ne;
                J += S.wJ[w];
            }
            if (lane == 0) {
                row[0] = J;
                row[1] = (double)off;
            }
        }
        __syncthreads();   // shared memory is reused by the next heavy chunk
#if KM_HEAVY_PROF
        if (tid == 0)
            printf("heavy h=%d chunk=%d gc=%d nt=%d,%d,%d,%d,%d,%d,%d,%d stage=%llu refine=%llu walk+agg=%llu row=%llu\n",
                   h, chunk, gc, S.wnt[0], S.wnt[1], S.wnt[2], S.wnt[3], S.wnt[4], S.wnt[5],
                   S.wnt[6], S.wnt[7], tp1 - tp0, tp2 - tp1, tp3 - tp2, (unsigned long long)global_ns() - tp3);
#endif
    }
}

// ---------------------------------------------------------------------------
// k_assign_heavy_tiles (large K, KM_HEAVY_TILES): the same heavy chunks, one
// 8-warp block per 128-point TILE instead of per chunk.  k_assign_heavy's
// length is its slowest chunk, and there one warp refines the whole super
// list (1024 entries: 2 x 32 dependent passes) and aggregates up to 128 slots
// alone; here the block's 8 warps share every step of one tile:
//   * the refinement: warp w tests list positions [128 w, 128 w + 128); the
//     minimiser of dmax2 (lowest position on ties) and the ascending tile list
//     are assembled across warps -- the same list as k_assign_heavy's;
//   * the argmin: the split walk (eighths, ascending strict-< combine) for
//     lists longer than kHeavySplit, else warp 0 alone;
//   * the sums: slot windows of 64 spread over the warps, each window's
//     entries at its prefix offset -- the same butterflies, so every entry is
//     bit-identical to k_assign_heavy's.
// A tile's entries go to its own stretch [T ts, T ts + ne) of the chunk row
// (ts = min(K, 128) >= its entry count) and its (J, ne) to htile; the block
// that completes the chunk's 8th tile (gpu fence + ticket, as in the
// threadfence reduction) moves the entries together in tile order and writes
// the row head with J summed in tile order: the row k_assign_heavy writes.
// ---------------------------------------------------------------------------
#ifndef KM_HEAVY_TILES
#define KM_HEAVY_TILES 1   // 1: k_assign_heavy_tiles, 0: k_assign_heavy (one block per chunk)
#endif
#ifndef KM_HEAVY_TILE_MINB
#define KM_HEAVY_TILE_MINB 4   // k_assign_heavy_tiles: resident blocks per SM (register cap)
#endif
constexpr int kHeavyTileSplit = kHeavyWarps;      // tile lists this long are walked by all 8 warps

// position of the r-th (0-based, ascending) set bit of m (r < popc(m))
__device__ __forceinline__ int nth_set_bit(unsigned m, int r) {
    int pos = 0;
#pragma unroll
    for (int w = 16; w > 0; w >>= 1) {
        const unsigned lowm = m & ((1u << w) - 1u);
        const int c = __popc(lowm);
        if (r >= c) {
            r -= c;
            m >>= w;
            pos += w;
        } else {
            m = lowm;
        }
    }
    return pos;
}

// Strict-< argmin of a lane's 4 points over positions [t0, t1) of a tile list
// whose centroids are gathered contiguously (tcl[t] = staged centroid of
// list position t): one LDS.128 per entry, four entries in flight per step;
// the updates stay in ascending position order (lowest position on ties).
template <int D>
__device__ __forceinline__ void argmin_walk_gathered(const float4* tcl, int t0, int t1, float2 xa,
                                                     float2 ya, float2 za, float2 xb, float2 yb,
                                                     float2 zb, float (&best)[4], int (&sl)[4]) {
    {
        const float4 cc = tcl[t0];
        const float2 da = form_d2<D>(xa, ya, za, cc), db = form_d2<D>(xb, yb, zb, cc);
        best[0] = da.x; best[1] = da.y; best[2] = db.x; best[3] = db.y;
        sl[0] = sl[1] = sl[2] = sl[3] = t0;
    }
    int t = t0 + 1;
    for (; t + 3 < t1; t += 4) {
        float2 da[4], db[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float4 cc = tcl[t + u];
            da[u] = form_d2<D>(xa, ya, za, cc);
            db[u] = form_d2<D>(xb, yb, zb, cc);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (da[u].x < best[0]) { best[0] = da[u].x; sl[0] = t + u; }
            if (da[u].y < best[1]) { best[1] = da[u].y; sl[1] = t + u; }
            if (db[u].x < best[2]) { best[2] = db[u].x; sl[2] = t + u; }
            if (db[u].y < best[3]) { best[3] = db[u].y; sl[3] = t + u; }
        }
    }
    for (; t < t1; ++t) {
        const float4 cc = tcl[t];
        const float2 da = form_d2<D>(xa, ya, za, cc), db = form_d2<D>(xb, yb, zb, cc);
        if (da.x < best[0]) { best[0] = da.x; sl[0] = t; }
        if (da.y < best[1]) { best[1] = da.y; sl[1] = t; }
        if (db.x < best[2]) { best[2] = db.x; sl[2] = t; }
        if (db.y < best[3]) { best[3] = db.y; sl[3] = t; }
    }
}

#ifndef KM_HEAVY_GATHER
#define KM_HEAVY_GATHER 1   // k_assign_heavy_tiles: tile-list centroids gathered before the walk
#endif

struct alignas(16) HeavyTileSmem {   // size a multiple of 16: float4 cl[] follows
    float2 part[kHeavyWarps][4][32];   // split walk: (distance, slot) per warp, point, lane
    float2 fin[4][32];                 // the tile's (distance, slot) per point and lane
    double wM[kHeavyWarps];
    int wMi[kHeavyWarps];
    int wcnt[kHeavyWarps];
    int last;
    // followed by float4 cl[K] (the super list's staged centroids), with
    // KM_HEAVY_GATHER float4 tcl[K] (the tile list's centroids), and
    // unsigned short tl[K] (the tile list: super-list positions)
};

template <int D, int MODE>
__global__ void __launch_bounds__(kHeavyWarps * 32, KM_HEAVY_TILE_MINB)
k_assign_heavy_tiles(const float* __restrict__ X, int64_t n, int K, const DevState* __restrict__ st,
                     int ignore_done, const int* __restrict__ slist,
                     const float4* __restrict__ scl, const int* __restrict__ scount,
                     const int* __restrict__ heavy, const int* __restrict__ heavy_count,
                     double* __restrict__ rows, int row_stride, int32_t* __restrict__ labels,
                     double2* __restrict__ htile, int* __restrict__ hctr) {
    if (!ignore_done && st->done) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    HeavyTileSmem& S = *reinterpret_cast<HeavyTileSmem*>(smem_raw);
    float4* cl = reinterpret_cast<float4*>(smem_raw + sizeof(HeavyTileSmem));   // [K]
    float4* tcl = cl + K;                                                       // [K] (gather)
    unsigned short* tl = reinterpret_cast<unsigned short*>(cl + (KM_HEAVY_GATHER ? 2 : 1) * K);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ts = K < kLaneTile ? K : kLaneTile;   // row entries reserved per tile
    (void)tcl;
    const int nitems = *heavy_count * kHeavyWarps;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        const int h = it / kHeavyWarps, T = it % kHeavyWarps;
        const int chunk = heavy[h];
#if KM_HEAVY_PROF
        const unsigned long long q0 = (unsigned long long)global_ns();
        unsigned long long q1 = 0, q2 = 0, q3 = 0, q4 = 0;
#endif
        const int* list = slist + (size_t)(chunk / kSuperChunks) * K;
        const int gc = scount[chunk / kSuperChunks];
        KM_CHECK(gc >= 1 && gc <= K && K <= 1024);
        // the tile's points: every warp holds all 128 (4 per lane)
        const int64_t pa = (int64_t)chunk * kSChunkPoints + T * kLaneTile + 2 * lane;
        const int64_t pb = pa + kWarpTile;
        const float2 xa = ld_stream2(tile_coord<D>(X, pa, 0));
        const float2 ya = ld_stream2(tile_coord<D>(X, pa, 1));
        const float2 za = (D == 3) ? ld_stream2(tile_coord<D>(X, pa, 2)) : make_float2(0.f, 0.f);
        const float2 xb = ld_stream2(tile_coord<D>(X, pb, 0));
        const float2 yb = ld_stream2(tile_coord<D>(X, pb, 1));
        const float2 zb = (D == 3) ? ld_stream2(tile_coord<D>(X, pb, 2)) : make_float2(0.f, 0.f);
        const float4* lcl = scl + (size_t)(chunk / kSuperChunks) * K;
        for (int i = tid; i < gc; i += blockDim.x) cl[i] = __ldg(&lcl[i]);
        const bool v[4] = {pa < n, pa + 1 < n, pb < n, pb + 1 < n};
        const float px[4] = {xa.x, xa.y, xb.x, xb.y}, py[4] = {ya.x, ya.y, yb.x, yb.y};
        const float pz[4] = {za.x, za.y, zb.x, zb.y};
        double tlo[3] = {0, 0, 0}, thi[3] = {0, 0, 0};
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const float* pj = j == 0 ? px : (j == 1 ? py : pz);
            float l_ = pos_inf(), h_ = -pos_inf();
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (v[i]) {
                    l_ = fminf(l_, pj[i]);
                    h_ = fmaxf(h_, pj[i]);
                }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                l_ = fminf(l_, __shfl_xor_sync(0xffffffffu, l_, o));
                h_ = fmaxf(h_, __shfl_xor_sync(0xffffffffu, h_, o));
            }
            tlo[j] = (double)l_;
            thi[j] = (double)h_;
        }
        const bool any_valid = tlo[0] <= thi[0];   // block-uniform; false for an all-padding tile
        __syncthreads();   // the super list's centroids are staged
#if KM_HEAVY_PROF
        q1 = (unsigned long long)global_ns();
#endif
        // ---- the super list refined against the tile box, across the warps ----
        int nt = 1;
        if (any_valid) {
            double Ml = (double)pos_inf();
            int Mil = 0x7fffffff;
#pragma unroll 4
            for (int i = warp * 32 + lane; i < gc; i += kHeavyWarps * 32) {
                const float4 c4 = cl[i];
                const float c[3] = {-c4.x, -c4.y, -c4.z};
                double a, b;
                box_bounds<D>(c, tlo, thi, a, b);
                if (b < Ml) {
                    Ml = b;
                    Mil = i;
                }
            }
            double M = Ml;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) M = fmin(M, __shfl_xor_sync(0xffffffffu, M, o));
            int Mi = (Ml == M) ? Mil : 0x7fffffff;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) Mi = min(Mi, __shfl_xor_sync(0xffffffffu, Mi, o));
            if (lane == 0) {
                S.wM[warp] = M;
                S.wMi[warp] = Mi;
            }
            __syncthreads();
            M = S.wM[0];
#pragma unroll
            for (int w = 1; w < kHeavyWarps; ++w) M = fmin(M, S.wM[w]);
            Mi = 0x7fffffff;   // the lowest position attaining M
#pragma unroll
            for (int w = 0; w < kHeavyWarps; ++w)
                if (S.wM[w] == M) Mi = min(Mi, S.wMi[w]);
            const float4 a4 = cl[Mi];
            const float ca[3] = {-a4.x, -a4.y, -a4.z};
            const double thr = prune_threshold(M);
            // warp w: positions [128 w, 128 w + 128) in 4 ballots; its candidates
            // follow those of warps < w (ascending positions = ascending k)
            unsigned m[4];
            int cnt = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int i = (warp * 4 + q) * 32 + lane;
                bool cand = false;
                if (i < gc) {
                    const float4 c4 = cl[i];
                    const float c[3] = {-c4.x, -c4.y, -c4.z};
                    double a, b;
                    box_bounds<D>(c, tlo, thi, a, b);
                    cand = a <= thr && !bisector_excludes<D>(c, ca, tlo, thi, b, M);
                }
                m[q] = __ballot_sync(0xffffffffu, cand);
                cnt += __popc(m[q]);
            }
            if (lane == 0) S.wcnt[warp] = cnt;
            __syncthreads();
            int off = 0;
            nt = 0;
#pragma unroll
            for (int w = 0; w < kHeavyWarps; ++w) {
                off += (w < warp) ? S.wcnt[w] : 0;
                nt += S.wcnt[w];
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if ((m[q] >> lane) & 1u)
                    tl[off + __popc(m[q] & ((1u << lane) - 1u))] = (unsigned short)((warp * 4 + q) * 32 + lane);
                off += __popc(m[q]);
            }
        } else if (tid == 0) {
            tl[0] = 0;   // an all-padding tile: list {position 0}, as k_assign_heavy
        }
        KM_CHECK(nt >= 1 && nt <= gc);
        __syncthreads();   // the tile list is complete
#if KM_HEAVY_PROF
        q2 = (unsigned long long)global_ns();
#endif
        // ---- exact argmin over the tile list (ascending k; strict <) ----
        float best[4];
        int sl[4];
        const bool split = nt >= kHeavyTileSplit;   // every eighth non-empty
#if KM_HEAVY_GATHER
        if (split) {   // long lists: the tile list's centroids made contiguous
            for (int i = tid; i < nt; i += blockDim.x) tcl[i] = cl[tl[i]];
            __syncthreads();
        }
#endif
        if (split) {
            const int t0 = (int)((int64_t)nt * warp / kHeavyWarps);
            const int t1 = (int)((int64_t)nt * (warp + 1) / kHeavyWarps);
#if KM_HEAVY_GATHER
            argmin_walk_gathered<D>(tcl, t0, t1, xa, ya, za, xb, yb, zb, best, sl);
#else
            argmin_walk<D>(tl, cl, t0, t1, xa, ya, za, xb, yb, zb, best, sl);
#endif
#pragma unroll
            for (int i = 0; i < 4; ++i) S.part[warp][i][lane] = make_float2(best[i], __int_as_float(sl[i]));
            __syncthreads();
        } else if (warp == 0) {
            argmin_walk<D>(tl, cl, 0, nt, xa, ya, za, xb, yb, zb, best, sl);
        }
        if (warp == 0) {
            if (split) {   // ascending eighths, strict <
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    for (int w = 1; w < kHeavyWarps; ++w) {
                        const float2 c2 = S.part[w][i][lane];
                        if (c2.x < best[i]) {
                            best[i] = c2.x;
                            sl[i] = __float_as_int(c2.y);
                        }
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) S.fin[i][lane] = make_float2(best[i], __int_as_float(sl[i]));
            if (MODE & kModeLabels) {
                *reinterpret_cast<int2*>(labels + pa) =
                    make_int2(__ldg(&list[tl[sl[0]]]), __ldg(&list[tl[sl[1]]]));
                *reinterpret_cast<int2*>(labels + pb) =
                    make_int2(__ldg(&list[tl[sl[2]]]), __ldg(&list[tl[sl[3]]]));
            }
        }
        if (MODE & kModeReduce) {
            __syncthreads();   // the tile's slots
#if KM_HEAVY_PROF
            q3 = (unsigned long long)global_ns();
#endif
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 f = S.fin[i][lane];
                best[i] = f.x;
                sl[i] = __float_as_int(f.y);
            }
            double* row = rows + (size_t)chunk * row_stride;
            const int nwin = any_valid ? (nt + kHeavySlots - 1) / kHeavySlots : 0;
            // slot windows of 64 in ascending order (block-uniform); the present
            // slots of a window are dealt round-robin to the warps, each entry
            // written at its rank -- entries stay in ascending k
            int ne = T * ts;   // the next entry of this tile's stretch
            for (int wi = 0; wi < nwin; ++wi) {
                const int w0 = wi * kHeavySlots;
                unsigned long long mine = 0ull;
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (v[i] && sl[i] >= w0 && sl[i] < w0 + kHeavySlots) mine |= 1ull << (sl[i] - w0);
                const unsigned plo = __reduce_or_sync(0xffffffffu, (unsigned)mine);
                const unsigned phi = __reduce_or_sync(0xffffffffu, (unsigned)(mine >> 32));
                const int nlo = __popc(plo), np = nlo + __popc(phi);
                for (int r = warp; r < np; r += kHeavyWarps) {
                    const int q = r < nlo ? nth_set_bit(plo, r) : 32 + nth_set_bit(phi, r - nlo);
                    double sx = 0.0, sy = 0.0, sz = 0.0;
                    unsigned cnt = 0u;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const bool mm = v[i] && sl[i] == w0 + q;
                        sx += mm ? (double)px[i] : 0.0;
                        sy += mm ? (double)py[i] : 0.0;
                        sz += mm ? (double)pz[i] : 0.0;
                        cnt += __popc(__ballot_sync(0xffffffffu, mm));
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        sx += __shfl_xor_sync(0xffffffffu, sx, o);
                        sy += __shfl_xor_sync(0xffffffffu, sy, o);
                        if (D == 3) sz += __shfl_xor_sync(0xffffffffu, sz, o);
                    }
                    if (lane == 0) {
                        KM_CHECK(ne + r < (T + 1) * ts);
                        double2* d2 = reinterpret_cast<double2*>(row + kRowHead) + 2 * (ne + r);
                        d2[0] = make_double2(sx, sy);
                        d2[1] = make_double2(sz, pack_kn(__ldg(&list[tl[w0 + q]]), (int)cnt));
                    }
                }
                ne += np;
            }
            if (warp == 0) {
                double j4 = 0.0;
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (v[i]) j4 += (double)best[i];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) j4 += __shfl_xor_sync(0xffffffffu, j4, o);
                if (lane == 0) htile[(size_t)h * kHeavyWarps + T] = make_double2(j4, (double)(ne - T * ts));
            }
            // ---- the chunk's last tile assembles the row ----
#if KM_HEAVY_PROF
            __syncthreads();
            q4 = (unsigned long long)global_ns();
#endif
            __threadfence();
            __syncthreads();
            if (tid == 0) S.last = atomicAdd(&hctr[h], 1) == kHeavyWarps - 1;
            __syncthreads();
            if (S.last) {   // block-uniform
                __threadfence();
                int cnt[kHeavyWarps], tot = 0;
                double J = 0.0;
#pragma unroll
                for (int u = 0; u < kHeavyWarps; ++u) {
                    const double2 jn = __ldcg(&htile[(size_t)h * kHeavyWarps + u]);
                    cnt[u] = (int)jn.y;
                    tot += cnt[u];
                    J += jn.x;
                }
                // every entry read before any is moved (the moves overlap)
                constexpr int kPer = kSChunkPoints / (kHeavyWarps * 32);   // 4 entries per thread
                double2 e0[kPer], e1[kPer];
                int dst[kPer];
#pragma unroll
                for (int r = 0; r < kPer; ++r) {
                    const int g = tid + r * kHeavyWarps * 32;   // position in the compacted row
                    dst[r] = -1;
                    if (g < tot) {
                        int u = 0, base = 0;
                        while (g >= base + cnt[u]) base += cnt[u++];
                        const double2* s2 = reinterpret_cast<const double2*>(row + kRowHead) +
                                            2 * (u * ts + g - base);
                        e0[r] = __ldcg(s2);
                        e1[r] = __ldcg(s2 + 1);
                        dst[r] = g;
                    }
                }
                __syncthreads();
#pragma unroll
                for (int r = 0; r < kPer; ++r)
                    if (dst[r] >= 0) {
                        double2* d2 = reinterpret_cast<double2*>(row + kRowHead) + 2 * dst[r];
                        d2[0] = e0[r];
                        d2[1] = e1[r];
                    }
                if (tid == 0) {
                    KM_CHECK(kRowHead + 4 * tot <= row_stride);
                    row[0] = J;
                    row[1] = (double)tot;
                    hctr[h] = 0;   // ready for the next iteration
                }
            }
        } else {
            __syncthreads();
        }
        __syncthreads();   // shared memory is reused by the next tile
#if KM_HEAVY_PROF
        if (tid == 0)
            printf("htile blk=%d h=%d T=%d chunk=%d gc=%d nt=%d start=%llu stage=%llu refine=%llu walk=%llu sums=%llu row=%llu\n",
                   blockIdx.x, h, T, chunk, gc, nt, q0, q1 - q0, q2 - q1, q3 - q2, q4 - q3,
                   (unsigned long long)global_ns() - q4);
#endif
    }
}

// ---------------------------------------------------------------------------
// k_prune (large K): candidates of each super box (kSuperChunks chunks) by the
// same exclusion test, listed in ascending k.
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256)
k_prune(const float4* __restrict__ cneg_buf, const DevState* __restrict__ st, int mu_sel,
        int ignore_done, int K, const float* __restrict__ sbox, int* __restrict__ slist,
        float4* __restrict__ scl,
        int* __restrict__ scount, int* __restrict__ heavy_count) {
    if (!ignore_done && st->done) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) *heavy_count = 0;   // the assign's heavy list
    __shared__ double wmin[8];
    __shared__ int wcnt[8];
    __shared__ int wmi[8];
    __shared__ int base_s;
    const int s = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float4* cneg = cneg_buf + (size_t)mu_sel * K;
    double lo[3], hi[3];
#pragma unroll
    for (int j = 0; j < D; ++j) {
        lo[j] = (double)sbox[(size_t)s * 2 * D + j];
        hi[j] = (double)sbox[(size_t)s * 2 * D + D + j];
    }
    auto bounds = [&](int k, double& dmin2, double& dmax2) {
        dmin2 = 0.0;
        dmax2 = 0.0;
        const float4 v = cneg[k];
        const float cv[3] = {-v.x, -v.y, -v.z};
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const double cj = (double)cv[j];
            const double dm = fmax(fmax(lo[j] - cj, cj - hi[j]), 0.0);
            dmin2 += dm * dm;
            const double dx = fmax(fabs(cj - lo[j]), fabs(hi[j] - cj));
            dmax2 += dx * dx;
        }
    };
    // thread tid takes centroids tid + 256 j (K <= 1024: j < 4); both passes
    // use the same bounds and centroid, kept in registers
    constexpr int kPer = 1024 / 256;
    KM_CHECK(K <= kPer * 256 && blockDim.x == 256);
    double ca_[kPer], cb_[kPer];
    float4 cv_[kPer];
    double Mt = (double)pos_inf();   // this thread's min dmax2 and its centroid
    int Mkt = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const int k = tid + 256 * j;
        ca_[j] = cb_[j] = 0.0;
        cv_[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k < K) {
            bounds(k, ca_[j], cb_[j]);
            cv_[j] = cneg[k];
            if (cb_[j] < Mt) {
                Mt = cb_[j];
                Mkt = k;
            }
        }
    }
    double M = Mt;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmin(M, __shfl_xor_sync(0xffffffffu, M, o));
    int Mk = (Mt == M) ? Mkt : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) Mk = min(Mk, __shfl_xor_sync(0xffffffffu, Mk, o));
    if (lane == 0) {
        wmin[warp] = M;
        wmi[warp] = Mk;
    }
    if (tid == 0) base_s = 0;
    __syncthreads();
    M = wmin[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) M = fmin(M, wmin[w]);
    Mk = 0x7fffffff;   // the lowest centroid attaining M: a
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
        if (wmin[w] == M) Mk = min(Mk, wmi[w]);
    const float4 av = cneg[Mk];
    const float ca[3] = {-av.x, -av.y, -av.z};
    const double thr = prune_threshold(M);
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        if (256 * j >= K) break;   // block-uniform
        const int k = tid + 256 * j;
        bool cand = false;
        const float4 v = cv_[j];
        if (k < K) {
            const float c[3] = {-v.x, -v.y, -v.z};
            cand = ca_[j] <= thr && !bisector_excludes<D>(c, ca, lo, hi, cb_[j], M);
        }
        const unsigned mask = __ballot_sync(0xffffffffu, cand);
        if (lane == 0) wcnt[warp] = __popc(mask);
        __syncthreads();
        int off = base_s;
        for (int w = 0; w < warp; ++w) off += wcnt[w];
        if (cand) {
            const size_t at = (size_t)s * K + off + __popc(mask & ((1u << lane) - 1u));
            slist[at] = k;
            scl[at] = make_float4(v.x, v.y, v.z, __int_as_float(k));   // staged centroid, k
        }
        __syncthreads();
        if (tid == 0) {
            int t = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += wcnt[w];
            base_s += t;
        }
        __syncthreads();
    }
    if (tid == 0) scount[s] = base_s;
}

// super boxes from the chunk boxes (create time)
__global__ void k_super_bbox(const float* __restrict__ cbox, int n_chunks, int d,
                             float* __restrict__ sbox) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    const int c0 = s * kSuperChunks;
    if (c0 >= n_chunks) return;
    const int c1 = min(n_chunks, c0 + kSuperChunks);
    for (int j = 0; j < d; ++j) {
        float lo = pos_inf(), hi = -pos_inf();
        for (int c = c0; c < c1; ++c) {
            lo = fminf(lo, cbox[(size_t)c * 2 * d + j]);
            hi = fmaxf(hi, cbox[(size_t)c * 2 * d + d + j]);
        }
        sbox[(size_t)s * 2 * d + j] = lo;
        sbox[(size_t)s * 2 * d + d + j] = hi;
    }
}

// ---------------------------------------------------------------------------
// k_merge_sparse: group g sums the sparse rows of its kGroupChunks chunks into
// a dense shared table T[K][4].  Entries are staged in shared memory with
// independent loads; then warp w adds, chunk by chunk in ascending order, the
// entries whose k lies in its own range of T -- every sum is taken in chunk
// order, no atomics, no block barrier per chunk.  Writes the group's column
// gpart[e][g] for k_merge.
// ---------------------------------------------------------------------------
constexpr int kMergeBatch = 512;   // entries staged per batch

template <int D>
__global__ void __launch_bounds__(256)
k_merge_sparse(const double* __restrict__ rows, int row_stride, int n_chunks, int K,
               double* __restrict__ gpart, int n_groups, const DevState* __restrict__ st,
               int ignore_done) {
    if (!ignore_done && st->done) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* T = reinterpret_cast<double*>(smem_raw);   // [K][4]: Sx Sy Sz n
    __shared__ double hj[kGroupChunks];
    __shared__ int cnt[kGroupChunks];
    __shared__ int off[kGroupChunks + 1];
    __shared__ double2 E[2 * kMergeBatch];   // entry = {Sx, Sy}, {Sz, kn}
    const int g = blockIdx.x, tid = threadIdx.x;
    const int c0 = g * kGroupChunks;
    const int nch = min(n_chunks, c0 + kGroupChunks) - c0;
    for (int q = tid; q < 4 * K; q += blockDim.x) T[q] = 0.0;
    for (int q = tid; q < nch; q += blockDim.x) {
        const double* row = rows + (size_t)(c0 + q) * row_stride;
        hj[q] = row[0];
        cnt[q] = (int)row[1];
        KM_CHECK(cnt[q] >= 0 && kRowHead + 4 * cnt[q] <= row_stride);
    }
    __syncthreads();
    if (tid < 32) {   // exclusive scan of the counts (warp 0, kPer consecutive per lane)
        constexpr int kPer = (kGroupChunks + 31) / 32;
        int a[kPer], sum = 0;
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            const int c = tid * kPer + i;
            a[i] = (c < nch) ? cnt[c] : 0;
            sum += a[i];
        }
        int x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (tid >= o) x += y;
        }
        int run = x - sum;
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            const int c = tid * kPer + i;
            if (c < nch) off[c] = run;
            run += a[i];
        }
        if (tid == 31) off[nch] = x;
    }
    __syncthreads();
    const int total = off[nch];
    for (int b0 = 0; b0 < total; b0 += kMergeBatch) {
        const int bn = min(kMergeBatch, total - b0);
        // stage entries [b0, b0 + bn) (2 double2 each): every thread issues its
        // (up to 4) independent loads before any store
        double2 tmp[4];
        int dst[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int q = tid + r * (int)blockDim.x;
            dst[r] = -1;
            if (q < 2 * bn) {
                const int idx = b0 + (q >> 1);
                int lo_ = 0, hi_ = nch;   // chunk with off[c] <= idx < off[c + 1]
                while (hi_ - lo_ > 1) {
                    const int mid = (lo_ + hi_) >> 1;
                    if (off[mid] <= idx) lo_ = mid; else hi_ = mid;
                }
                const double* row = rows + (size_t)(c0 + lo_) * row_stride + kRowHead;
                tmp[r] = reinterpret_cast<const double2*>(row)[2 * (idx - off[lo_]) + (q & 1)];
                dst[r] = q;
            }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
            if (dst[r] >= 0) E[dst[r]] = tmp[r];
        __syncthreads();
        // warp w owns k in [w kw, (w + 1) kw) and walks the batch's entries in
        // windows of 32 consecutive entries (entry order = chunk order).  Lanes
        // of one window holding the same k (entries of different chunks) are
        // found with __match_any_sync and add in lane order, one round per
        // rank; __syncwarp orders the rounds and the windows -- every T[k] is
        // summed in ascending chunk order, no atomics, no block barrier
        {
            const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
            const int kw = (K + nw - 1) / nw, klo = warp * kw, khi = klo + kw;
            for (int w0 = 0; w0 < bn; w0 += 32) {
                const int e = w0 + lane;
                double2 v0 = make_double2(0.0, 0.0), v1 = make_double2(0.0, 0.0);
                int k = -1;
                if (e < bn) {
                    v1 = E[2 * e + 1];
                    const int2 kn = *reinterpret_cast<const int2*>(&v1.y);   // {k, n}
                    KM_CHECK(kn.x >= 0 && kn.x < K && kn.y >= 0);
                    if (kn.x >= klo && kn.x < khi) { k = kn.x; v0 = E[2 * e]; }
                }
                const unsigned peers = __match_any_sync(0xffffffffu, k);
                const int rank = __popc(peers & ((1u << lane) - 1u));
                const int rmax = __reduce_max_sync(0xffffffffu, k >= 0 ? rank : 0);
                const double n = (double)reinterpret_cast<const int2*>(&v1.y)->y;
                for (int r = 0; r <= rmax; ++r) {
                    if (k >= 0 && rank == r) {
                        double2* t = reinterpret_cast<double2*>(T + 4 * k);
                        double2 a = t[0], b = t[1];
                        a.x += v0.x;
                        a.y += v0.y;
                        b.x += v1.x;
                        b.y += n;
                        t[0] = a;
                        t[1] = b;
                    }
                    __syncwarp();
                }
            }
        }
        __syncthreads();   // the batch buffer is reused
    }
    __syncthreads();
    for (int k = tid; k < K; k += blockDim.x) {
        for (int j = 0; j < D; ++j) gpart[(size_t)(k * D + j) * n_groups + g] = T[4 * k + j];
        gpart[(size_t)(K * D + k) * n_groups + g] = T[4 * k + 3];
    }
    if (tid == 0) {
        double J = 0.0;
        for (int cc = 0; cc < nch; ++cc) J += hj[cc];
        gpart[(size_t)(K * D + K) * n_groups + g] = J;
    }
}

// ---------------------------------------------------------------------------
// block_merge_groups: rs[e] = red[e] = sum over the G group columns of part
// [e][G], in the order of k_merge (lane l: groups l, l + 32, ... ascending,
// then a butterfly over the lanes) -- bit-identical to k_merge.  Warp w takes
// entries w, w + nwarp, ... four at a time so that 16 loads are in flight per
// lane.
// ---------------------------------------------------------------------------
template <int R = 4>   // entries per warp per pass (all loads of a pass in flight at once)
__device__ __forceinline__ void block_merge_groups(const double* part, int G, int nE,
                                                   double* rs, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    for (int e0 = warp; e0 < nE; e0 += R * nwarp) {
        double v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = 0.0;
#pragma unroll 4
        for (int b = lane; b < G; b += 32) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int e = e0 + r * nwarp;
                if (e < nE) v[r] += __ldcg(part + (size_t)e * G + b);   // L2: may be written by other blocks of this kernel
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v[r] += __shfl_xor_sync(0xffffffffu, v[r], o);
            const int e = e0 + r * nwarp;
            if (lane == 0 && e < nE) {
                rs[e] = v[r];
                if (red) red[e] = v[r];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// k_merge_sparse16 (sorted path, K <= 16): group g = chunks [1024 g, 1024 (g+1)),
// thread = chunk.  Each lane holds its row's head and up to kMergeRegs entries
// in registers (two loaded speculatively with the head, the rest in one more
// round when some lane needs them); then for every k present in the warp
// (ascending) the 32 lanes' contributions are added by a fixed butterfly, and
// the 32 warp results in warp order -> gpart[e][g].  Entries beyond kMergeRegs
// (rare) are added afterwards, rows in lane order.  Fixed order, no atomics.
// ---------------------------------------------------------------------------
constexpr int kMergeRegs = 6;

template <int D>
__device__ __forceinline__ void merge16_body(const double* __restrict__ cpart, int n_chunks, int K,
                                             double* __restrict__ gpart, int n_groups,
                                             const DevState* __restrict__ st, int ignore_done,
                                             const int g) {
    __shared__ __align__(16) double T[kMergeWarps][16][4];   // [warp][k]{Sx, Sy, Sz, n}
    __shared__ double WJ[kMergeWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = g * kRowGroup + tid;
    const double* row = cpart + (size_t)c * kRowDoubles;
    const double2* ent = reinterpret_cast<const double2*>(row + kRowHead);
    // round 1 (independent loads): done flag, head, entry slots 0 and 1
    const int done = ignore_done ? 0 : st->done;
    double2 head = make_double2(0.0, 0.0);
    double2 ea[kMergeRegs], eb[kMergeRegs];
#pragma unroll
    for (int i = 0; i < kMergeRegs; ++i) ea[i] = eb[i] = make_double2(0.0, 0.0);
    if (c < n_chunks) {
        head = *reinterpret_cast<const double2*>(row);
        ea[0] = ent[0];
        eb[0] = ent[1];
        ea[1] = ent[2];
        eb[1] = ent[3];
    }
    if (done) return;
    for (int i = tid; i < kMergeWarps * 32; i += blockDim.x)   // kMergeWarps * 64 doubles
        reinterpret_cast<double2*>(&T[0][0][0])[i] = make_double2(0.0, 0.0);
    const int n = (int)head.y;
    // round 2 (only warps with a longer row): entries 2 .. kMergeRegs - 1
    if (__any_sync(0xffffffffu, n > 2)) {
#pragma unroll
        for (int i = 2; i < kMergeRegs; ++i)
            if (i < n) {
                ea[i] = ent[2 * i];
                eb[i] = ent[2 * i + 1];
            }
    }
    KM_CHECK(n >= 0 && n <= 16);
    int kk[kMergeRegs];
    unsigned kset = 0u;
#pragma unroll
    for (int i = 0; i < kMergeRegs; ++i) {
        kk[i] = (i < n) ? __double2loint(eb[i].y) : -1;
        KM_CHECK(i >= n || (kk[i] >= 0 && kk[i] < K));
        if (i < n) kset |= 1u << kk[i];
    }
    double J = head.x;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) J += __shfl_xor_sync(0xffffffffu, J, o);
    if (lane == 0) WJ[warp] = J;
    unsigned m = __reduce_or_sync(0xffffffffu, kset);
    __syncthreads();   // T zeroed
    while (m) {
        const int k = __ffs(m) - 1;
        m &= m - 1;
        double sx = 0.0, sy = 0.0, sz = 0.0, cn = 0.0;
#pragma unroll
        for (int i = 0; i < kMergeRegs; ++i)
            if (kk[i] == k) {
                sx = ea[i].x;
                sy = ea[i].y;
                sz = eb[i].x;
                cn = (double)__double2hiint(eb[i].y);
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sx += __shfl_xor_sync(0xffffffffu, sx, o);
            sy += __shfl_xor_sync(0xffffffffu, sy, o);
            if (D == 3) sz += __shfl_xor_sync(0xffffffffu, sz, o);
            cn += __shfl_xor_sync(0xffffffffu, cn, o);
        }
        if (lane == 0) {
            T[warp][k][0] = sx;
            T[warp][k][1] = sy;
            T[warp][k][2] = sz;
            T[warp][k][3] = cn;
        }
    }
    // entries kMergeRegs.. of the (rare) longer rows: rows in lane order, the
    // warp loading one row's extra entries at a time (distinct k within a row)
    unsigned more = __ballot_sync(0xffffffffu, n > kMergeRegs);
    const double2* wrow = reinterpret_cast<const double2*>(
        cpart + (size_t)(g * kRowGroup + warp * 32) * kRowDoubles + kRowHead) + 2 * kMergeRegs;
    constexpr int kRowD2 = kRowDoubles / 2;
    // software-pipelined: the next long row's entries load while this one is added
    int j = more ? __ffs(more) - 1 : 0;
    int nx = __shfl_sync(0xffffffffu, n, j) - kMergeRegs;
    double2 v = make_double2(0.0, 0.0);
    if (more && lane < 2 * nx) v = wrow[(size_t)j * kRowD2 + lane];   // nx <= 16 - kMergeRegs
    while (more) {
        more &= more - 1;
        const int jn = more ? __ffs(more) - 1 : 0;
        const int nxn = __shfl_sync(0xffffffffu, n, jn) - kMergeRegs;
        double2 vn = make_double2(0.0, 0.0);
        if (more && lane < 2 * nxn) vn = wrow[(size_t)jn * kRowD2 + lane];
        const double kn = __shfl_sync(0xffffffffu, v.y, lane | 1);
        if (lane < 2 * nx) {
            double* t = &T[warp][__double2loint(kn)][2 * (lane & 1)];
            t[0] += v.x;
            t[1] += (lane & 1) ? (double)__double2hiint(v.y) : v.y;
        }
        __syncwarp();
        v = vn;
        nx = nxn;
    }
    __syncthreads();
    if (tid == 64) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < kMergeWarps; ++w) s += WJ[w];
        gpart[(size_t)(K * D + K) * n_groups + g] = s;
    } else if (tid < 64) {
        const int k = tid >> 2, q = tid & 3;
        if (k < K && (q < D || q == 3)) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < kMergeWarps; ++w) s += T[w][k][q];
            if (q < D) gpart[(size_t)(k * D + q) * n_groups + g] = s;
            else gpart[(size_t)(K * D + k) * n_groups + g] = s;
        }
    }
}

template <int D>
__global__ void __launch_bounds__(kRowGroup)
k_merge_sparse16(const double* __restrict__ cpart, int n_chunks, int K, double* __restrict__ gpart,
                 int n_groups, const DevState* __restrict__ st, int ignore_done) {
    pdl_trigger();
    pdl_wait();   // the rows are written
    merge16_body<D>(cpart, n_chunks, K, gpart, n_groups, st, ignore_done, blockIdx.x);
}


// k_merge_rows (dense rows): group g sums the rows of chunks
// [kDenseGroup g, kDenseGroup (g+1)).  Thread (r, q), r < 4, sums entry q of rows
// c0 + r, c0 + r + 4, ... in ascending order; the four stripes are then added
// in order r = 0..3 -- a fixed summation tree.  Scatters to gpart[e][g].
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(288)
k_merge_rows(const double* __restrict__ cpart, int n_chunks, int K, double* __restrict__ gpart,
             int n_groups, const DevState* __restrict__ st, int ignore_done) {
    if (!ignore_done && st->done) return;
    __shared__ double P[4][65];
    const int tid = threadIdx.x;
    const int r = tid / 65, q = tid - 65 * r;   // stripe, row entry (64 = J)
    const int g = blockIdx.x;
    const int c0 = g * kDenseGroup;
    const int c1 = min(n_chunks, c0 + kDenseGroup);
    if (r < 4) {
        double v = 0.0;
#pragma unroll 8
        for (int c = c0 + r; c < c1; c += 4) v += cpart[(size_t)c * kRowDoubles + q];
        P[r][q] = v;
    }
    __syncthreads();
    if (tid > 64) return;
    const double v = ((P[0][tid] + P[1][tid]) + P[2][tid]) + P[3][tid];
    if (tid == 64) {
        gpart[(size_t)(K * D + K) * n_groups + g] = v;
        return;
    }
    const int k = tid >> 2, j = tid & 3;
    if (k < K) {
        if (j < D) gpart[(size_t)(k * D + j) * n_groups + g] = v;
        else if (j == 3) gpart[(size_t)(K * D + k) * n_groups + g] = v;
    }
}

// ---------------------------------------------------------------------------
// Large-K full scan (16 < K <= 1024; KMEANS_FLAG_NO_SORT and shards the sorted
// path does not take).  The work is K form-D distances per point (6 FP32
// lane-ops each): FP32-pipe bound, so the design is about
// issue slots per (point, centroid) pair.
//   - Each warp step covers NPL 128-point sub-tiles (4 points per lane
//     each, packed f32x2 pairs), the next step's points prefetched into
//     registers while this one runs.
//   - Centroids staged once per launch in smem as negated float4, padded to a
//     multiple of kLargeKT with +inf (their distances are +inf); one broadcast
//     LDS.128 feeds 4 x NPL points.  NPL = 2 (more independent chains per
//     warp) when the smem accumulators allow one block per SM only, else 1
//     (fewer registers: two or more blocks per SM).
//   - Argmin in steps of kLargeKT centroids: per point, a 3-input min tree
//     (FMNMX3) over the step's distances and the running best, then one
//     compare-select of the step index when the min strictly drops -- ~0.75
//     issue slots per pair at 8 instead of a compare and two selects.  Strict < keeps the
//     first step reaching the minimum; after the scan the winning step's 8
//     distances are recomputed (the same RN operations, so bit-identical) and
//     the lowest k with d_k == min is the label: exactly the serial strict-<
//     argmin (lowest index on ties).  All distances +inf -> label 0.
//   - Sums: per-warp fp64 accumulators accS[w][k][D] and counts accN[w][k] in
//     smem.  Per point slot the lanes with equal labels (match_any) are summed
//     in a fixed tree over their ranks and the group's lowest lane adds the
//     result, so the sums are deterministic and a warp whose 32 points share
//     one label costs 5 shuffle levels, not 32 serial rounds; the block row is
//     the sum over warps in warp order.
// ---------------------------------------------------------------------------
#ifndef KM_LARGE_KT
#define KM_LARGE_KT 8    // centroids per argmin step
#endif
constexpr int kLargeKT = KM_LARGE_KT;
static_assert(kLargeKT == 8 || kLargeKT == 16, "argmin step: 8 or 16 centroids");
#ifndef KM_LARGE_UNROLL
#define KM_LARGE_UNROLL 1   // argmin steps per loop iteration
#endif
constexpr int kLargeUnroll = KM_LARGE_UNROLL;

__host__ __device__ constexpr int large_kpad(int K) {
    return (K + kLargeKT - 1) / kLargeKT * kLargeKT;
}

template <int D>
__device__ __forceinline__ void load_lane_pts(const float* __restrict__ X, int64_t sub, int lane,
                                              LanePts& P) {
    const int64_t pa = sub * kLaneTile + 2 * lane, pb = pa + kWarpTile;
    P.xa = ld_stream2(tile_coord<D>(X, pa, 0));
    P.ya = ld_stream2(tile_coord<D>(X, pa, 1));
    P.za = (D == 3) ? ld_stream2(tile_coord<D>(X, pa, 2)) : make_float2(0.f, 0.f);
    P.xb = ld_stream2(tile_coord<D>(X, pb, 0));
    P.yb = ld_stream2(tile_coord<D>(X, pb, 1));
    P.zb = (D == 3) ? ld_stream2(tile_coord<D>(X, pb, 2)) : make_float2(0.f, 0.f);
}

// min(best, v[0..KT)) by a 3-input min tree (FMNMX3)
template <int KT>
__device__ __forceinline__ float min_tree(const float (&v)[KT], float best) {
    if constexpr (KT == 8) {
        const float a = fminf(fminf(v[0], v[1]), v[2]);
        const float b = fminf(fminf(v[3], v[4]), v[5]);
        const float c = fminf(fminf(v[6], v[7]), best);
        return fminf(fminf(a, b), c);
    } else {
        const float a = fminf(fminf(v[0], v[1]), v[2]);
        const float b = fminf(fminf(v[3], v[4]), v[5]);
        const float c = fminf(fminf(v[6], v[7]), v[8]);
        const float d = fminf(fminf(v[9], v[10]), v[11]);
        const float e = fminf(fminf(v[12], v[13]), v[14]);
        const float f = fminf(v[15], best);
        return fminf(fminf(fminf(a, b), c), fminf(fminf(d, e), f));
    }
}

// Negated fl32 centroids (RN) in smem, +inf past K.
template <int D>
__device__ __forceinline__ void large_stage(float4* cen, const double* mu, int K, int Kp, int tid,
                                            int nthr) {
    for (int k = tid; k < Kp; k += nthr) {
        float4 c = make_float4(pos_inf(), pos_inf(), pos_inf(), 0.0f);
        if (k < K) {
            c.x = -__double2float_rn(mu[k * D + 0]);
            c.y = -__double2float_rn(mu[k * D + 1]);
            c.z = (D == 3) ? -__double2float_rn(mu[k * D + 2]) : 0.0f;
        }
        cen[k] = c;
    }
}

// One point slot of a warp into its accumulators: the lanes sharing a label
// (match_any) form a group; its sum is a fixed tree over the group's ranks
// (pointer jumping through the next member), and the group's lowest lane adds
// it and the group size -- ~log2(group size) shuffle levels whatever the mix.
template <int D>
__device__ __forceinline__ void large_accum_slot(bool v, int lab, float x, float y, float z,
                                                 double* __restrict__ myS, int* __restrict__ myN,
                                                 int lane) {
    const unsigned peers = __match_any_sync(0xffffffffu, v ? lab : -1 - lane);
    const int r = __popc(peers & ((1u << lane) - 1u)), g = __popc(peers);
    const int maxg = __reduce_max_sync(0xffffffffu, (unsigned)g);
    double ax = (double)x, ay = (double)y, az = (double)z;
    const unsigned above = peers & (0xfffffffeu << lane);
    int nxt = above ? __ffs(above) - 1 : lane;   // rank r + 1
    for (int st = 1; st < maxg; st <<= 1) {       // nxt = rank r + st
        const double ox = __shfl_sync(0xffffffffu, ax, nxt);
        const double oy = __shfl_sync(0xffffffffu, ay, nxt);
        const double oz = (D == 3) ? __shfl_sync(0xffffffffu, az, nxt) : 0.0;
        const int nn = __shfl_sync(0xffffffffu, nxt, nxt);
        if ((r & (2 * st - 1)) == 0 && r + st < g) {
            ax += ox;
            ay += oy;
            if (D == 3) az += oz;
        }
        nxt = nn;
    }
    if (v && r == 0) {
        double* sp = myS + (size_t)lab * D;
        sp[0] += ax;
        sp[1] += ay;
        if (D == 3) sp[2] += az;
        myN[lab] += g;
    }
    __syncwarp();
}

// The block's row: part[e][blockIdx] = sum over warps (warp order) of the
// per-warp accumulators; J from each warp's lane-order butterfly.
template <int D>
__device__ __forceinline__ void large_block_row(const double* accS, const int* accN,
                                                double* warpJ, double J, int K, int W, int tid,
                                                int nthr, double* __restrict__ part) {
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) J += __shfl_xor_sync(0xffffffffu, J, o);
    if (lane == 0) warpJ[warp] = J;
    __syncthreads();
    const int G = gridDim.x;
    const int nE = K * D + K + 1;
    for (int e = tid; e < nE; e += nthr) {
        double v = 0.0;
        if (e < K * D) {
            for (int w = 0; w < W; ++w) v += accS[(size_t)w * K * D + e];
        } else if (e < K * D + K) {
            long long c = 0;
            for (int w = 0; w < W; ++w) c += accN[w * K + (e - K * D)];
            v = (double)c;
        } else {
            for (int w = 0; w < W; ++w) v += warpJ[w];
        }
        part[(size_t)e * G + blockIdx.x] = v;
    }
}

// MODE as elsewhere; SPLIT: labels only, no accumulators in smem (the sums
// come from k_accum_large over the written labels), for K where the per-warp
// accumulators would cap the warps per SM.
template <int D, int MODE, int NPL, bool SPLIT = false>
__global__ void __launch_bounds__(kLargeTPBMax)
k_assign_large(const float* __restrict__ X, int64_t ldx, int64_t n, int K,
               const double* __restrict__ mu_buf, const DevState* __restrict__ st,
               int mu_sel, int ignore_done, double* __restrict__ part,
               int32_t* __restrict__ labels) {
    (void)ldx;   // whole 128-point sub-tiles: the padded tail of X is zeros
    if (!ignore_done && st->done) return;
    constexpr int NP = 4 * NPL;   // points per lane per step
    constexpr bool RED = !SPLIT && (MODE & kModeReduce);
    constexpr bool LAB = SPLIT || (MODE & kModeLabels);
    const int t_it = st->t;
    const double* mu = mu_buf + (size_t)((t_it - mu_sel) & 1) * K * D;
    const int Kp = large_kpad(K);

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x;
    const int nthr = blockDim.x;
    const int W = nthr >> 5;
    const int lane = tid & 31, warp = tid >> 5;
    float4* cen = reinterpret_cast<float4*>(smem_raw);                  // [Kp]
    double* accS = reinterpret_cast<double*>(cen + Kp);                 // [W][K][D]
    int* accN = reinterpret_cast<int*>(accS + (size_t)W * K * D);        // [W][K]
    double* warpJ = reinterpret_cast<double*>(accN + W * K + ((W * K) & 1));  // [W]

    large_stage<D>(cen, mu, K, Kp, tid, nthr);
    if (RED) {
        for (int q = tid; q < W * K * D; q += nthr) accS[q] = 0.0;
        for (int q = tid; q < W * K; q += nthr) accN[q] = 0;
    }
    __syncthreads();

    double* myS = accS + (size_t)warp * K * D;
    int* myN = accN + warp * K;
    double J = 0.0;

    // warp step = NPL consecutive 128-point sub-tiles
    const int64_t n_tiles = (n + NPL * kLaneTile - 1) / (NPL * kLaneTile);
    const int64_t stride = (int64_t)gridDim.x * W;
    int64_t tile = (int64_t)blockIdx.x * W + warp;
    LanePts P[NPL];
    if (tile < n_tiles) {
#pragma unroll
        for (int h = 0; h < NPL; ++h) load_lane_pts<D>(X, tile * NPL + h, lane, P[h]);
    }
#pragma unroll 1
    for (; tile < n_tiles; tile += stride) {
        LanePts Q[NPL];
#pragma unroll
        for (int h = 0; h < NPL; ++h) Q[h] = P[h];
        if (tile + stride < n_tiles) {
#pragma unroll
            for (int h = 0; h < NPL; ++h)
                load_lane_pts<D>(X, (tile + stride) * NPL + h, lane, Q[h]);
        }

        float best[NP];
        int bt[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            best[i] = pos_inf();
            bt[i] = 0;
        }
#pragma unroll kLargeUnroll
        for (int k0 = 0; k0 < Kp; k0 += kLargeKT) {
            float s[NP][kLargeKT];
#pragma unroll
            for (int u = 0; u < kLargeKT; ++u) {
                const float4 cc = cen[k0 + u];
#pragma unroll
                for (int h = 0; h < NPL; ++h) {
                    const float2 da = form_d2<D>(P[h].xa, P[h].ya, P[h].za, cc);
                    const float2 db = form_d2<D>(P[h].xb, P[h].yb, P[h].zb, cc);
                    s[4 * h + 0][u] = da.x;
                    s[4 * h + 1][u] = da.y;
                    s[4 * h + 2][u] = db.x;
                    s[4 * h + 3][u] = db.y;
                }
            }
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                const float m = min_tree<kLargeKT>(s[i], best[i]);
                bt[i] = (m < best[i]) ? k0 : bt[i];
                best[i] = m;
            }
        }
#pragma unroll
        for (int h = 0; h < NPL; ++h) {
            const float px[4] = {P[h].xa.x, P[h].xa.y, P[h].xb.x, P[h].xb.y};
            const float py[4] = {P[h].ya.x, P[h].ya.y, P[h].yb.x, P[h].yb.y};
            const float pz[4] = {P[h].za.x, P[h].za.y, P[h].zb.x, P[h].zb.y};
            int lab[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {   // lowest k of the winning step with d_k == best
                const int b0 = bt[4 * h + i];
                const float bv = best[4 * h + i];
                int l = b0 + kLargeKT;
#pragma unroll
                for (int u = kLargeKT - 1; u >= 0; --u) {
                    const float4 cc = cen[b0 + u];
                    const float e0 = __fadd_rn(px[i], cc.x), e1 = __fadd_rn(py[i], cc.y);
                    float d2 = __fmul_rn(e0, e0);
                    d2 = __fmaf_rn(e1, e1, d2);
                    if (D == 3) {
                        const float e2 = __fadd_rn(pz[i], cc.z);
                        d2 = __fmaf_rn(e2, e2, d2);
                    }
                    l = (d2 == bv) ? b0 + u : l;
                }
                KM_CHECK(l < K);
                lab[i] = l;
            }
            const int64_t pa = (tile * NPL + h) * kLaneTile + 2 * lane, pb = pa + kWarpTile;
            if (LAB) {
                *reinterpret_cast<int2*>(labels + pa) = make_int2(lab[0], lab[1]);
                *reinterpret_cast<int2*>(labels + pb) = make_int2(lab[2], lab[3]);
            }
            if (RED) {
                const bool v[4] = {pa < n, pa + 1 < n, pb < n, pb + 1 < n};
#pragma unroll
                for (int i = 0; i < 4; ++i) {   // slot i of every lane, sub-tile order
                    if (v[i]) J += (double)best[4 * h + i];
                    large_accum_slot<D>(v[i], lab[i], px[i], py[i], pz[i], myS, myN, lane);
                }
            }
        }
#pragma unroll
        for (int h = 0; h < NPL; ++h) P[h] = Q[h];
    }
    if (RED) large_block_row<D>(accS, accN, warpJ, J, K, W, tid, nthr, part);
}

// Second pass of the split large-K path: points + their labels -> the block
// rows.  J re-evaluates form D against the assigned centroid with the same RN
// operations as the argmin (bit-identical to its minimum); sums as in the
// fused kernel.  HBM-bound (16 or 12 B per point).
template <int D>
__global__ void __launch_bounds__(kLargeTPBMax)
k_accum_large(const float* __restrict__ X, int64_t n, int K, const double* __restrict__ mu_buf,
              const DevState* __restrict__ st, int mu_sel, int ignore_done,
              const int32_t* __restrict__ labels, double* __restrict__ part) {
    if (!ignore_done && st->done) return;
    const double* mu = mu_buf + (size_t)((st->t - mu_sel) & 1) * K * D;
    const int Kp = large_kpad(K);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, nthr = blockDim.x, W = nthr >> 5;
    const int lane = tid & 31, warp = tid >> 5;
    float4* cen = reinterpret_cast<float4*>(smem_raw);
    double* accS = reinterpret_cast<double*>(cen + Kp);
    int* accN = reinterpret_cast<int*>(accS + (size_t)W * K * D);
    double* warpJ = reinterpret_cast<double*>(accN + W * K + ((W * K) & 1));
    large_stage<D>(cen, mu, K, Kp, tid, nthr);
    for (int q = tid; q < W * K * D; q += nthr) accS[q] = 0.0;
    for (int q = tid; q < W * K; q += nthr) accN[q] = 0;
    __syncthreads();
    double* myS = accS + (size_t)warp * K * D;
    int* myN = accN + warp * K;
    double J = 0.0;
    const int64_t n_sub = (n + kLaneTile - 1) / kLaneTile;
    const int64_t stride = (int64_t)gridDim.x * W;
    int64_t sub = (int64_t)blockIdx.x * W + warp;
    LanePts P;
    int2 la = make_int2(0, 0), lb = make_int2(0, 0);
    auto fetch = [&](int64_t t, LanePts& Q, int2& qa, int2& qb) {
        load_lane_pts<D>(X, t, lane, Q);
        const int64_t pa = t * kLaneTile + 2 * lane;
        qa = __ldcs(reinterpret_cast<const int2*>(labels + pa));
        qb = __ldcs(reinterpret_cast<const int2*>(labels + pa + kWarpTile));
    };
    if (sub < n_sub) fetch(sub, P, la, lb);
#pragma unroll 1
    for (; sub < n_sub; sub += stride) {
        LanePts Q = P;
        int2 qa = la, qb = lb;
        if (sub + stride < n_sub) fetch(sub + stride, Q, qa, qb);
        const int64_t pa = sub * kLaneTile + 2 * lane, pb = pa + kWarpTile;
        const bool v[4] = {pa < n, pa + 1 < n, pb < n, pb + 1 < n};
        const int lab[4] = {la.x, la.y, lb.x, lb.y};
        const float px[4] = {P.xa.x, P.xa.y, P.xb.x, P.xb.y};
        const float py[4] = {P.ya.x, P.ya.y, P.yb.x, P.yb.y};
        const float pz[4] = {P.za.x, P.za.y, P.zb.x, P.zb.y};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int l = v[i] ? lab[i] : 0;
            KM_CHECK(l >= 0 && l < K);
            const float4 cc = cen[l];
            const float e0 = __fadd_rn(px[i], cc.x), e1 = __fadd_rn(py[i], cc.y);
            float d2 = __fmul_rn(e0, e0);
            d2 = __fmaf_rn(e1, e1, d2);
            if (D == 3) {
                const float e2 = __fadd_rn(pz[i], cc.z);
                d2 = __fmaf_rn(e2, e2, d2);
            }
            if (v[i]) J += (double)d2;
            large_accum_slot<D>(v[i], l, px[i], py[i], pz[i], myS, myN, lane);
        }
        P = Q;
        la = qa;
        lb = qb;
    }
    large_block_row<D>(accS, accN, warpJ, J, K, W, tid, nthr, part);
}

// ---------------------------------------------------------------------------
// k_stage: cneg[0][k] = -fl32(mu_k) (RN) from the fp64 master mu^t in buffer
// (t & 1); slot 1 (the previous iteration's) gets the same when `both`.
// ---------------------------------------------------------------------------
__global__ void k_stage(const double* __restrict__ mu_buf, const DevState* __restrict__ st,
                        int K, int d, float4* __restrict__ cneg, int both) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    const double* mu = mu_buf + (size_t)(st->t & 1) * K * d;
    float4 v;
    v.x = -__double2float_rn(mu[k * d + 0]);
    v.y = -__double2float_rn(mu[k * d + 1]);
    v.z = (d == 3) ? -__double2float_rn(mu[k * d + 2]) : 0.0f;
    v.w = 0.0f;
    cneg[k] = v;
    if (both) cneg[K + k] = v;
}

// ---------------------------------------------------------------------------
// k_merge: red[e] = sum_b part[e * G + b], one warp per entry, fixed order
// (lane l sums b = l, l+32, ... ascending; then a butterfly).
// ---------------------------------------------------------------------------
__global__ void k_merge(const double* __restrict__ part, int G, int nE,
                        double* __restrict__ red, const DevState* __restrict__ st,
                        int ignore_done) {
    if (!ignore_done && st->done) return;
    const int lane = threadIdx.x & 31;
    const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (e >= nE) return;
    const double* row = part + (size_t)e * G;
    double v = 0.0;
#pragma unroll 8
    for (int b = lane; b < G; b += 32) v += row[b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[e] = v;
}

// ---------------------------------------------------------------------------
// The update (one block): the mean step of PAPER.md:50-62 and the error term of
// PAPER.md:66-69; then t += 1 and the stop decision of PAPER.md:70.  `red` is
// the merged (and, distributed, allreduced) vector.
// ---------------------------------------------------------------------------
// E = sum_k sum_j (mu^{t+1} - mu^t)^2.  Up to kSerialE
// entries it is summed serially, k-major with j inner, without FMA
// contraction: the oracle's order, so E -- and the E < tol decision -- has the
// oracle's bits on every device path (k_fused_iterate and the persistent
// kernel sum the same way).  Beyond that (K > 170 in 3D) the serial chain of
// dependent fp64 adds costs ~9 ns per entry on the update's critical path
// (measured: +27 us per iteration at K = 1024), so every device path sums it
// in the same fixed tree instead (identical bits across paths; within a few
// ulps of the oracle's E).
constexpr int kSerialE = 512;

template <int D>
__device__ void update_body(double* __restrict__ mu_buf, int K, const double* red,
                            DevState* __restrict__ st, double* __restrict__ trace_E,
                            double* __restrict__ trace_J, int trace_cap,
                            float4* __restrict__ cneg) {
    __shared__ double e_sm[kSerialE];   // (kSerialE >= 256: the tree's partials too)
    const int t = st->t;
    const double* mu_old = mu_buf + (size_t)(t & 1) * K * D;
    double* mu_new = mu_buf + (size_t)((t + 1) & 1) * K * D;
    const int tid = threadIdx.x;
    const bool serial = K * D <= kSerialE;
    double e_acc = 0.0;
    for (int q = tid; q < K * D; q += blockDim.x) {
        const int k = q / D;
        const double nk = red[K * D + k];
        const double old = mu_old[q];
        const double nw = (nk > 0.0) ? red[q] / nk : old;   // empty cluster keeps mu^t
        mu_new[q] = nw;
        if (cneg) {   // staged fp32 copies: [1] <- mu^t, [0] <- mu^{t+1} (pruned path)
            const int j = q - k * D;
            reinterpret_cast<float*>(&cneg[K + k])[j] = -__double2float_rn(old);
            reinterpret_cast<float*>(&cneg[k])[j] = -__double2float_rn(nw);
        }
        if (serial) {
            const double diff = nw - old;
            e_sm[q] = __dmul_rn(diff, diff);   // no FMA contraction (oracle: -ffp-contract=off)
        }
    }
    double E = 0.0;
    if (serial) {
        __syncthreads();
        if (tid == 0) {
            const int n = K * D;
            int q = 0;
            for (; q + 8 <= n; q += 8) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = e_sm[q + u];
#pragma unroll
                for (int u = 0; u < 8; ++u) E = __dadd_rn(E, v[u]);
            }
            for (; q < n; ++q) E = __dadd_rn(E, e_sm[q]);
        }
    } else {
        // fixed tree independent of blockDim (>= 256 on every path): 256
        // strided partial sums in ascending q, then pairwise halving
        __syncthreads();   // mu_new written
        if (tid < 256) {
            for (int q = tid; q < K * D; q += 256) {
                const double diff = mu_new[q] - mu_old[q];
                e_acc = __dadd_rn(e_acc, __dmul_rn(diff, diff));
            }
            e_sm[tid] = e_acc;
        }
        __syncthreads();
        for (int h = 128; h > 0; h >>= 1) {
            if (tid < h) e_sm[tid] = __dadd_rn(e_sm[tid], e_sm[tid + h]);
            __syncthreads();
        }
        E = e_sm[0];
    }
    if (tid == 0) {
        const double J = red[K * D + K];
        st->E = E;
        st->J = J;
        if (t < trace_cap) {
            trace_E[t] = E;
            trace_J[t] = J;
        }
        st->t = t + 1;
        st->done = (E < st->tol) || (t + 1 >= st->max_iter);
    }
}

template <int D>
__global__ void k_update(double* __restrict__ mu_buf, int K, const double* __restrict__ red,
                         DevState* __restrict__ st, double* __restrict__ trace_E,
                         double* __restrict__ trace_J, int trace_cap,
                         float4* __restrict__ cneg) {
    if (st->done) return;
    update_body<D>(mu_buf, K, red, st, trace_E, trace_J, trace_cap, cneg);
}

// k_merge_update (single GPU): the group merge of k_merge and the update in one
// block -- warp w sums entries e = w, w + 32, ... over the groups in the fixed
// k_merge order (lane l: groups l, l + 32, ...; then a butterfly), into shared
// memory; then the update.  Saves a launch per iteration.
template <int D>
__global__ void __launch_bounds__(1024)
k_merge_update(const double* __restrict__ part, int G, int nE, double* __restrict__ red,
               double* __restrict__ mu_buf, int K, DevState* __restrict__ st,
               double* __restrict__ trace_E, double* __restrict__ trace_J, int trace_cap,
               float4* __restrict__ cneg) {
    pdl_trigger();
    pdl_wait();   // the group columns are written
    if (st->done) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* rs = reinterpret_cast<double*>(smem_raw);   // [nE]
    block_merge_groups(part, G, nE, rs, red);
    __syncthreads();
    update_body<D>(mu_buf, K, rs, st, trace_E, trace_J, trace_cap, cneg);
}


// ---------------------------------------------------------------------------
// k_fused_iterate (full-scan path, K <= 16, one GPU): up to n_iter whole Lloyd
// iterations in ONE cooperative launch -- for the small shards where an
// iteration is a few microseconds of work and launch latency dominates.
//
// Per iteration: warp w of the grid takes the 128-point warp-tiles w, w + W,
// ... (loads prefetched two tiles ahead; the data is L2-resident after the
// first iteration) and runs the same form-D distances, exact argmin and fused
// accumulation as k_assign_chunk into its lane columns,
// warps -> block row (fixed order) -> brow[t & 1][e][b]; one grid barrier;
// then EVERY block merges the G block rows in the k_merge order and applies
// the update (mu = S / n, empty keeps mu^t, E summed
// k-major in the oracle's order, stop rule) to its shared copy of mu -- the
// same bits in every block, so all blocks stop together and the next
// iteration needs no second barrier (brow is double-buffered by iteration
// parity).  Block 0 publishes mu^{t+1}, E, J, the traces and the state.
// ---------------------------------------------------------------------------
constexpr int kFusedWarps = 8;

template <int KP>
struct FusedSmem {
    double2 A[KP][32];   // {Sx, Sy} per (k, lane)
    double2 B[KP][32];   // {Sz, n|pad} per (k, lane)
};

template <int D, int KP>
__global__ void __launch_bounds__(kFusedWarps * 32, 1)
k_fused_iterate(const float* __restrict__ X, int64_t n, int K, int n_chunks,
                double* __restrict__ mu_buf, DevState* __restrict__ st,
                double* __restrict__ trace_E, double* __restrict__ trace_J, int trace_cap,
                double* __restrict__ brow, double* __restrict__ red, int n_iter) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, b = blockIdx.x;
    FusedSmem<KP>& S = reinterpret_cast<FusedSmem<KP>*>(smem_raw)[warp];
    double* wrow = reinterpret_cast<double*>(smem_raw + sizeof(FusedSmem<KP>) * kFusedWarps);
    double* mu_s = wrow + kFusedWarps * 66;   // [K*D] mu^t
    double* mu_n = mu_s + KP * D;             // [K*D] mu^{t+1}
    double* rs = mu_n + KP * D;               // [nE] merged vector
    __shared__ double sh_E;
    const int nE = K * D + K + 1;
    const int64_t ntiles = (n + kLaneTile - 1) / kLaneTile;   // 128-point warp-tiles
    const int64_t tw = (int64_t)G * kFusedWarps;              // warps in the grid
    const int64_t gw = (int64_t)b * kFusedWarps + warp;
    int t = st->t;
    bool done = st->done != 0;
    const int max_iter = st->max_iter;
    const double tol = st->tol;
    for (int q = tid; q < K * D; q += blockDim.x) mu_s[q] = mu_buf[(size_t)(t & 1) * K * D + q];
    __syncthreads();

    struct Pts {
        float2 xa, ya, za, xb, yb, zb;
    };
    auto load = [&](int64_t tile, Pts& P) {   // this lane's 4 points of a warp-tile
        const int64_t pa = tile * kLaneTile + 2 * lane, pb = pa + kWarpTile;
        P.xa = __ldg(reinterpret_cast<const float2*>(tile_coord<D>(X, pa, 0)));
        P.ya = __ldg(reinterpret_cast<const float2*>(tile_coord<D>(X, pa, 1)));
        P.za = (D == 3) ? __ldg(reinterpret_cast<const float2*>(tile_coord<D>(X, pa, 2)))
                        : make_float2(0.f, 0.f);
        P.xb = __ldg(reinterpret_cast<const float2*>(tile_coord<D>(X, pb, 0)));
        P.yb = __ldg(reinterpret_cast<const float2*>(tile_coord<D>(X, pb, 1)));
        P.zb = (D == 3) ? __ldg(reinterpret_cast<const float2*>(tile_coord<D>(X, pb, 2)))
                        : make_float2(0.f, 0.f);
    };
    auto accumulate = [&](int l, float px, float py, float pz) {
        double2 a = S.A[l][lane], c = S.B[l][lane];
        a.x += (double)px;
        a.y += (double)py;
        if (D == 3) c.x += (double)pz;
        int2 cn = *reinterpret_cast<int2*>(&c.y);
        cn.x += 1;
        c.y = *reinterpret_cast<double*>(&cn);
        S.A[l][lane] = a;
        S.B[l][lane] = c;
    };

    for (int it = 0; it < n_iter && !done; ++it) {
        // stage c_k = fl32(mu_k^t) (RN), negated; padded slots -inf (never win)
        float nc[KP][D];
#pragma unroll
        for (int k = 0; k < KP; ++k)
#pragma unroll
            for (int j = 0; j < D; ++j)
                nc[k][j] = (k < K) ? -__double2float_rn(mu_s[k * D + j]) : -pos_inf();
        zero_columns<KP>(S, lane);
        __syncwarp();
        double J = 0.0;
        // this warp's tiles gw, gw + tw, ... ascending; two tiles prefetched
        Pts P0, P1;
        if (gw < ntiles) load(gw, P0);
        if (gw + tw < ntiles) load(gw + tw, P1);
        for (int64_t tile = gw; tile < ntiles; tile += tw) {
            const Pts P = P0;
            P0 = P1;
            if (tile + 2 * tw < ntiles) load(tile + 2 * tw, P1);
            float da0[KP], da1[KP], db0[KP], db1[KP], m[4];
            int l[4];
            form_d_pair<D, KP>(nc, P.xa, P.ya, P.za, da0, da1);
            form_d_pair<D, KP>(nc, P.xb, P.yb, P.zb, db0, db1);
            exact_argmin<KP>(da0, m[0], l[0]);
            exact_argmin<KP>(da1, m[1], l[1]);
            exact_argmin<KP>(db0, m[2], l[2]);
            exact_argmin<KP>(db1, m[3], l[3]);
            const int64_t pa = tile * kLaneTile + 2 * lane, pb = pa + kWarpTile;
            if (pa < n) { accumulate(l[0], P.xa.x, P.ya.x, P.za.x); J += (double)m[0]; }
            if (pa + 1 < n) { accumulate(l[1], P.xa.y, P.ya.y, P.za.y); J += (double)m[1]; }
            if (pb < n) { accumulate(l[2], P.xb.x, P.yb.x, P.zb.x); J += (double)m[2]; }
            if (pb + 1 < n) { accumulate(l[3], P.xb.y, P.yb.y, P.zb.y); J += (double)m[3]; }
        }
        __syncwarp();
        const double2 out = columns_to_row<KP>(S, lane);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) J += __shfl_xor_sync(0xffffffffu, J, o);
        reinterpret_cast<double2*>(wrow + warp * 66)[lane] = out;
        if (lane == 0) wrow[warp * 66 + 64] = J;
        __syncthreads();
        // block row -> brow[t & 1][e][b] (warps in order)
        double* bp = brow + (size_t)(t & 1) * nE * G;
        if (tid < 65) {
            const int k = tid >> 2, q = tid & 3;
            int e = -1;
            if (tid == 64) e = K * D + K;
            else if (k < K && q < D) e = k * D + q;
            else if (k < K && q == 3) e = K * D + k;
            if (e >= 0) {
                double v = 0.0;
#pragma unroll
                for (int w = 0; w < kFusedWarps; ++w) v += wrow[w * 66 + tid];
                bp[(size_t)e * G + b] = v;
            }
        }
        grid.sync();
        // every block: the merged vector (k_merge order) and the update
        // one pass: every entry's loads in flight at once (nE <= 8 R)
        block_merge_groups<(KP * (D + 1) + 1 + kFusedWarps - 1) / kFusedWarps>(
            bp, G, nE, rs, b == 0 ? red : nullptr);
        __syncthreads();
        for (int q = tid; q < K * D; q += blockDim.x) {
            const double nk = rs[K * D + q / D];
            mu_n[q] = (nk > 0.0) ? rs[q] / nk : mu_s[q];   // empty cluster keeps mu^t
        }
        __syncthreads();
        if (tid == 0) {
            double E = 0.0;   // k-major, j inner: the oracle's order
            for (int q = 0; q < K * D; ++q) {
                const double dlt = mu_n[q] - mu_s[q];
                E = __dadd_rn(E, __dmul_rn(dlt, dlt));   // no FMA contraction
            }
            sh_E = E;
        }
        __syncthreads();
        const double E = sh_E, Jt = rs[K * D + K];
        if (b == 0) {
            for (int q = tid; q < K * D; q += blockDim.x)
                mu_buf[(size_t)((t + 1) & 1) * K * D + q] = mu_n[q];
            if (tid == 0) {
                if (t < trace_cap) {
                    trace_E[t] = E;
                    trace_J[t] = Jt;
                }
                st->E = E;
                st->J = Jt;
                st->t = t + 1;
                st->done = (E < tol) || (t + 1 >= max_iter);
            }
        }
        for (int q = tid; q < K * D; q += blockDim.x) mu_s[q] = mu_n[q];
        t += 1;
        done = (E < tol) || (t >= max_iter);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// P2P exchange (multi-GPU): the allreduce of the K(d+1)+1
// partials as one kernel over peer memory instead of a collective library call.
// Every rank owns an exchange buffer in its own HBM, mapped into every peer
// (CUDA IPC over NVLink): xb[slot][P][cap] doubles and xf[slot][P] epochs.
// Rank r stores its vector into xb[slot][r] of EVERY rank (remote stores),
// fences at system scope, then publishes `epoch` in xf[slot][r] of every rank
// (st.release.sys); it waits until its own xf[slot][q] == epoch for all q
// (ld.acquire.sys) and sums xb[slot][0..P-1] in rank order -- the same bits on
// every rank.  Slots alternate with the exchange parity, so a rank can only
// overwrite a slot after every peer has published the next exchange, i.e.
// finished reading that slot.  Epochs are unique per exchange (generation,
// iteration) so stale flags never match.
// ---------------------------------------------------------------------------
constexpr int kXSlots = 4;   // 0/1: iteration exchanges (parity of t), 2/3: host-driven ones

struct P2PView {
    double* const* xb;       // [P] exchange buffers (index rank = own)
    uint64_t* const* xf;     // [P] epoch flags
    int P, rank, cap;
    uint64_t timeout_ns;     // bound on the wait for a peer's epoch (0 = none)
};

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Block-wide: out[i] = sum over ranks q (ascending) of rank q's local[i], i < n.
// `out` may alias `local` (local is fully sent before out is written).
// Returns false (the same in every thread; out untouched) when some peer's
// epoch did not arrive within v.timeout_ns -- a dead or hung rank fails the
// exchange instead of hanging this one forever.
__device__ bool p2p_exchange(const P2PView& v, const double* local, int n, int slot, uint64_t epoch,
                             double* out) {
    __shared__ int s_late;
    const int tid = threadIdx.x;
    if (tid == 0) s_late = 0;
    for (int i = tid; i < n; i += blockDim.x) {
        const double x = local[i];
        for (int q = 0; q < v.P; ++q) v.xb[q][((size_t)slot * v.P + v.rank) * v.cap + i] = x;
    }
    __threadfence_system();
    __syncthreads();
    if (tid < v.P) st_release_sys(&v.xf[tid][slot * v.P + v.rank], epoch);
    if (tid < v.P) {
        const uint64_t* f = &v.xf[v.rank][slot * v.P + tid];
        const uint64_t t0 = v.timeout_ns ? global_ns() : 0;
        while (ld_acquire_sys(f) != epoch) {
            if (v.timeout_ns && global_ns() - t0 > v.timeout_ns) {
                s_late = 1;
                break;
            }
            __nanosleep(64);
        }
    }
    __threadfence_system();
    __syncthreads();
    if (s_late) return false;
    const double* mine = v.xb[v.rank] + (size_t)slot * v.P * v.cap;
    for (int i = tid; i < n; i += blockDim.x) {
        double s = 0.0;
        for (int q = 0; q < v.P; ++q) s += __ldcv(mine + (size_t)q * v.cap + i);
        out[i] = s;
    }
    __syncthreads();
    return true;
}

__device__ __forceinline__ uint64_t iter_epoch(const DevState* st) {
    return ((uint64_t)(unsigned)(st->gen & 0x7fffffff) << 32) | (uint64_t)(unsigned)(st->t + 1);
}

// A failed exchange stops the run: err records it, done turns every later
// kernel of the iteration into a no-op; the host reports KMEANS_ENCCL.
__device__ __forceinline__ void exchange_failed(DevState* st) {
    if (threadIdx.x == 0) {
        st->err = kErrExchangeTimeout;
        st->done = 1;
    }
}

// Host-driven exchange (mu^0 assembly, kmeans_assign): buf <- sum over ranks.
__global__ void k_p2p_allreduce(P2PView v, double* buf, int n, int slot, uint64_t epoch,
                                DevState* st) {
    if (!p2p_exchange(v, buf, n, slot, epoch, buf)) exchange_failed(st);
}

// The iteration's exchange fused with the update: red <- sum over ranks of the
// local merged vector, then the update of k_update (one block).
// part != nullptr: the group merge (k_merge's order) is done here first, by the
// same block -- one kernel for merge + exchange + update when G x nE is small.
template <int D>
__global__ void k_p2p_update(P2PView v, double* __restrict__ red, int nE, double* __restrict__ mu_buf,
                             int K, DevState* __restrict__ st, double* __restrict__ trace_E,
                             double* __restrict__ trace_J, int trace_cap, float4* __restrict__ cneg,
                             const double* __restrict__ part, int G) {
    if (st->done) return;
    if (part) {
        extern __shared__ __align__(16) unsigned char smem_raw[];
        block_merge_groups(part, G, nE, reinterpret_cast<double*>(smem_raw), red);
        __threadfence_block();
        __syncthreads();
    }
    if (!p2p_exchange(v, red, nE, st->t & 1, iter_epoch(st), red)) {
        exchange_failed(st);
        return;
    }
    __threadfence();
    __syncthreads();
    update_body<D>(mu_buf, K, red, st, trace_E, trace_J, trace_cap, cneg);
}

// One-GPU emulation of P ranks for the tests (PROFILING guide: ranks that wait
// on one another must not be separate launches on one GPU): ONE cooperative
// launch, block r = rank r, each with its own exchange buffer in this GPU's
// memory.  Round i: rank r contributes vals[i][r][0..n) and writes what it
// received to out[i][r][0..n).  dead_rank (>= 0) never publishes: the others
// must time out (failed[r] = round + 1) instead of hanging.
__global__ void k_p2p_emulate(double* const* xb, uint64_t* const* xf, int P, int cap, int n,
                              int rounds, const double* __restrict__ vals, double* __restrict__ out,
                              double* __restrict__ scratch, int dead_rank, uint64_t timeout_ns,
                              int* __restrict__ failed, uint64_t epoch_base) {
    P2PView v{xb, xf, P, (int)blockIdx.x, cap, timeout_ns};
    double* loc = scratch + (size_t)blockIdx.x * cap;
    if ((int)blockIdx.x == dead_rank) return;   // a rank that never publishes
    for (int i = 0; i < rounds; ++i) {
        for (int e = threadIdx.x; e < n; e += blockDim.x)
            loc[e] = vals[((size_t)i * P + blockIdx.x) * n + e];
        __syncthreads();
        if (!p2p_exchange(v, loc, n, 2 + (i & 1), epoch_base + (uint64_t)i + 1, loc)) {
            if (threadIdx.x == 0) failed[blockIdx.x] = i + 1;   // round of the failure
            return;
        }
        for (int e = threadIdx.x; e < n; e += blockDim.x)
            out[((size_t)i * P + blockIdx.x) * n + e] = loc[e];
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// k_generate: the synthetic Gaussian-mixture points of
// DESIGN.md "Inputs" ("mixture of Bivariate Gaussian
// Distributions"), generated in HBM by the same counter-based recipe as
// paper_2405_12052_b200/datagen.py (an independent implementation of it):
//   u(i, s) = mix64(mix64(seed) + (8 i + s + 1) * golden) >> 11, times 2^-53
//   blob    = min(floor(u(i,0) M), M - 1)
//   n0, n1  = Box-Muller(u(i,1), u(i,2)); n2 = Box-Muller cos part of (u(i,3), u(i,4))
//   x_ij    = fp32(center[blob][j] + sigma n_j)            (fp64, one rounding)
// planted duplicates (C5): point g (N / G) + q, q < r, is site g.  Points
// [start, start + count) of the dataset, AoS.  The fp64 log1p / cos / sin may
// differ from the host libm by an ulp, which moves an fp32 result by one ulp
// in rare cases (bounded in the tests).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t mix64_dev(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

__global__ void k_generate(uint64_t key, int d, int M, const double* __restrict__ centers,
                           double sigma, int G, int r, const double* __restrict__ sites,
                           int64_t N, int64_t start, int64_t count, float* __restrict__ out) {
    constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += stride) {
        const int64_t i = start + t;
        auto U = [&](int s_) {
            const uint64_t z = mix64_dev(key + ((uint64_t)i * 8ull + (uint64_t)s_ + 1ull) * kGolden);
            return (double)(z >> 11) * (1.0 / 9007199254740992.0);
        };
        int blob = (int)(U(0) * (double)M);
        blob = blob < M - 1 ? blob : M - 1;
        const double u1 = U(1), u2 = U(2);
        const double rr = sqrt(__dmul_rn(-2.0, log1p(-u1)));
        const double th = __dmul_rn(2.0 * 3.141592653589793, u2);
        double col[3];
        col[0] = __dmul_rn(rr, cos(th));
        col[1] = __dmul_rn(rr, sin(th));
        if (d > 2) {
            const double u3 = U(3), u4 = U(4);
            col[2] = __dmul_rn(sqrt(__dmul_rn(-2.0, log1p(-u3))),
                               cos(__dmul_rn(2.0 * 3.141592653589793, u4)));
        }
        int site = -1;
        if (G > 0) {
            const int64_t st_ = N / G;
            const int64_t g = i / st_, q = i - g * st_;
            if (g < G && q < r) site = (int)g;
        }
        for (int j = 0; j < d; ++j) {
            // mul then add, each rounded (no FMA contraction), as on the host
            const double v = (site >= 0) ? sites[site * d + j]
                                         : __dadd_rn(centers[blob * d + j], __dmul_rn(sigma, col[j]));
            out[t * d + j] = (float)v;
        }
    }
}

}  // namespace km
