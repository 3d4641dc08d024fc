// persist.cuh -- the sorted-path Lloyd iteration as ONE persistent kernel
// ("one kernel per iteration, no host in the loop";
// reassignment, mean, error, stop rule -- and PAPER.md:97-99,
// the merge of the threads' partials into the global variable and the master
// update).
//
// k_persist_iterate runs up to n_iter whole iterations of the sorted small-K
// path (K <= 16) in one cooperative launch, one block of W warps per SM:
//
//   * work: chunk c belongs to warp c mod TW (TW = warps in the grid), every
//     iteration -- a static round-robin, no atomics; a warp's chunks of all
//     iterations form ONE continuous stream of 256-point TMA units through
//     its ring, so the next chunk's (and the next iteration's) first units
//     are in flight while the current one is computed (the points do not
//     depend on the centroids).  Each chunk runs small_chunk -- the same
//     candidates, form D, exact argmin and fused sums as k_assign_pruned --
//     and adds its entries to the warp's dense table in shared memory
//     (chunks in the warp's fixed order; no per-chunk global traffic).
//   * merge, no grid barrier: the last warp of a block to finish (shared-
//     memory counter) sums the block's warp tables in warp order into the
//     block's column; the last block to finish (one global atomic per block
//     and iteration) sums the block columns in block order into the vector,
//     runs the exchange over peer memory when the context is one rank of a
//     P2P group (k_p2p_update's protocol), the update (mu = S / n, empty keeps
//     mu^t, E serially k-major, J, stop flag) and the staging of
//     -fl32(mu^{t+1}), then releases the iteration flag that every other warp
//     waits on before its next chunk's candidates.
//
// Status: correct (parity-tested against the oracle and the graph path) but
// OPT-IN (KMEANS_FLAG_PERSIST): measured slower than the per-iteration kernel
// graph at every shard size (tools/sweep.py):
//   * the static partition cannot balance: a warp whose range crosses Voronoi
//     boundaries (2-candidate chunks) is slower EVERY iteration, and the
//     iteration waits for it, whereas the graph's one-warp CTAs are balanced
//     by the hardware scheduler (no-wait timing experiment KM_PERSIST_NOWAIT:
//     1.25e7 points 43.6 us vs the assign kernel's 29 us);
//   * even balanced (K = 4 at N = 1e8, 1.01 candidates per chunk) the stream
//     is ~15% slower (191 vs 166 us): 20 warps per SM keep fewer bytes in
//     flight than 28 one-warp CTAs, and 28 warps in one block spill;
//   * the iteration's hand-off (block / group / grid last arrivers, update,
//     flag) costs ~14 us against the graph's kernel boundaries.
// Earlier designs measured on the way: dynamic chunk tickets with per-chunk
// rows and a gpu-scope fence + atomic per chunk (2.4x slower: the fences),
// and a single-warp final merge of every block column (~20 us per iteration:
// one warp's L2 round trips).
//
// Sums are taken in a fixed order at every level (chunk: lanes + butterfly;
// warp: chunks in order; block: warps in order; grid: blocks in order), so a
// run is bit-reproducible; the order differs from the multi-kernel path's,
// within reading R13's bar of the oracle.
#pragma once

namespace km {

constexpr int kBlockGroup = 16;   // block columns per group column (merge level 2)
constexpr int kMaxBlockGroups = 32;

struct PersistSync {
    unsigned long long flag;          // iterations completed in this launch (host-zeroed)
    int fcount[2];                    // block groups done, by iteration parity
    int gcount[2][kMaxBlockGroups];   // blocks of each group done, by iteration parity
};

__device__ __forceinline__ void st_release_gpu(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Warp-level P2P exchange (p2p_exchange's protocol, one warp): out[i] = sum
// over ranks q ascending of rank q's local[i].  false on a peer timeout.
__device__ bool p2p_exchange_warp(const P2PView& v, const double* local, int n, int slot,
                                  uint64_t epoch, double* out) {
    const int lane = threadIdx.x & 31;
    for (int i = lane; i < n; i += 32) {
        const double x = local[i];
        for (int q = 0; q < v.P; ++q) v.xb[q][((size_t)slot * v.P + v.rank) * v.cap + i] = x;
    }
    __threadfence_system();
    __syncwarp();
    bool late = false;
    for (int q = lane; q < v.P; q += 32) st_release_sys(&v.xf[q][slot * v.P + v.rank], epoch);
    for (int q = lane; q < v.P; q += 32) {
        const uint64_t* f = &v.xf[v.rank][slot * v.P + q];
        const uint64_t t0 = v.timeout_ns ? global_ns() : 0;
        while (ld_acquire_sys(f) != epoch) {
            if (v.timeout_ns && global_ns() - t0 > v.timeout_ns) {
                late = true;
                break;
            }
            __nanosleep(64);
        }
    }
    if (__any_sync(0xffffffffu, late)) return false;
    __threadfence_system();
    const double* mine = v.xb[v.rank] + (size_t)slot * v.P * v.cap;
    for (int i = lane; i < n; i += 32) {
        double s = 0.0;
        for (int q = 0; q < v.P; ++q) s += __ldcv(mine + (size_t)q * v.cap + i);
        out[i] = s;
    }
    __syncwarp();
    return true;
}

// One warp: out[e][oc] = sum over columns g in [g0, g1) ascending of
// in[e][g] (lane l takes entries e = l, l + 32, l + 64; nE <= 65 for K <= 16).
__device__ __forceinline__ void merge_cols_warp(const double* __restrict__ in, int Gin, int g0,
                                                int g1, int nE, double* __restrict__ out,
                                                int Gout, int oc) {
    const int lane = threadIdx.x & 31;
    for (int e = lane; e < nE; e += 32) {
        const double* col = in + (size_t)e * Gin;
        double v = 0.0;
        int g = g0;
        for (; g + 8 <= g1; g += 8) {
            double a[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] = __ldcg(col + g + u);
#pragma unroll
            for (int u = 0; u < 8; ++u) v += a[u];
        }
        for (; g < g1; ++g) v += __ldcg(col + g);
        out[(size_t)e * Gout + oc] = v;
    }
}

// The last warp of the iteration: [exchange,] the update of PAPER.md:50-70 on
// the merged vector red.  Returns false if the exchange failed (then err and
// done are set).
template <int D>
__device__ bool update_warp(int K, double* __restrict__ red, double* __restrict__ mu_buf,
                            float4* __restrict__ cneg, DevState* __restrict__ st,
                            double* __restrict__ trace_E, double* __restrict__ trace_J,
                            int trace_cap, int t, double* __restrict__ T, const P2PView& pv) {
    const int lane = threadIdx.x & 31;
    const int nE = K * D + K + 1;
    __threadfence();
    __syncwarp();
    if (pv.xb) {   // distributed (P2P group, any P): the sum over ranks
        if (!p2p_exchange_warp(pv, red, nE, t & 1,
                               ((uint64_t)(unsigned)(st->gen & 0x7fffffff) << 32) |
                                   (uint64_t)(unsigned)(t + 1),
                               red)) {
            if (lane == 0) {
                st->err = kErrExchangeTimeout;
                st->done = 1;
            }
            return false;
        }
        __threadfence();
        __syncwarp();
    }
    const double* mu_old = mu_buf + (size_t)(t & 1) * K * D;
    double* mu_new = mu_buf + (size_t)((t + 1) & 1) * K * D;
    for (int q = lane; q < K * D; q += 32) {   // K * D <= 48 <= 64 slots of T
        const int k = q / D, j = q - k * D;
        const double nk = __ldcg(red + K * D + k);
        const double old = mu_old[q];
        const double nw = (nk > 0.0) ? __ldcg(red + q) / nk : old;   // empty keeps mu^t
        mu_new[q] = nw;
        reinterpret_cast<float*>(&cneg[K + k])[j] = -__double2float_rn(old);
        reinterpret_cast<float*>(&cneg[k])[j] = -__double2float_rn(nw);
        const double diff = nw - old;
        T[q] = __dmul_rn(diff, diff);
    }
    __syncwarp();
    if (lane == 0) {
        double E = 0.0;   // serially, k-major: the oracle's order
        for (int q = 0; q < K * D; ++q) E = __dadd_rn(E, T[q]);
        const double J = __ldcg(red + K * D + K);
        st->E = E;
        st->J = J;
        if (t < trace_cap) {
            trace_E[t] = E;
            trace_J[t] = J;
        }
        st->t = t + 1;
        st->done = (E < st->tol) || (t + 1 >= st->max_iter);
    }
    __syncwarp();
    return true;
}

#ifndef KM_PERSIST_WARPS_3D
#define KM_PERSIST_WARPS_3D 20   // measured: 28 / 24 / 20 -> 20 best (28 and 24 spill)
#endif
#ifndef KM_PERSIST_WARPS_2D
#define KM_PERSIST_WARPS_2D 20
#endif
template <int D>
struct PersistCfg {
    static constexpr int kWarps = D == 2 ? KM_PERSIST_WARPS_2D : KM_PERSIST_WARPS_3D;
};

// Counter increment with release semantics after every lane's stores; returns
// (warp-uniform) whether this warp is the last of `total` arrivals, in which
// case it resets the counter (for the iteration two ahead) and acquires.
__device__ __forceinline__ bool arrive_last(int* counter, int total) {
    __threadfence();   // every lane's stores before the count (release)
    __syncwarp();
    int last = 0;
    if ((threadIdx.x & 31) == 0) {
        last = atomicAdd(counter, 1) == total - 1;
        if (last) *counter = 0;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) __threadfence();   // acquire: the other arrivals' stores
    return last;
}

constexpr int kAccStride = 72;   // doubles per warp table: [16][4] + J, padded

// bcol: block columns [nE][gridDim.x]; gcol: block-group columns [nE][kMaxBlockGroups].
template <int D, int CHT>
__global__ void __launch_bounds__(PersistCfg<D>::kWarps * 32, 1)
k_persist_iterate(const float* __restrict__ X, int64_t n, int K, int n_chunks,
                  const float* __restrict__ cbox, float4* __restrict__ cneg,
                  double* __restrict__ mu_buf, DevState* __restrict__ st,
                  double* __restrict__ trace_E, double* __restrict__ trace_J, int trace_cap,
                  double* __restrict__ bcol, double* __restrict__ gcol, double* __restrict__ red,
                  PersistSync* __restrict__ ps, int64_t keep_n, int n_iter, P2PView pv) {
    constexpr int W = PersistCfg<D>::kWarps;
    constexpr int SS = kSortedStages;
    constexpr int CHP = CHT * kLaneTile, CHU = CHP / kSortedUnit;
    constexpr int kUnitFloats = D * kSortedUnit;
    constexpr unsigned kUnitBytes = kUnitFloats * 4;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int bcount[2];   // warps of this block done, by iteration parity
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) bcount[0] = bcount[1] = 0;
    __syncthreads();
    PrunedSmem<D, false>& S = reinterpret_cast<PrunedSmem<D, false>*>(smem_raw)[warp];
    double* acc_all = reinterpret_cast<double*>(smem_raw + W * sizeof(PrunedSmem<D, false>));
    double* acc = acc_all + warp * kAccStride;
    const int TW = gridDim.x * W;
    const int gw = blockIdx.x * W + warp;
    // static partition of the shard's 256-point units: warp gw owns the
    // contiguous range [ua, ub) (sizes differ by at most one unit), the same
    // every iteration; a range crossing chunk boundaries is processed as one
    // segment per chunk, each pruned with its chunk's box
    const int64_t U = (n + kSortedUnit - 1) / kSortedUnit;
    const int64_t ua = U * gw / TW, ub = U * (gw + 1) / TW;
    const unsigned upi = (unsigned)(ub - ua);   // units per iteration of this warp
    // (the host launches this kernel only when U >= TW: every warp owns a unit)
    const int G = gridDim.x;
    const int nE = K * D + K + 1;
    KM_CHECK(upi >= 1);
    const int t0 = *(volatile int*)&st->t;
    if (*(volatile int*)&st->done) return;
    // iterations this launch may run (the stop rule can end it earlier)
    const int n_run = min(n_iter, st->max_iter - t0);
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < SS; ++s) mbar_init(&S.bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const uint64_t pol_first = l2_policy_evict_first(), pol_last = l2_policy_evict_last();
    const unsigned n_units = upi * (unsigned)n_run;   // the stream of the whole launch

    // ---- the warp's unit stream: stream unit u = shard unit ua + u % upi of
    // iteration u / upi; lane 0 issues ----
    unsigned issued = 0, consumed = 0;
    auto issue_one = [&]() {
        if (issued >= n_units) return;   // nothing past the launch's last iteration
        if (lane == 0) {
            const int64_t su = ua + issued % upi;   // shard unit (units are contiguous)
            const int s = issued % SS;
            mbar_expect_tx(&S.bar[s], kUnitBytes);
            bulk_g2s_pol(S.ring_at(s), X + su * kUnitFloats, kUnitBytes, &S.bar[s],
                         su * kSortedUnit < keep_n ? pol_last : pol_first);
        }
        ++issued;
    };
    auto drain = [&]() {   // wait for the units in flight (before leaving early)
        for (unsigned u = consumed; u < issued; ++u) mbar_wait(&S.bar[u % SS], (u / SS) & 1u);
        consumed = issued;
    };
    for (int s = 0; s < SS; ++s) issue_one();

    for (int it = 0; it < n_run; ++it) {
        const int t = t0 + it;
#ifndef KM_PERSIST_NOWAIT
#define KM_PERSIST_NOWAIT 0   // timing experiment only: never wait for the update (wrong results)
#endif
        if (it > 0 && !KM_PERSIST_NOWAIT) {   // centroids of iteration t published?
            // bounded: a bug or a dead peer must not hang the GPU (the flag's
            // writer itself waits at most pv.timeout_ns in the exchange)
            const uint64_t w0 = global_ns();
            const uint64_t wmax = (pv.timeout_ns > 10000000000ull ? pv.timeout_ns : 10000000000ull) +
                                  1000000000ull;
            while (ld_acquire_gpu(&ps->flag) < (unsigned long long)it) {
                if (global_ns() - w0 > wmax) {
                    if (lane == 0) {
                        st->err = kErrIterationTimeout;
                        st->done = 1;
                    }
                    drain();
                    return;
                }
                __nanosleep(200);
            }
            __threadfence();
            if (*(volatile int*)&st->done) {
                drain();
                return;
            }
        }
        const float4 cl = (lane < K) ? __ldcg(&cneg[lane]) : make_float4(0.f, 0.f, 0.f, 0.f);
        for (int q = lane; q < kAccStride; q += 32) acc[q] = 0.0;
        __syncwarp();
        for (int64_t sa = ua; sa < ub;) {   // one segment per chunk touched
            const int c = (int)(sa / CHU);
            const int64_t sb = min(ub, (int64_t)(c + 1) * CHU);
            const int64_t base = sa * kSortedUnit;
            const int64_t rem = n - base;
            const int nunit = (int)(sb - sa);
            const int npts = rem < (int64_t)nunit * kSortedUnit ? (int)rem : nunit * kSortedUnit;
            const float bx = (lane < 2 * D) ? __ldg(&cbox[(size_t)c * 2 * D + lane]) : 0.0f;
            const unsigned u0 = consumed;   // the segment's first unit in the stream
            auto fetch = [&](unsigned q, LanePts (&P)[kUnitSub]) {
                const unsigned u = u0 + q;
                const int s = u % SS;
                mbar_wait(&S.bar[s], (u / SS) & 1u);
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
                issue_one();   // the stage just read takes the stream's next unit
            };
            small_chunk<D, kModeReduce, true>(S, lane, K, cl, bx, base, n, nunit, npts, nullptr,
                                              nullptr, nullptr, fetch, acc);
            consumed = u0 + nunit;
            sa = sb;
            __syncwarp();
        }
        // ---- the block's last warp: warp tables (in warp order) -> block column ----
        __threadfence_block();
        int last = 0;
        if (lane == 0) {
            last = atomicAdd(&bcount[t & 1], 1) == W - 1;
            if (last) bcount[t & 1] = 0;
        }
        if (!__shfl_sync(0xffffffffu, last, 0)) continue;
        __threadfence_block();
        for (int e = lane; e < nE; e += 32) {
            // e -> table slot: S_kj at 4 k + j, n_k at 4 k + 3, J at 64
            const int q = e < K * D ? 4 * (e / D) + e % D : (e < K * D + K ? 4 * (e - K * D) + 3 : 64);
            double v = 0.0;
            for (int w = 0; w < W; ++w) v += acc_all[w * kAccStride + q];
            bcol[(size_t)e * G + blockIdx.x] = v;
        }
        // ---- the last block of a group of kBlockGroup: block columns -> group column ----
        const int grp = blockIdx.x / kBlockGroup;
        const int b0 = grp * kBlockGroup, b1 = min(G, b0 + kBlockGroup);
        if (!arrive_last(&ps->gcount[t & 1][grp], b1 - b0)) continue;
        merge_cols_warp(bcol, G, b0, b1, nE, gcol, kMaxBlockGroups, grp);
        // ---- the last group: group columns (ascending) -> the vector, the update, the flag ----
        const int ngrp = (G + kBlockGroup - 1) / kBlockGroup;
        if (!arrive_last(&ps->fcount[t & 1], ngrp)) continue;
        merge_cols_warp(gcol, kMaxBlockGroups, 0, ngrp, nE, red, 1, 0);
        update_warp<D>(K, red, mu_buf, cneg, st, trace_E, trace_J, trace_cap, t, S.T, pv);
        __threadfence();   // mu^{t+1}, the staged centroids, the state ...
        __syncwarp();
        if (lane == 0) st_release_gpu(&ps->flag, (unsigned long long)(it + 1));   // ... then the flag
    }
    drain();
}

}  // namespace km
