// runtime.cu -- host runtime (kmeans_ctx) and the C ABI of include/kmeans.h.
//
// One context = one GPU's shard of the points, resident in HBM as padded SoA
// fp32, plus the iteration state (mu ping-pong buffers, per-block partials,
// merged partials, DevState, E/J traces).  One Lloyd iteration is captured once
// into a CUDA graph [assign+reduce -> merge -> (NCCL allreduce) -> update] and
// replayed; the stop rule lives on the device (DevState::done), so the host only
// polls between graph replays.
#include <type_traits>
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <climits>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <unordered_map>
#include <string>
#include <thread>
#include <vector>

#ifdef KMEANS_WITH_NCCL
#include <nccl.h>
#endif

#include "../../include/kmeans.h"
#include "kernels.cuh"
#include "persist.cuh"

using km::DevState;

// ---------------------------------------------------------------------------
// Device memory: a per-device cache of freed blocks in front of cudaMalloc
// (like a caching allocator).  Blocks are returned to the cache only when idle
// (every free site has synchronised the context's stream first), so a later
// create reuses them without paying cudaMalloc / cudaFree of gigabytes again.
// A failed cudaMalloc flushes the cache and retries; kmeans_release_memory
// gives the cached blocks back to the driver.
// ---------------------------------------------------------------------------
namespace {
constexpr int kMaxDevices = 64;
std::mutex g_mem_mu;
std::multimap<size_t, void*> g_cache[kMaxDevices];   // size -> idle block
struct Live {
    int dev;
    size_t size;    // block size (cache key)
    size_t bytes;   // requested bytes (KM_CHECKS: the red zone starts here)
};
std::unordered_map<void*, Live> g_live;   // block -> owner

#ifndef KM_CHECKS
#define KM_CHECKS 0
#endif
// KM_CHECKS builds: every block carries a kRedZone-byte red zone right after
// the requested bytes, filled with 0xA5 at allocation and verified when the
// block is freed (the owner synchronised its stream first): a kernel writing
// past the end of a buffer aborts the process with the buffer named by size.
constexpr size_t kRedZone = KM_CHECKS ? 4096 : 0;

size_t round_block(size_t bytes) {
    const size_t g = bytes >= (1u << 20) ? (2u << 20) : 512;
    return (bytes + g - 1) / g * g;
}

void flush_cache_locked(int dev) {
    for (auto& kv : g_cache[dev]) cudaFree(kv.second);
    g_cache[dev].clear();
}

void arm_red_zone(void* p, size_t bytes) {
    if (!kRedZone) return;
    cudaMemset(static_cast<char*>(p) + bytes, 0xA5, kRedZone);
    cudaDeviceSynchronize();   // (legacy stream; checked builds only)
}

void check_red_zone(void* p, const Live& l) {
    if constexpr (kRedZone == 0) return;
    std::vector<unsigned char> h(kRedZone);
    if (cudaMemcpy(h.data(), static_cast<char*>(p) + l.bytes, kRedZone, cudaMemcpyDeviceToHost) !=
        cudaSuccess) {
        cudaGetLastError();
        return;
    }
    for (size_t i = 0; i < h.size(); ++i)
        if (h[i] != 0xA5) {
            fprintf(stderr, "KM_CHECKS: device buffer of %zu bytes overrun at byte %zu past its end\n",
                    l.bytes, i);
            abort();
        }
}

cudaError_t cached_malloc(int dev, void** p, size_t bytes) {
    *p = nullptr;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    const size_t sz = round_block((bytes ? bytes : 1) + kRedZone);
    std::lock_guard<std::mutex> lk(g_mem_mu);
    auto& c = g_cache[dev];
    auto it = c.lower_bound(sz);
    if (it != c.end() && it->first <= sz + sz / 4 + (8u << 20)) {   // close fit only
        *p = it->second;
        g_live[*p] = {dev, it->first, bytes};
        c.erase(it);
        arm_red_zone(*p, bytes);
        return cudaSuccess;
    }
    cudaError_t e = cudaMalloc(p, sz);
    if (e != cudaSuccess) {   // give the cache back and retry once
        cudaGetLastError();
        flush_cache_locked(dev);
        e = cudaMalloc(p, sz);
    }
    if (e == cudaSuccess) {
        g_live[*p] = {dev, sz, bytes};
        arm_red_zone(*p, bytes);
    }
    return e;
}

// Pinned host blocks for the device state mirror (one per context):
// cudaMallocHost / cudaFreeHost synchronise the device and page-lock memory,
// milliseconds per create / destroy, so idle blocks are kept for the next one.
std::vector<void*> g_pinned_state;

cudaError_t pinned_state_get(void** p, size_t bytes) {
    {
        std::lock_guard<std::mutex> lk(g_mem_mu);
        if (!g_pinned_state.empty()) {
            *p = g_pinned_state.back();
            g_pinned_state.pop_back();
            return cudaSuccess;
        }
    }
    return cudaMallocHost(p, bytes);
}

void pinned_state_put(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_mem_mu);
    g_pinned_state.push_back(p);
}

void cached_free(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_mem_mu);
    auto it = g_live.find(p);
    if (it == g_live.end()) return;
    check_red_zone(p, it->second);
    g_cache[it->second.dev].emplace(it->second.size, p);
    g_live.erase(it);
}
}  // namespace


namespace {

thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
}

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

}  // namespace

struct kmeans_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int64_t N = 0, ldx = 0, global_N = 0, global_offset = 0;
    int d = 0, K = 0;
    void* comm = nullptr;
    int nranks = 1, rank = 0;
    bool group = false;           // distributed: NCCL communicator or a P2P-only group
    double comm_timeout_s = 60.0;

    float* X = nullptr;          // AoSoA fp32: ldx/64 tiles of [x64 y64 (z64)]
    double* mu = nullptr;        // 2 x Kpad x d (ping-pong by t & 1)
    float4* cneg = nullptr;      // 2 x K staged -fl32(mu): [0] current, [1] previous
    double* part = nullptr;      // nE x G per-block partials
    double* red = nullptr;       // nE merged partials
    DevState* st = nullptr;
    DevState* st_host = nullptr;  // pinned: reading the state never blocks the host in
                                  // cudaMemcpy (so sync() can poll NCCL while it waits)
    double* trace_E = nullptr;
    double* trace_J = nullptr;
    int trace_cap = 0;
    int32_t* labels = nullptr;   // ldx, lazily
    int64_t* idx_dev = nullptr;  // K
    int* flag = nullptr;

    int G = 0, tpb = 0, smem = 0, path = 0;   // G = columns of part (blocks or groups)
    int large_npl = 1;            // k_assign_large: 128-point sub-tiles per warp step
    bool large_split = false;     // large K: labels pass + k_accum_large (see configure)
    int large_grid1 = 0, large_tpb1 = 0, large_smem1 = 0;   // its labels pass
    int n_chunks = 0;
    int chunk_points = 0;         // points per chunk row (sorted / unsorted differ)
    double* cpart = nullptr;      // n_chunks x row_stride chunk rows (path 0 / sorted)
    int row_stride = 0;           // doubles per chunk row
    int n_super = 0;              // prune super-boxes (sorted, large K)
    float* sbox = nullptr;        // super-box bounding boxes
    int* slist = nullptr;         // n_super x K candidate lists
    float4* scl = nullptr;        // the same lists' staged centroids (k in .w)
    int* scount = nullptr;        // candidates per super-box
    int merge_smem = 0;           // k_merge_sparse dynamic shared memory (K x 4 doubles)
    int* heavy = nullptr;         // chunks deferred to k_assign_heavy (sorted, large K)
    int* heavy_count = nullptr;
    int heavy_smem = 0;
    int heavy_grid = 0;
    double2* htile = nullptr;     // KM_HEAVY_TILES: per heavy chunk and tile (J, entries)
    int* hctr = nullptr;          // KM_HEAVY_TILES: tiles done per heavy chunk (0 between launches)
    bool sorted = false;          // points held in Morton order (path 0 default)
    int64_t keep_n = 0;           // sorted small K: points [0, keep_n) kept resident in L2
    int32_t* perm = nullptr;      // sorted position -> caller's index (sorted only)
    int2* init_pairs = nullptr;   // (local index, k) of the initial indices (sorted only)
    int32_t* init_pos = nullptr;  // their sorted positions (k_find_pos)
    float* cbox = nullptr;        // per-chunk bounding boxes (sorted only)
    int* cand_count = nullptr;    // candidates per chunk, last assign (sorted only)
    int32_t* labels_sorted = nullptr;  // labels in sorted order (sorted only)
    int nE = 0;
    cudaGraphExec_t graph = nullptr;    // one iteration
    cudaGraphExec_t graph_u = nullptr;  // kGraphUnroll iterations (fewer graph launches)
    int flags = 0;            // kmeans_opts.flags
    // P2P exchange (kmeans_p2p_handle / kmeans_p2p_open): replaces the NCCL allreduce
    bool p2p = false;
    int gen = 0;              // kmeans_start generation (iteration exchange epochs)
    uint64_t xcount = 0;      // host-driven exchanges so far
    int xcap = 0;             // doubles per exchange slot
    void* xown = nullptr;     // own exchange buffer (cudaMalloc, IPC-exported)
    std::vector<void*> xopened;   // peers' buffers opened by IPC (closed at destroy)
    void** xtab = nullptr;    // device [2P]: xb pointers then xf pointers
    bool fused = false;       // small full-scan shard: k_fused_iterate (one launch, many iterations)
    bool persist = false;     // sorted K <= 16: k_persist_iterate (one launch, many iterations)
    int persist_grid = 0;
    int persist_smem = 0;
    km::PersistSync* psync = nullptr;
    double* pcol = nullptr;   // k_persist_iterate block columns [nE][persist_grid]
    int fused_grid = 0;
    int fused_smem = 0;
    double* brow = nullptr;   // k_fused_iterate block rows [2][nE][fused_grid]
    int64_t launches = 0;
    kmeans_status sticky = KMEANS_OK;
    bool assigned = false;
    std::vector<double> mu_host;   // mu^t given to the last kmeans_assign
};

namespace {

// KMEANS_TRACE=1: kmeans_create prints a per-phase timeline to stderr
// (synchronising the stream at every mark -- a tuning aid, off by default).
struct CreateTrace {
    bool on = false;
    const char* tag;
    std::chrono::steady_clock::time_point t0;
    explicit CreateTrace(const char* t = "kmeans_create") : tag(t) {
        const char* e = getenv("KMEANS_TRACE");
        on = e && *e && *e != '0';
        t0 = std::chrono::steady_clock::now();
    }
    void mark(cudaStream_t s, const char* what) {
        if (!on) return;
        if (s) cudaStreamSynchronize(s);
        const double ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        fprintf(stderr, "[%s] %8.2f ms  %s\n", tag, ms, what);
    }
};

#ifndef KM_BIG_CHUNK_TILES
#define KM_BIG_CHUNK_TILES 16   // 2048-point chunks for large shards
#endif
#ifndef KM_BIG_CHUNK_MIN_N
#define KM_BIG_CHUNK_MIN_N 40000000   // shards of >= this many points use 2048-point chunks
#endif
#ifndef KM_FUSED_TPW
#define KM_FUSED_TPW 2   // measured: 1, 2, 4, 8, 16, 32 -- 2 best from N = 1e4 to 1e6
#endif
#ifndef KM_MORTON_EXTRA
#define KM_MORTON_EXTRA 6   // Morton bits per axis beyond log2(N) / d
#endif
#ifndef KM_HILBERT
#define KM_HILBERT -1   // point order: 1 Hilbert curve, 0 Z-curve, -1 by shard (sort_points)
#endif
#ifndef KM_MORTON32
#define KM_MORTON32 0   // 32-bit Morton keys (see sort_points): 2 ms faster create at
                        // NS, but 10 bits per axis over a box stretched by far outliers
                        // (C5's planted sites) destroy the chunks' locality (C5: 360
                        // candidates per chunk, 7.7 ms per iteration) -- off
#endif
#ifndef KM_PDL
#define KM_PDL 1   // programmatic dependent launch between the iteration's kernels
#endif

// Launch with programmatic stream serialization (PDL) when `pdl`: the kernel
// may start while its stream predecessor drains (it synchronises with
// griddepcontrol.wait before reading the predecessor's results).
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     bool pdl, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = (pdl && KM_PDL) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}


// Device allocation for a context (through the block cache).  Freed blocks
// must be idle: callers synchronise ctx->stream before pool_free.
template <class T>
cudaError_t pool_alloc(kmeans_ctx* ctx, T** p, size_t bytes) {
    return cached_malloc(ctx->device, reinterpret_cast<void**>(p), bytes);
}

void pool_free(kmeans_ctx*, void* p) { cached_free(p); }

bool fused_update(const kmeans_ctx* ctx);
bool p2p_one_kernel(const kmeans_ctx* ctx);

// kernels of this library per iteration: [prune], assign, [heavy], [row merge],
// merge + update (fused into one kernel on a single GPU when small enough)
bool persist_active(const kmeans_ctx* ctx);

int kernels_per_iter(const kmeans_ctx* ctx) {
    if (ctx->fused || persist_active(ctx)) return 1;   // one launch covers many iterations
    int n = ctx->sorted ? (ctx->path == 1 ? 6 : 4) : (ctx->path == 0 ? 4 : 3);
    if (!ctx->sorted && ctx->large_split) n += 1;
    if (fused_update(ctx) || p2p_one_kernel(ctx)) n -= 1;
    return n;
}

kmeans_status cuda_fail(kmeans_ctx* c, cudaError_t e, const char* what) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    if (c) c->sticky = KMEANS_ECUDA;
    return KMEANS_ECUDA;
}

#define CK(call)                                                      \
    do {                                                              \
        cudaError_t _e = (call);                                      \
        if (_e != cudaSuccess) return cuda_fail(ctx, _e, #call);      \
    } while (0)

#define CHECK_CTX(c)                                                  \
    do {                                                              \
        if (!(c)) { set_error("NULL context"); return KMEANS_EINVAL; } \
        if ((c)->sticky != KMEANS_OK) {                               \
            set_error("context is in a sticky error state");          \
            return (c)->sticky;                                       \
        }                                                             \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// --- kernel selection --------------------------------------------------------
// path 0 (K <= 16): k_assign_chunk, one-warp blocks over 2048-point chunks.
// path 1 (K > 16):  k_assign_large, persistent blocks, smem centroids.
using ChunkFn = void (*)(const float*, int64_t, int, const double*, const DevState*, int, int,
                         double*, int32_t*);
using LargeFn = void (*)(const float*, int64_t, int64_t, int, const double*, const DevState*,
                         int, int, double*, int32_t*);

// Raise (never lower) a kernel's dynamic shared memory limit: the attribute
// is per function and process-wide, so contexts with different sizes (K, N)
// must not shrink it under one another.
cudaError_t allow_smem(const void* f, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> set;   // (device, kernel) -> bytes
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    int& cur = set[{dev, f}];
    if (bytes <= cur) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) cur = bytes;
    return e;
}

int small_kp(int K) { return K <= 4 ? 4 : (K <= 8 ? 8 : 16); }

using FusedFn = void (*)(const float*, int64_t, int, int, double*, DevState*, double*, double*,
                         int, double*, double*, int);

FusedFn pick_fused(int d, int K) {
    const int kp = small_kp(K);
    if (d == 2) return kp == 4 ? km::k_fused_iterate<2, 4>
                               : (kp == 8 ? km::k_fused_iterate<2, 8> : km::k_fused_iterate<2, 16>);
    return kp == 4 ? km::k_fused_iterate<3, 4>
                   : (kp == 8 ? km::k_fused_iterate<3, 8> : km::k_fused_iterate<3, 16>);
}

int fused_smem(int d, int K) {
    const int kp = small_kp(K);
    const int nE = K * d + K + 1;
    const size_t cs = kp == 4 ? sizeof(km::FusedSmem<4>)
                              : (kp == 8 ? sizeof(km::FusedSmem<8>) : sizeof(km::FusedSmem<16>));
    return (int)(cs * km::kFusedWarps +
                 sizeof(double) * (km::kFusedWarps * 66 + 2 * kp * d + nE));
}

template <int D, int MODE>
ChunkFn pick_chunk_kp(int K) {
    if (K <= 4) return km::k_assign_chunk<D, 4, MODE>;
    if (K <= 8) return km::k_assign_chunk<D, 8, MODE>;
    return km::k_assign_chunk<D, 16, MODE>;
}

ChunkFn pick_chunk(int d, int K, int mode) {
    if (d == 2) {
        if (mode == 1) return pick_chunk_kp<2, 1>(K);
        if (mode == 2) return pick_chunk_kp<2, 2>(K);
        return pick_chunk_kp<2, 3>(K);
    }
    if (mode == 1) return pick_chunk_kp<3, 1>(K);
    if (mode == 2) return pick_chunk_kp<3, 2>(K);
    return pick_chunk_kp<3, 3>(K);
}

using PrunedFn = void (*)(const float*, int64_t, int, const float4*, const DevState*, int, int,
                          const float*, const int*, const float4*, const int*, double*, int,
                          int32_t*, int*, int*, int*, int64_t);
using HeavyFn = void (*)(const float*, int64_t, int, const float4*, const DevState*, int, int,
                         const float*, const int*, const float4*, const int*, const int*,
                         const int*, double*, int, int32_t*);

using HeavyTileFn = void (*)(const float*, int64_t, int, const DevState*, int, const int*,
                             const float4*, const int*, const int*, const int*, double*, int,
                             int32_t*, double2*, int*);

HeavyTileFn pick_heavy_tiles(int d, int mode) {
    if (d == 2) {
        if (mode == 1) return km::k_assign_heavy_tiles<2, 1>;
        if (mode == 2) return km::k_assign_heavy_tiles<2, 2>;
        return km::k_assign_heavy_tiles<2, 3>;
    }
    if (mode == 1) return km::k_assign_heavy_tiles<3, 1>;
    if (mode == 2) return km::k_assign_heavy_tiles<3, 2>;
    return km::k_assign_heavy_tiles<3, 3>;
}

HeavyFn pick_heavy(int d, int mode) {
    if (d == 2) {
        if (mode == 1) return km::k_assign_heavy<2, 1>;
        if (mode == 2) return km::k_assign_heavy<2, 2>;
        return km::k_assign_heavy<2, 3>;
    }
    if (mode == 1) return km::k_assign_heavy<3, 1>;
    if (mode == 2) return km::k_assign_heavy<3, 2>;
    return km::k_assign_heavy<3, 3>;
}

template <bool LARGE, int CHT>
PrunedFn pick_pruned_l(int d, int mode) {
    if (d == 2) {
        if (mode == 1) return km::k_assign_pruned<2, 1, LARGE, CHT>;
        if (mode == 2) return km::k_assign_pruned<2, 2, LARGE, CHT>;
        return km::k_assign_pruned<2, 3, LARGE, CHT>;
    }
    if (mode == 1) return km::k_assign_pruned<3, 1, LARGE, CHT>;
    if (mode == 2) return km::k_assign_pruned<3, 2, LARGE, CHT>;
    return km::k_assign_pruned<3, 3, LARGE, CHT>;
}

// chunk_points: 1024, or (small K) 2048 for large shards
PrunedFn pick_pruned(int d, int K, int mode, int chunk_points = km::kSChunkPoints) {
    if (K > 16) return pick_pruned_l<true, KM_SORTED_CHUNK_TILES>(d, mode);
    return chunk_points == KM_BIG_CHUNK_TILES * km::kLaneTile
               ? pick_pruned_l<false, KM_BIG_CHUNK_TILES>(d, mode)
               : pick_pruned_l<false, KM_SORTED_CHUNK_TILES>(d, mode);
}

using PersistFn = void (*)(const float*, int64_t, int, int, const float*, float4*, double*,
                           DevState*, double*, double*, int, double*, double*, double*,
                           km::PersistSync*, int64_t, int, km::P2PView);

PersistFn pick_persist(int d, int chunk_points) {
    const bool big = chunk_points == KM_BIG_CHUNK_TILES * km::kLaneTile;
    if (d == 2)
        return big ? km::k_persist_iterate<2, KM_BIG_CHUNK_TILES>
                   : km::k_persist_iterate<2, KM_SORTED_CHUNK_TILES>;
    return big ? km::k_persist_iterate<3, KM_BIG_CHUNK_TILES>
               : km::k_persist_iterate<3, KM_SORTED_CHUNK_TILES>;
}

int pruned_smem(int d, int K) {
    if (K <= 16)
        return d == 2 ? sizeof(km::PrunedSmem<2, false>) : sizeof(km::PrunedSmem<3, false>);
    return d == 2 ? sizeof(km::PrunedSmem<2, true>) : sizeof(km::PrunedSmem<3, true>);
}

int chunk_smem(int d, int K) {
    const int kp = small_kp(K);
    if (d == 2)
        return kp == 4 ? sizeof(km::ChunkSmem<2, 4>)
                       : (kp == 8 ? sizeof(km::ChunkSmem<2, 8>) : sizeof(km::ChunkSmem<2, 16>));
    return kp == 4 ? sizeof(km::ChunkSmem<3, 4>)
                   : (kp == 8 ? sizeof(km::ChunkSmem<3, 8>) : sizeof(km::ChunkSmem<3, 16>));
}

#ifndef KM_LARGE_SPLIT_WARPS
#define KM_LARGE_SPLIT_WARPS 8    // split the large-K full scan below this many fused warps / SM
#endif
#ifndef KM_LARGE_SPLIT_NPL
#define KM_LARGE_SPLIT_NPL 3      // sub-tiles per warp step of the labels pass
#endif
#ifndef KM_LARGE_SPLIT_TPB
#define KM_LARGE_SPLIT_TPB 128    // threads per block of the labels pass
#endif
#ifndef KM_LARGE_NPL2
#define KM_LARGE_NPL2 1   // allow the wide k_assign_large step (see configure)
#endif
#ifndef KM_LARGE_NPL_BIG
#define KM_LARGE_NPL_BIG 2   // its 128-point sub-tiles per warp step
#endif

LargeFn pick_large(int d, int mode, int npl) {
    if (d == 2) {
        if (npl == 2) {
            if (mode == 1) return km::k_assign_large<2, 1, KM_LARGE_NPL_BIG>;
            if (mode == 2) return km::k_assign_large<2, 2, KM_LARGE_NPL_BIG>;
            return km::k_assign_large<2, 3, KM_LARGE_NPL_BIG>;
        }
        if (mode == 1) return km::k_assign_large<2, 1, 1>;
        if (mode == 2) return km::k_assign_large<2, 2, 1>;
        return km::k_assign_large<2, 3, 1>;
    }
    if (npl == 2) {
        if (mode == 1) return km::k_assign_large<3, 1, KM_LARGE_NPL_BIG>;
        if (mode == 2) return km::k_assign_large<3, 2, KM_LARGE_NPL_BIG>;
        return km::k_assign_large<3, 3, KM_LARGE_NPL_BIG>;
    }
    if (mode == 1) return km::k_assign_large<3, 1, 1>;
    if (mode == 2) return km::k_assign_large<3, 2, 1>;
    return km::k_assign_large<3, 3, 1>;
}


LargeFn pick_large_labels(int d) {
    return d == 2 ? km::k_assign_large<2, 2, KM_LARGE_SPLIT_NPL, true>
                  : km::k_assign_large<3, 2, KM_LARGE_SPLIT_NPL, true>;
}

int large_smem(int d, int K, int tpb) {
    const int W = tpb / 32;
    return km::large_kpad(K) * 16 + W * K * d * 8 + (W * K + 1) * 4 + 8 + W * 8;
}

kmeans_status configure(kmeans_ctx* ctx) {
    // (cudaDeviceGetAttribute: cudaGetDeviceProperties costs milliseconds)
    int sms = 0, maxSmem = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    CK(cudaDeviceGetAttribute(&maxSmem, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
    ctx->nE = ctx->K * ctx->d + ctx->K + 1;
    ctx->path = ctx->K <= 16 ? 0 : 1;
    if (ctx->sorted) {
        // Morton-sorted shard, per-chunk pruning (any K), sparse chunk rows
        ctx->tpb = 32;
        ctx->smem = pruned_smem(ctx->d, ctx->K);
        // small K: 2048-point chunks for large shards (fewer rows and CTAs: 2-3%
        // per iteration at N = 1e8), 1024 below (shorter CTAs: 14% at 1.25e7)
        const bool big = ctx->N >= (int64_t)KM_BIG_CHUNK_MIN_N ||
                         (ctx->flags & KMEANS_FLAG_BIG_CHUNKS);
        ctx->chunk_points = (ctx->K <= 16 && big) ? KM_BIG_CHUNK_TILES * km::kLaneTile
                                                  : km::kSChunkPoints;
        {   // L2-resident prefix of the point stream (small K): shards of up to
            // ~2.5x the 126 MB L2 keep their first 64 MB evict_last across
            // iterations (measured: the 1.25e7-point NS shard 35.2 -> 34.0 us per
            // iteration; 2.5e7 points unchanged); tuning: KMEANS_L2_KEEP_MB
            const double shard_mb = 4.0 * ctx->d * (double)ctx->N / 1e6;
            const char* e = getenv("KMEANS_L2_KEEP_MB");
            const double mb = e ? atof(e) : (shard_mb <= 320.0 ? 64.0 : 0.0);
            ctx->keep_n = (int64_t)(mb * 1e6 / (4.0 * ctx->d));
        }
        for (int mode = 1; mode <= 3; ++mode)
            CK(allow_smem((const void*)pick_pruned(ctx->d, ctx->K, mode, ctx->chunk_points), ctx->smem));
        ctx->n_chunks = (int)((ctx->N + ctx->chunk_points - 1) / ctx->chunk_points);
        // sparse rows: <= 16 entries (k_merge_sparse16) or up to K (k_merge_sparse)
        ctx->row_stride = ctx->K <= 16 ? km::kRowDoubles : km::kRowHead + 4 * km::large_row_entries(ctx->K);
        // groups: kRowGroup rows (k_merge_sparse16) or kGroupChunks rows (k_merge_sparse)
        ctx->G = ctx->K <= 16 ? (ctx->n_chunks + km::kRowGroup - 1) / km::kRowGroup
                              : (ctx->n_chunks + km::kGroupChunks - 1) / km::kGroupChunks;
        ctx->n_super = (ctx->n_chunks + km::kSuperChunks - 1) / km::kSuperChunks;
        ctx->merge_smem = 4 * ctx->K * (int)sizeof(double);   // k_merge_sparse table
        CK(allow_smem((const void*)km::k_merge_sparse<2>, ctx->merge_smem));
        CK(allow_smem((const void*)km::k_merge_sparse<3>, ctx->merge_smem));
        if (ctx->path == 1) {
            // per-warp slot tables and entry lists, the staged super list (K
            // float4), then 8 tile lists of K u16
            int hocc = 0;   // one resident block per heavy chunk (tile) when possible
            if (KM_HEAVY_TILES) {
                // the staged super list (K float4) and one tile list (K u16)
                ctx->heavy_smem = (int)(sizeof(km::HeavyTileSmem) +
                                        sizeof(float4) * (KM_HEAVY_GATHER ? 2 : 1) * ctx->K +
                                        sizeof(unsigned short) * ctx->K);
                for (int mode = 1; mode <= 3; ++mode)
                    CK(allow_smem((const void*)pick_heavy_tiles(ctx->d, mode), ctx->heavy_smem));
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                    &hocc, (const void*)pick_heavy_tiles(ctx->d, 1), 256, ctx->heavy_smem));
            } else {
                ctx->heavy_smem = (int)(sizeof(km::HeavySmem<3>) + sizeof(float4) * ctx->K +
                                        sizeof(unsigned short) * km::kHeavyWarps * ctx->K);
                for (int mode = 1; mode <= 3; ++mode)
                    CK(allow_smem((const void*)pick_heavy(ctx->d, mode), ctx->heavy_smem));
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                    &hocc, (const void*)pick_heavy(ctx->d, 1), 256, ctx->heavy_smem));
            }
            ctx->heavy_grid = sms * std::max(hocc, 1);
        }
        if (ctx->path == 0 && (ctx->flags & KMEANS_FLAG_PERSIST)) {
            // the whole iteration as one persistent kernel (one block per SM)
            PersistFn pf = pick_persist(ctx->d, ctx->chunk_points);
            const int W = ctx->d == 2 ? km::PersistCfg<2>::kWarps : km::PersistCfg<3>::kWarps;
            ctx->persist_smem = W * ctx->smem + W * km::kAccStride * (int)sizeof(double);
            int occ = 0, coop = 0;
            if (ctx->persist_smem <= maxSmem &&
                cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device) ==
                    cudaSuccess &&
                coop &&
                allow_smem((const void*)pf, ctx->persist_smem) == cudaSuccess &&
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)pf, W * 32,
                                                              ctx->persist_smem) == cudaSuccess &&
                occ >= 1) {
                // every warp of the grid must own >= 1 of the shard's 256-point units
                ctx->persist = sms <= km::kBlockGroup * km::kMaxBlockGroups &&
                               (ctx->N + km::kSortedUnit - 1) / km::kSortedUnit >= (int64_t)sms * W;
                ctx->persist_grid = sms;
            }
            cudaGetLastError();
        }
    } else if (ctx->path == 0) {
        ctx->tpb = 32;
        ctx->smem = chunk_smem(ctx->d, ctx->K);
        for (int mode = 1; mode <= 3; ++mode)
            CK(allow_smem((const void*)pick_chunk(ctx->d, ctx->K, mode), ctx->smem));
        ctx->chunk_points = km::kChunkPoints;
        ctx->n_chunks = (int)((ctx->N + ctx->chunk_points - 1) / ctx->chunk_points);
        ctx->row_stride = km::kRowDoubles;
        ctx->G = (ctx->n_chunks + km::kDenseGroup - 1) / km::kDenseGroup;  // groups
        // small single-GPU shard: whole iterations in one cooperative launch
        if (!ctx->group && !(ctx->flags & KMEANS_FLAG_NO_FUSED) &&
            ctx->n_chunks <= 4 * sms * km::kFusedWarps) {
            ctx->fused_smem = fused_smem(ctx->d, ctx->K);
            FusedFn ff = pick_fused(ctx->d, ctx->K);
            int occ = 0;
            if (ctx->fused_smem <= maxSmem &&
                allow_smem((const void*)ff, ctx->fused_smem) == cudaSuccess &&
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)ff,
                                                              km::kFusedWarps * 32,
                                                              ctx->fused_smem) == cudaSuccess &&
                occ >= 1) {
                // ~KM_FUSED_TPW warp-tiles (128 points each) per warp, <= 1 block per
                // SM (co-resident)
                const int64_t tiles = (ctx->N + 127) / 128;
                const int64_t per = (int64_t)KM_FUSED_TPW * km::kFusedWarps;
                const int64_t need = (tiles + per - 1) / per;
                ctx->fused_grid = (int)std::min<int64_t>(std::max<int64_t>(need, 1), sms);
                ctx->fused = true;
            }
            cudaGetLastError();
        }
    } else {
        int tpb = km::kLargeTPBMax;
        while (tpb > 64 && large_smem(ctx->d, ctx->K, tpb) > maxSmem - 4096) tpb -= 32;
        ctx->tpb = tpb;
        ctx->smem = large_smem(ctx->d, ctx->K, tpb);
        if (ctx->smem > maxSmem) {
            set_error("K=%d needs %d B of shared memory (max %d)", ctx->K, ctx->smem, maxSmem);
            return KMEANS_EINVAL;
        }
        // two 128-point sub-tiles per warp step where the accumulators leave
        // room for one block per SM anyway; one (fewer registers) otherwise
        int occ = 0;
        for (int npl = 1; npl <= 2; ++npl) {
            for (int mode = 1; mode <= 3; ++mode)
                CK(allow_smem((const void*)pick_large(ctx->d, mode, npl), ctx->smem));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &occ, (const void*)pick_large(ctx->d, 1, npl), ctx->tpb, ctx->smem));
            ctx->large_npl = npl;
            if (occ >= 2 || KM_LARGE_NPL2 == 0) break;
        }
        occ = std::max(occ, 1);
        ctx->G = sms * occ;  // persistent grid: every SM busy, static tile schedule
        // Where the per-warp accumulators cap the fused kernel below
        // KM_LARGE_SPLIT_WARPS warps per SM (K >= ~500 in 3D), split it: an
        // argmin pass with only the centroids in smem (occupancy set by
        // registers) writes the labels, then k_accum_large (the fused
        // kernel's grid, block and smem) sums points by label -- 16 B per
        // point more HBM traffic for ~2x the warps on the FP32-bound pass.
        ctx->large_split = occ * (ctx->tpb / 32) < KM_LARGE_SPLIT_WARPS;
        if (ctx->large_split) {
            auto acc = ctx->d == 2 ? km::k_accum_large<2> : km::k_accum_large<3>;
            CK(allow_smem((const void*)acc, ctx->smem));
            int occ2 = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, (const void*)acc, ctx->tpb,
                                                             ctx->smem));
            ctx->G = sms * std::max(occ2, 1);
            ctx->large_tpb1 = KM_LARGE_SPLIT_TPB;
            ctx->large_smem1 = km::large_kpad(ctx->K) * 16;
            int occ1 = 0;
            CK(allow_smem((const void*)pick_large_labels(ctx->d), ctx->large_smem1));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &occ1, (const void*)pick_large_labels(ctx->d), ctx->large_tpb1, ctx->large_smem1));
            ctx->large_grid1 = sms * std::max(occ1, 1);
            if (!ctx->labels) CK(pool_alloc(ctx, &ctx->labels, sizeof(int32_t) * ctx->ldx));
        }
    }
    return KMEANS_OK;
}

// stages: 1 = the assign kernels ([prune], assign, [heavy]), 2 = the chunk-row
// merge; 3 = both (the iteration).  Split only for kmeans_profile_stage.
kmeans_status launch_assign(kmeans_ctx* ctx, int mode, int mu_sel, int ignore_done,
                            int stages = 3) {
    const bool A = stages & 1, Mg = (stages & 2) && (mode & km::kModeReduce);
    if ((mode & km::kModeLabels) && !ctx->labels) {
        CK(pool_alloc(ctx, &ctx->labels, sizeof(int32_t) * ctx->ldx));
    }
    if (ctx->sorted) {
        if ((mode & km::kModeLabels) && !ctx->labels_sorted)
            CK(pool_alloc(ctx, &ctx->labels_sorted, sizeof(int32_t) * ctx->ldx));
        if (A && ctx->path == 1) {
            // super-box candidate lists (large K)
            if (ctx->d == 2)
                km::k_prune<2><<<ctx->n_super, 256, 0, ctx->stream>>>(
                    ctx->cneg, ctx->st, mu_sel, ignore_done, ctx->K, ctx->sbox, ctx->slist,
                    ctx->scl, ctx->scount, ctx->heavy_count);
            else
                km::k_prune<3><<<ctx->n_super, 256, 0, ctx->stream>>>(
                    ctx->cneg, ctx->st, mu_sel, ignore_done, ctx->K, ctx->sbox, ctx->slist,
                    ctx->scl, ctx->scount, ctx->heavy_count);
            ctx->launches += 1;
        }
        PrunedFn f = pick_pruned(ctx->d, ctx->K, mode, ctx->chunk_points);
        if (A)
            CK(launch_k(f, ctx->n_chunks, 32, ctx->smem, ctx->stream, ctx->path == 0, ctx->X,
                        ctx->N, ctx->K, (const float4*)ctx->cneg, (const DevState*)ctx->st, mu_sel,
                        ignore_done, (const float*)ctx->cbox, (const int*)ctx->slist,
                        (const float4*)ctx->scl, (const int*)ctx->scount, ctx->cpart,
                        ctx->row_stride, ctx->labels_sorted,
                        ctx->cand_count, ctx->heavy, ctx->heavy_count, ctx->keep_n));
        if (A) ctx->launches += 1;
        if (A && ctx->path == 1 && KM_HEAVY_TILES) {
            HeavyTileFn hf = pick_heavy_tiles(ctx->d, mode);
            hf<<<ctx->heavy_grid, 256, ctx->heavy_smem, ctx->stream>>>(
                ctx->X, ctx->N, ctx->K, ctx->st, ignore_done, ctx->slist, ctx->scl, ctx->scount,
                ctx->heavy, ctx->heavy_count, ctx->cpart, ctx->row_stride, ctx->labels_sorted,
                ctx->htile, ctx->hctr);
            ctx->launches += 1;
        } else if (A && ctx->path == 1) {
            HeavyFn hf = pick_heavy(ctx->d, mode);
            hf<<<ctx->heavy_grid, 256, ctx->heavy_smem, ctx->stream>>>(
                ctx->X, ctx->N, ctx->K, ctx->cneg, ctx->st, mu_sel, ignore_done, ctx->cbox,
                ctx->slist, ctx->scl, ctx->scount, ctx->heavy, ctx->heavy_count, ctx->cpart,
                ctx->row_stride, ctx->labels_sorted);
            ctx->launches += 1;
        }
        if (Mg && ctx->path == 0) {
            // sparse chunk rows (<= 16 entries) -> group columns of part (fixed order)
            CK(launch_k(ctx->d == 2 ? km::k_merge_sparse16<2> : km::k_merge_sparse16<3>, ctx->G,
                        km::kRowGroup, 0, ctx->stream, true, (const double*)ctx->cpart,
                        ctx->n_chunks, ctx->K, ctx->part, ctx->G, (const DevState*)ctx->st,
                        ignore_done));
            ctx->launches += 1;
        } else if (Mg) {
            // sparse chunk rows -> group columns of part (fixed ascending order)
            if (ctx->d == 2)
                km::k_merge_sparse<2><<<ctx->G, 256, ctx->merge_smem, ctx->stream>>>(
                    ctx->cpart, ctx->row_stride, ctx->n_chunks, ctx->K, ctx->part, ctx->G,
                    ctx->st, ignore_done);
            else
                km::k_merge_sparse<3><<<ctx->G, 256, ctx->merge_smem, ctx->stream>>>(
                    ctx->cpart, ctx->row_stride, ctx->n_chunks, ctx->K, ctx->part, ctx->G,
                    ctx->st, ignore_done);
            ctx->launches += 1;
        }
    } else if (ctx->path == 0) {
        ChunkFn f = pick_chunk(ctx->d, ctx->K, mode);
        if (A) f<<<ctx->n_chunks, 32, ctx->smem, ctx->stream>>>(ctx->X, ctx->N, ctx->K, ctx->mu, ctx->st,
                                                         mu_sel, ignore_done, ctx->cpart,
                                                         ctx->labels);
        if (A) ctx->launches += 1;
        if (Mg) {
            // chunk rows -> group columns of part (fixed ascending order)
            if (ctx->d == 2)
                km::k_merge_rows<2><<<ctx->G, 288, 0, ctx->stream>>>(
                    ctx->cpart, ctx->n_chunks, ctx->K, ctx->part, ctx->G, ctx->st, ignore_done);
            else
                km::k_merge_rows<3><<<ctx->G, 288, 0, ctx->stream>>>(
                    ctx->cpart, ctx->n_chunks, ctx->K, ctx->part, ctx->G, ctx->st, ignore_done);
            ctx->launches += 1;
        }
    } else {
        if (A && ctx->large_split) {
            pick_large_labels(ctx->d)<<<ctx->large_grid1, ctx->large_tpb1, ctx->large_smem1,
                                        ctx->stream>>>(ctx->X, ctx->ldx, ctx->N, ctx->K, ctx->mu,
                                                       ctx->st, mu_sel, ignore_done, nullptr,
                                                       ctx->labels);
            ctx->launches += 1;
            if (mode & km::kModeReduce) {
                (ctx->d == 2 ? km::k_accum_large<2> : km::k_accum_large<3>)
                    <<<ctx->G, ctx->tpb, ctx->smem, ctx->stream>>>(
                        ctx->X, ctx->N, ctx->K, ctx->mu, ctx->st, mu_sel, ignore_done,
                        ctx->labels, ctx->part);
                ctx->launches += 1;
            }
        } else if (A) {
            LargeFn f = pick_large(ctx->d, mode, ctx->large_npl);
            ctx->launches += 1;
            f<<<ctx->G, ctx->tpb, ctx->smem, ctx->stream>>>(ctx->X, ctx->ldx, ctx->N, ctx->K,
                                                            ctx->mu, ctx->st, mu_sel, ignore_done,
                                                            ctx->part, ctx->labels);
        }
    }
    CK(cudaGetLastError());
    if (A && (mode & km::kModeLabels) && ctx->sorted) {
        // back to the caller's order
        const int blocks = (int)std::min<int64_t>((ctx->N + 255) / 256, 148 * 8);
        km::k_scatter_labels<<<blocks, 256, 0, ctx->stream>>>(ctx->labels_sorted, ctx->perm,
                                                              ctx->N, ctx->labels);
        ctx->launches += 1;
        CK(cudaGetLastError());
    }
    return KMEANS_OK;
}

kmeans_status launch_merge(kmeans_ctx* ctx, int ignore_done) {
    const int wpb = 8;
    km::k_merge<<<(ctx->nE + wpb - 1) / wpb, wpb * 32, 0, ctx->stream>>>(
        ctx->part, ctx->G, ctx->nE, ctx->red, ctx->st, ignore_done);
    ctx->launches += 1;
    CK(cudaGetLastError());
    return KMEANS_OK;
}

km::P2PView p2p_view(const kmeans_ctx* ctx) {
    km::P2PView v;
    v.xb = reinterpret_cast<double* const*>(ctx->xtab);
    v.xf = reinterpret_cast<uint64_t* const*>(ctx->xtab + ctx->nranks);
    v.P = ctx->nranks;
    v.rank = ctx->rank;
    v.cap = ctx->xcap;
    v.timeout_ns = (uint64_t)(ctx->comm_timeout_s * 1e9);
    return v;
}

kmeans_status allreduce(kmeans_ctx* ctx, double* buf, size_t count) {
    if (ctx->p2p) {   // host-driven exchange over peer memory (slots 2/3)
        const uint64_t n = ++ctx->xcount;
        km::k_p2p_allreduce<<<1, 256, 0, ctx->stream>>>(p2p_view(ctx), buf, (int)count,
                                                       2 + (int)(n & 1), (1ull << 63) | n,
                                                       ctx->st);
        ctx->launches += 1;
        CK(cudaGetLastError());
        return KMEANS_OK;
    }
    if (!ctx->group) return KMEANS_OK;
    if (!ctx->comm) {   // a P2P-only group before kmeans_p2p_open: nothing to exchange with
        set_error("P2P-only group: call kmeans_p2p_handle / kmeans_p2p_open first");
        return KMEANS_ESTATE;
    }
#ifdef KMEANS_WITH_NCCL
    ncclResult_t r = ncclAllReduce(buf, buf, count, ncclFloat64, ncclSum, (ncclComm_t)ctx->comm,
                                   ctx->stream);
    if (r != ncclSuccess) {
        set_error("ncclAllReduce: %s", ncclGetErrorString(r));
        ctx->sticky = KMEANS_ENCCL;
        return KMEANS_ENCCL;
    }
    return KMEANS_OK;
#else
    (void)buf;
    (void)count;
    set_error("library built without NCCL");
    ctx->sticky = KMEANS_ENCCL;
    return KMEANS_ENCCL;
#endif
}

kmeans_status launch_update(kmeans_ctx* ctx) {
    // one block; enough threads that each handles <= ~4 of the K d entries
    const int tpb = std::min(1024, std::max(256, ((ctx->K * ctx->d + 3) / 4 + 31) / 32 * 32));
    if (ctx->d == 2)
        km::k_update<2><<<1, tpb, 0, ctx->stream>>>(ctx->mu, ctx->K, ctx->red, ctx->st,
                                                    ctx->trace_E, ctx->trace_J, ctx->trace_cap,
                                                    ctx->sorted ? ctx->cneg : nullptr);
    else
        km::k_update<3><<<1, tpb, 0, ctx->stream>>>(ctx->mu, ctx->K, ctx->red, ctx->st,
                                                    ctx->trace_E, ctx->trace_J, ctx->trace_cap,
                                                    ctx->sorted ? ctx->cneg : nullptr);
    ctx->launches += 1;
    CK(cudaGetLastError());
    return KMEANS_OK;
}

// The persistent kernel runs the iteration when the context has it and the
// exchange (if any) is the P2P one (an NCCL call cannot run inside a kernel).
bool persist_active(const kmeans_ctx* ctx) {
    return ctx->persist && (!ctx->group || ctx->p2p);
}

// Single GPU and a small enough group table: merge + update in one block.
bool fused_update(const kmeans_ctx* ctx) {
    return !ctx->group && (int64_t)ctx->nE * ctx->G <= 400000 && ctx->nE * 8 <= 48 * 1024;
}

// P2P exchange and a small group table: merge + exchange + update in one block.
bool p2p_one_kernel(const kmeans_ctx* ctx) {
    return ctx->p2p && (int64_t)ctx->nE * ctx->G <= 400000 && ctx->nE * 8 <= 48 * 1024;
}

kmeans_status launch_merge_update(kmeans_ctx* ctx) {
    const int tpb = 1024;
    const size_t sm = sizeof(double) * ctx->nE;
    // PDL after the sorted small-K row merge (k_merge_sparse16 triggers it)
    const bool pdl = ctx->sorted && ctx->path == 0;
    CK(launch_k(ctx->d == 2 ? km::k_merge_update<2> : km::k_merge_update<3>, 1, tpb, sm,
                ctx->stream, pdl, (const double*)ctx->part, ctx->G, ctx->nE, ctx->red, ctx->mu,
                ctx->K, ctx->st, ctx->trace_E, ctx->trace_J, ctx->trace_cap,
                ctx->sorted ? ctx->cneg : (float4*)nullptr));
    ctx->launches += 1;
    CK(cudaGetLastError());
    return KMEANS_OK;
}

// One iteration: assign+reduce, merge, [allreduce], update.
kmeans_status enqueue_iteration(kmeans_ctx* ctx) {
    kmeans_status s;
    if ((s = launch_assign(ctx, km::kModeReduce, 0, 0)) != KMEANS_OK) return s;
    if (fused_update(ctx)) return launch_merge_update(ctx);
    if (ctx->p2p) {   // [local group merge,] the exchange over peer memory, the update
        // small group table: the merge runs in the same block (one kernel)
        const bool one = p2p_one_kernel(ctx);
        if (!one && (s = launch_merge(ctx, 0)) != KMEANS_OK) return s;
        const int tpb = one ? 1024 : 256;
        const size_t sm = one ? sizeof(double) * ctx->nE : 0;
        const double* part = one ? ctx->part : nullptr;
        if (ctx->d == 2)
            km::k_p2p_update<2><<<1, tpb, sm, ctx->stream>>>(
                p2p_view(ctx), ctx->red, ctx->nE, ctx->mu, ctx->K, ctx->st, ctx->trace_E,
                ctx->trace_J, ctx->trace_cap, ctx->sorted ? ctx->cneg : nullptr, part, ctx->G);
        else
            km::k_p2p_update<3><<<1, tpb, sm, ctx->stream>>>(
                p2p_view(ctx), ctx->red, ctx->nE, ctx->mu, ctx->K, ctx->st, ctx->trace_E,
                ctx->trace_J, ctx->trace_cap, ctx->sorted ? ctx->cneg : nullptr, part, ctx->G);
        ctx->launches += 1;
        CK(cudaGetLastError());
        return KMEANS_OK;
    }
    if ((s = launch_merge(ctx, 0)) != KMEANS_OK) return s;
    if ((s = allreduce(ctx, ctx->red, ctx->nE)) != KMEANS_OK) return s;
    return launch_update(ctx);
}

constexpr int kGraphUnroll = 8;

kmeans_status capture_iterations(kmeans_ctx* ctx, int n, cudaGraphExec_t* out) {
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    const int64_t before = ctx->launches;
    kmeans_status s = KMEANS_OK;
    for (int i = 0; i < n && s == KMEANS_OK; ++i) s = enqueue_iteration(ctx);
    cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
    ctx->launches = before;  // capture is not a launch
    if (s != KMEANS_OK) {
        if (g) cudaGraphDestroy(g);
        return s;
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(out, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaGraphInstantiate");
    return KMEANS_OK;
}

// The iteration as CUDA graphs: one iteration, and kGraphUnroll iterations
// back to back (the device stop flag makes iterations after convergence no-ops).
kmeans_status ensure_graph(kmeans_ctx* ctx) {
    kmeans_status s;
    if (!ctx->graph && (s = capture_iterations(ctx, 1, &ctx->graph)) != KMEANS_OK) return s;
    if (!ctx->graph_u && (s = capture_iterations(ctx, kGraphUnroll, &ctx->graph_u)) != KMEANS_OK)
        return s;
    return KMEANS_OK;
}

#ifdef KMEANS_WITH_NCCL
// Communicators this library aborted (kmeans_comm_destroy must not free them again).
std::mutex g_abort_mu;
std::vector<void*> g_aborted;
#endif

// Waits for the context's stream.  With an NCCL communicator in use the wait
// is a poll: ncclCommGetAsyncError is checked while the stream runs, and a
// reported error or a wait longer than comm_timeout_s (a dead or hung peer)
// aborts the communicator -- KMEANS_ENCCL, sticky -- instead of blocking this
// rank forever.  (The P2P exchange bounds its own spin on the device.)
kmeans_status sync(kmeans_ctx* ctx) {
#ifdef KMEANS_WITH_NCCL
    if (ctx->comm && !ctx->p2p) {
        const auto t0 = std::chrono::steady_clock::now();
        for (int spin = 0;; ++spin) {
            const cudaError_t e = cudaStreamQuery(ctx->stream);
            if (e == cudaSuccess) return KMEANS_OK;
            if (e != cudaErrorNotReady) return cuda_fail(ctx, e, "cudaStreamQuery");
            ncclResult_t ar = ncclSuccess;
            ncclCommGetAsyncError((ncclComm_t)ctx->comm, &ar);
            const double waited =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if ((ar != ncclSuccess && ar != ncclInProgress) || waited > ctx->comm_timeout_s) {
                if (ar != ncclSuccess && ar != ncclInProgress)
                    set_error("NCCL asynchronous error: %s", ncclGetErrorString(ar));
                else
                    set_error("collective did not complete within %.1f s (peer dead or hung)",
                              ctx->comm_timeout_s);
                ncclCommAbort((ncclComm_t)ctx->comm);
                {
                    std::lock_guard<std::mutex> lk(g_abort_mu);
                    g_aborted.push_back(ctx->comm);
                }
                ctx->sticky = KMEANS_ENCCL;
                return KMEANS_ENCCL;
            }
            if (spin > 100) std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
    }
#endif
    CK(cudaStreamSynchronize(ctx->stream));
    return KMEANS_OK;
}

kmeans_status read_state(kmeans_ctx* ctx, DevState* h) {
    // through the context's pinned staging copy: a copy to pageable memory
    // would block right here until the whole stream drained
    CK(cudaMemcpyAsync(ctx->st_host, ctx->st, sizeof(DevState), cudaMemcpyDeviceToHost,
                       ctx->stream));
    kmeans_status s = sync(ctx);
    if (s != KMEANS_OK) return s;
    *h = *ctx->st_host;
    if (h->err == km::kErrExchangeTimeout) {   // a P2P exchange timed out (the run was stopped)
        set_error("P2P exchange: a peer did not publish within %.1f s (dead or hung rank)",
                  ctx->comm_timeout_s);
        ctx->sticky = KMEANS_ENCCL;
        return KMEANS_ENCCL;
    }
    if (h->err) {   // the persistent kernel waited too long for an iteration's update
        set_error("k_persist_iterate: an iteration's update was not published in time");
        ctx->sticky = KMEANS_ECUDA;
        return KMEANS_ECUDA;
    }
    return KMEANS_OK;
}

kmeans_status write_state(kmeans_ctx* ctx, int t, int done, int max_iter, double tol) {
    DevState h{};
    h.t = t;
    h.done = done;
    h.max_iter = max_iter;
    h.tol = tol;
    h.gen = ctx->gen;
    CK(cudaMemcpyAsync(ctx->st, &h, sizeof(DevState), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));  // h is a stack object
    return KMEANS_OK;
}

// cneg[0] (and [1]) <- -fl32(mu^t) for the pruned kernels; call after the
// fp64 master and DevState::t are set.
kmeans_status stage_centroids(kmeans_ctx* ctx) {
    if (!ctx->sorted) return KMEANS_OK;
    km::k_stage<<<(ctx->K + 127) / 128, 128, 0, ctx->stream>>>(ctx->mu, ctx->st, ctx->K, ctx->d,
                                                                 ctx->cneg, 1);
    ctx->launches += 1;
    CK(cudaGetLastError());
    return KMEANS_OK;
}

// Device E/J traces: kmeans_start keeps kTraceCap entries (the kernels skip
// t >= trace_cap); kmeans_fit_ctx grows them to max_iter only when the caller
// asks for the traces (its own buffers bound the size).
constexpr int kTraceCap = 4096;

kmeans_status ensure_trace(kmeans_ctx* ctx, int cap) {
    if (cap <= ctx->trace_cap) return KMEANS_OK;
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->graph) {
        cudaGraphExecDestroy(ctx->graph);  // captured the old trace pointers
        ctx->graph = nullptr;
        if (ctx->graph_u) cudaGraphExecDestroy(ctx->graph_u);
        ctx->graph_u = nullptr;
    }
    pool_free(ctx, ctx->trace_E);
    pool_free(ctx, ctx->trace_J);
    ctx->trace_E = ctx->trace_J = nullptr;
    ctx->trace_cap = 0;
    if (pool_alloc(ctx, &ctx->trace_E, sizeof(double) * cap) != cudaSuccess ||
        pool_alloc(ctx, &ctx->trace_J, sizeof(double) * cap) != cudaSuccess) {
        cudaGetLastError();
        set_error("trace allocation failed");
        return KMEANS_ENOMEM;
    }
    ctx->trace_cap = cap;
    return KMEANS_OK;
}

// Reads K init indices (host or device memory) and validates them against
// [0, global_N): distinct and in range.
kmeans_status fetch_init_idx(kmeans_ctx* ctx, const int64_t* init_idx, std::vector<int64_t>& out) {
    out.resize(ctx->K);
    CK(cudaMemcpy(out.data(), init_idx, sizeof(int64_t) * ctx->K, cudaMemcpyDefault));
    std::vector<int64_t> s(out);
    std::sort(s.begin(), s.end());
    for (int k = 0; k < ctx->K; ++k) {
        if (s[k] < 0 || s[k] >= ctx->global_N) {
            set_error("init_idx[%d] out of range [0, %lld)", k, (long long)ctx->global_N);
            return KMEANS_EINVAL;
        }
        if (k && s[k] == s[k - 1]) {
            set_error("init_idx holds %lld twice", (long long)s[k]);
            return KMEANS_EINVAL;
        }
    }
    return KMEANS_OK;
}

kmeans_status fetch_centroids(kmeans_ctx* ctx, const double* cent, std::vector<double>& out) {
    const size_t n = (size_t)ctx->K * ctx->d;
    out.resize(n);
    CK(cudaMemcpy(out.data(), cent, sizeof(double) * n, cudaMemcpyDefault));
    for (size_t q = 0; q < n; ++q) {
        if (!std::isfinite(out[q])) {
            set_error("centroid entry %zu is not finite", q);
            return KMEANS_ENONFINITE;
        }
    }
    return KMEANS_OK;
}

// Morton-order the shard once (sorted path): global box + finiteness, keys,
// stable CUB radix sort, gather into the AoSoA layout, per-chunk boxes.
kmeans_status sort_points(kmeans_ctx* ctx, const float* src, int64_t si, int64_t sj,
                          CreateTrace& tr) {
    const int64_t N = ctx->N;
    const int d = ctx->d;
    unsigned* box = nullptr;
    void *keys = nullptr, *keys2 = nullptr;
    int32_t* iota = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    kmeans_status st = KMEANS_OK;
    auto cleanup = [&]() {
        cudaStreamSynchronize(ctx->stream);   // temporaries idle before they are cached
        pool_free(ctx, box);
        pool_free(ctx, keys);
        pool_free(ctx, keys2);
        pool_free(ctx, iota);
        pool_free(ctx, tmp);
    };
    // Morton resolution: 2^qbits cells per axis with qbits = ceil(log2 N / d) + 6
    // (>= 64 cells per point per axis on average; sharper order buys nothing for
    // 1024-point chunks), capped by the key: 64-bit keys (21 / 32 bits per axis),
    // or with KM_MORTON32 32-bit keys (10 / 16 bits per axis, 4 radix passes over
    // 8-byte pairs); the sort only visits d * qbits bits.
    int lg = 1;
    while (lg < 40 && (int64_t(1) << lg) < N) ++lg;
    const bool k32 = KM_MORTON32 != 0;
    const int qcap = k32 ? 32 / d : (d == 2 ? 32 : 21);
    const int qbits = std::min(qcap, (lg + d - 1) / d + KM_MORTON_EXTRA);
    const size_t ksz = k32 ? sizeof(uint32_t) : sizeof(unsigned long long);
    // the Hilbert curve (no jumps: compact chunk boxes, fewer candidates) in
    // 3D, and in 2D below the 2048-point-chunk sizes; measured (DESIGN.md
    // section 4): C5 6.9 -> 5.0 candidates per chunk, 0.420 -> 0.380 ms per
    // iteration, NS 1.25e7-point shard 37.7 -> 34.8 us; C3 (2D, 1e8) 122 -> 126 us
    const int hilbert = KM_HILBERT >= 0 ? KM_HILBERT
                                        : (d == 3 || N < (int64_t)KM_BIG_CHUNK_MIN_N ? 1 : 0);
    if (pool_alloc(ctx, &ctx->perm, sizeof(int32_t) * N) != cudaSuccess ||
        pool_alloc(ctx, &ctx->init_pairs, sizeof(int2) * ctx->K) != cudaSuccess ||
        pool_alloc(ctx, &ctx->init_pos, sizeof(int32_t) * ctx->K) != cudaSuccess ||
        pool_alloc(ctx, &ctx->cbox, sizeof(float) * 2 * d * (size_t)ctx->n_chunks) != cudaSuccess ||
        pool_alloc(ctx, &ctx->cand_count, sizeof(int) * (size_t)ctx->n_chunks) != cudaSuccess ||
        pool_alloc(ctx, &box, sizeof(unsigned) * 6) != cudaSuccess ||
        pool_alloc(ctx, (char**)&keys, ksz * N) != cudaSuccess ||
        pool_alloc(ctx, (char**)&keys2, ksz * N) != cudaSuccess ||
        pool_alloc(ctx, &iota, sizeof(int32_t) * N) != cudaSuccess) {
        cudaGetLastError();
        cleanup();
        set_error("sort buffers: allocation failed");
        return KMEANS_ENOMEM;
    }
    unsigned hb2[6];
    for (int j = 0; j < d; ++j) {
        hb2[j] = 0xffffffffu;
        hb2[d + j] = 0u;
    }
    const int blocks = (int)std::min<int64_t>((N + 255) / 256, 148 * 8);
    cudaError_t e = cudaMemcpyAsync(box, hb2, sizeof(unsigned) * 2 * d, cudaMemcpyHostToDevice,
                                    ctx->stream);
    auto radix = [&](auto* k1, auto* k2) {
        using KeyT = std::remove_pointer_t<decltype(k1)>;
        (d == 2 ? km::k_morton<KeyT, 2> : km::k_morton<KeyT, 3>)<<<blocks, 256, 0, ctx->stream>>>(
            src, N, si, sj, box, qbits, hilbert, k1, iota);
        ctx->launches += 1;
        tr.mark(ctx->stream, "bbox + morton keys");
        cudaError_t r = cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k1, k2, iota,
                                                        ctx->perm, N, 0, d * qbits, ctx->stream);
        if (r == cudaSuccess) r = pool_alloc(ctx, &tmp, tmp_bytes);
        if (r == cudaSuccess)
            r = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k1, k2, iota, ctx->perm, N, 0,
                                                d * qbits, ctx->stream);
        return r;
    };
    if (e == cudaSuccess) {
        (d == 2 ? km::k_input_bbox<2> : km::k_input_bbox<3>)<<<blocks, 256, 0, ctx->stream>>>(
            src, N, si, sj, box, ctx->flag);
        ctx->launches += 1;
        e = k32 ? radix((uint32_t*)keys, (uint32_t*)keys2)
                : radix((unsigned long long*)keys, (unsigned long long*)keys2);
    }
    tr.mark(ctx->stream, "radix sort");
    if (e == cudaSuccess) {
        const int gb = (int)std::min<int64_t>((ctx->ldx + 255) / 256, 148 * 8);
        km::k_gather_sorted<<<gb, 256, 0, ctx->stream>>>(src, N, d, si, sj, ctx->perm,
                                                         ctx->X, ctx->ldx);
        tr.mark(ctx->stream, "gather");
        const int cb = (ctx->n_chunks * 32 + 255) / 256;
        km::k_chunk_bbox<<<cb, 256, 0, ctx->stream>>>(ctx->X, N, d, ctx->chunk_points,
                                                      ctx->n_chunks, ctx->cbox);
        ctx->launches += 2;
        if (ctx->sbox) {
            km::k_super_bbox<<<(ctx->n_super + 127) / 128, 128, 0, ctx->stream>>>(
                ctx->cbox, ctx->n_chunks, d, ctx->sbox);
            ctx->launches += 1;
        }
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);  // before freeing temporaries
    if (e != cudaSuccess) st = cuda_fail(ctx, e, "sort_points");
    cleanup();
    return st;
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

int kmeans_abi_version(void) { return KMEANS_ABI_VERSION; }

kmeans_status kmeans_p2p_handle(kmeans_ctx* ctx, unsigned char handle[64]) {
    CHECK_CTX(ctx);
    if (!handle || !ctx->group || ctx->p2p) {
        set_error("kmeans_p2p_handle: needs a handle buffer and a distributed context not yet opened");
        return KMEANS_EINVAL;
    }
    DeviceGuard g(ctx->device);
    const int P = ctx->nranks;
    if (!ctx->xown) {
        ctx->xcap = ctx->nE;
        const size_t bytes = sizeof(double) * km::kXSlots * P * (size_t)ctx->xcap +
                             sizeof(uint64_t) * km::kXSlots * P;
        CK(cudaMalloc(&ctx->xown, bytes));   // own allocation: IPC-exportable
        CK(cudaMemset(ctx->xown, 0, bytes));
        CK(cudaDeviceSynchronize());
    }
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, ctx->xown));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    memcpy(handle, &h, 64);
    return KMEANS_OK;
}

kmeans_status kmeans_p2p_open(kmeans_ctx* ctx, const unsigned char* handles) {
    CHECK_CTX(ctx);
    if (!handles || !ctx->xown || ctx->p2p) {
        set_error("kmeans_p2p_open: call kmeans_p2p_handle first (once)");
        return KMEANS_EINVAL;
    }
    DeviceGuard g(ctx->device);
    const int P = ctx->nranks;
    std::vector<void*> tab(2 * (size_t)P);
    for (int q = 0; q < P; ++q) {
        void* base = nullptr;
        if (q == ctx->rank) {
            base = ctx->xown;
        } else {
            cudaIpcMemHandle_t h;
            memcpy(&h, handles + 64 * (size_t)q, 64);
            const cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) {
                // not sticky: undo the mappings made so far and leave the context
                // usable, so that every rank can fall back to the NCCL allreduce
                cudaGetLastError();
                for (void* o : ctx->xopened) cudaIpcCloseMemHandle(o);
                ctx->xopened.clear();
                cudaGetLastError();
                set_error("kmeans_p2p_open: cudaIpcOpenMemHandle(rank %d): %s", q,
                          cudaGetErrorString(e));
                return KMEANS_ECUDA;
            }
            ctx->xopened.push_back(base);
        }
        tab[q] = base;
        tab[P + q] = static_cast<double*>(base) + (size_t)km::kXSlots * P * ctx->xcap;
    }
    if (!ctx->xtab) CK(pool_alloc(ctx, &ctx->xtab, sizeof(void*) * 2 * P));
    CK(cudaMemcpyAsync(ctx->xtab, tab.data(), sizeof(void*) * 2 * P, cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->p2p = true;
    if (ctx->graph) cudaGraphExecDestroy(ctx->graph);   // the iteration changes
    if (ctx->graph_u) cudaGraphExecDestroy(ctx->graph_u);
    ctx->graph = ctx->graph_u = nullptr;
    return KMEANS_OK;
}

kmeans_status kmeans_p2p_loopback(kmeans_ctx* ctx, int rounds, int n, const double* vals,
                                  double* out) {
    CHECK_CTX(ctx);
    if (!ctx->p2p || rounds < 1 || n < 1 || n > ctx->xcap || !vals || !out) {
        set_error("kmeans_p2p_loopback: needs an opened P2P group, rounds >= 1, 1 <= n <= %d",
                  ctx->xcap);
        return KMEANS_EINVAL;
    }
    DeviceGuard g(ctx->device);
    int coop = 0;
    CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device));
    if (!coop) {
        set_error("kmeans_p2p_loopback: no cooperative launch on this device");
        return KMEANS_ECUDA;
    }
    const int P = ctx->nranks;
    const size_t nv = (size_t)rounds * P * n;
    double *dv = nullptr, *dout = nullptr, *scratch = nullptr;
    int* dfail = nullptr;
    CK(cudaStreamSynchronize(ctx->stream));   // no exchange of this context in flight
    cudaError_t e = cudaMalloc(&dv, sizeof(double) * nv);
    if (e == cudaSuccess) e = cudaMalloc(&dout, sizeof(double) * nv);
    if (e == cudaSuccess) e = cudaMalloc(&scratch, sizeof(double) * P * (size_t)ctx->xcap);
    if (e == cudaSuccess) e = cudaMalloc(&dfail, sizeof(int) * P);
    if (e == cudaSuccess) e = cudaMemset(dfail, 0, sizeof(int) * P);
    if (e == cudaSuccess) e = cudaMemcpy(dv, vals, sizeof(double) * nv, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        // every rank of the group emulated by one block, over the real buffers:
        // this rank's own and the peers' (mapped by CUDA IPC); epochs of their
        // own (bit 41) so no iteration or host-driven exchange can match them
        double* const* xb = reinterpret_cast<double* const*>(ctx->xtab);
        uint64_t* const* xf = reinterpret_cast<uint64_t* const*>(ctx->xtab + P);
        int P_ = P, cap_ = ctx->xcap, n_ = n, r_ = rounds, dead = -1;
        uint64_t tmo = (uint64_t)(ctx->comm_timeout_s * 1e9);
        ctx->xcount += 1;
        uint64_t ebase = (1ull << 41) + (ctx->xcount << 16);
        void* args[] = {(void*)&xb,      (void*)&xf,   (void*)&P_,      (void*)&cap_,
                        (void*)&n_,      (void*)&r_,   (void*)&dv,      (void*)&dout,
                        (void*)&scratch, (void*)&dead, (void*)&tmo,     (void*)&dfail,
                        (void*)&ebase};
        e = cudaLaunchCooperativeKernel((const void*)km::k_p2p_emulate, dim3(P), dim3(128), args,
                                        0, ctx->stream);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    std::vector<int> hf(P, 0);
    if (e == cudaSuccess) e = cudaMemcpy(hf.data(), dfail, sizeof(int) * P, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(out, dout, sizeof(double) * nv, cudaMemcpyDeviceToHost);
    cudaFree(dv);
    cudaFree(dout);
    cudaFree(scratch);
    cudaFree(dfail);
    CK(e);
    for (int r = 0; r < P; ++r)
        if (hf[r]) {
            set_error("kmeans_p2p_loopback: emulated rank %d timed out in round %d", r, hf[r]);
            return KMEANS_ENCCL;
        }
    return KMEANS_OK;
}

kmeans_status kmeans_p2p_disable(kmeans_ctx* ctx) {
    CHECK_CTX(ctx);
    DeviceGuard g(ctx->device);
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->p2p) {
        ctx->p2p = false;
        if (ctx->graph) cudaGraphExecDestroy(ctx->graph);   // back to the NCCL iteration
        if (ctx->graph_u) cudaGraphExecDestroy(ctx->graph_u);
        ctx->graph = ctx->graph_u = nullptr;
    }
    return KMEANS_OK;
}

kmeans_status kmeans_p2p_selftest(int device, int P, int n, int rounds, const double* vals,
                                  double* out, int dead_rank, double timeout_s, int* failed) {
    if (P < 1 || P > 64 || n < 1 || rounds < 1 || !vals || !out || dead_rank >= P ||
        !(timeout_s >= 0.0)) {
        set_error("kmeans_p2p_selftest: bad argument");
        return KMEANS_EINVAL;
    }
    const uint64_t tmo = (uint64_t)((timeout_s > 0.0 ? timeout_s : 60.0) * 1e9);
    DeviceGuard g(device);
    kmeans_ctx* ctx = nullptr;   // for CK
    int coop = 0;
    CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
    const int cap = n;
    const size_t per = sizeof(double) * km::kXSlots * P * (size_t)cap +
                       sizeof(uint64_t) * km::kXSlots * P;
    char* arena = nullptr;
    double *dv = nullptr, *dout = nullptr, *scratch = nullptr;
    int* dfail = nullptr;
    void** tab = nullptr;
    const size_t nv = (size_t)rounds * P * n;
    cudaError_t e = cudaMalloc(&arena, per * P);
    if (e == cudaSuccess) e = cudaMalloc(&dfail, sizeof(int) * P);
    if (e == cudaSuccess) e = cudaMemset(dfail, 0, sizeof(int) * P);
    if (e == cudaSuccess) e = cudaMemset(arena, 0, per * P);
    if (e == cudaSuccess) e = cudaMalloc(&dv, sizeof(double) * nv);
    if (e == cudaSuccess) e = cudaMalloc(&dout, sizeof(double) * nv);
    if (e == cudaSuccess) e = cudaMalloc(&scratch, sizeof(double) * P * (size_t)cap);
    if (e == cudaSuccess) e = cudaMalloc(&tab, sizeof(void*) * 2 * P);
    std::vector<void*> h(2 * (size_t)P);
    for (int q = 0; q < P; ++q) {
        h[q] = arena + per * q;
        h[P + q] = static_cast<double*>(h[q]) + (size_t)km::kXSlots * P * cap;
    }
    if (e == cudaSuccess) e = cudaMemcpy(tab, h.data(), sizeof(void*) * 2 * P, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(dv, vals, sizeof(double) * nv, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        double* const* xb = reinterpret_cast<double* const*>(tab);
        uint64_t* const* xf = reinterpret_cast<uint64_t* const*>(tab + P);
        int cap_ = cap, P_ = P, n_ = n, r_ = rounds, dead = dead_rank;
        uint64_t tmo_ = tmo, ebase = 1ull << 40;
        void* args[] = {(void*)&xb,   (void*)&xf,    (void*)&P_,      (void*)&cap_,
                        (void*)&n_,   (void*)&r_,    (void*)&dv,      (void*)&dout,
                        (void*)&scratch, (void*)&dead, (void*)&tmo_, (void*)&dfail,
                        (void*)&ebase};
        // all P "ranks" co-resident (they wait on one another): a cooperative launch
        e = coop ? cudaLaunchCooperativeKernel((const void*)km::k_p2p_emulate, dim3(P), dim3(128),
                                               args, 0, 0)
                 : cudaErrorNotSupported;
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(out, dout, sizeof(double) * nv, cudaMemcpyDeviceToHost);
    std::vector<int> hf(P, 0);
    if (e == cudaSuccess) e = cudaMemcpy(hf.data(), dfail, sizeof(int) * P, cudaMemcpyDeviceToHost);
    cudaFree(dfail);
    cudaFree(arena);
    cudaFree(dv);
    cudaFree(dout);
    cudaFree(scratch);
    cudaFree(tab);
    CK(e);
    if (failed) memcpy(failed, hf.data(), sizeof(int) * P);
    for (int r = 0; r < P; ++r)
        if (hf[r]) {
            set_error("kmeans_p2p_selftest: rank %d timed out in round %d", r, hf[r]);
            return KMEANS_ENCCL;
        }
    return KMEANS_OK;
}

kmeans_status kmeans_generate(const kmeans_mixture* mix, int64_t start, int64_t count, float* out,
                              int device, void* stream) {
    if (!mix || !out || (mix->d != 2 && mix->d != 3) || mix->M < 1 || !mix->centers ||
        mix->n_sites < 0 || (mix->n_sites > 0 && (!mix->sites || mix->site_dups < 0)) ||
        mix->N < 1 || start < 0 || count < 0 || start + count > mix->N) {
        set_error("kmeans_generate: invalid argument");
        return KMEANS_EINVAL;
    }
    if (count == 0) return KMEANS_OK;
    DeviceGuard g(device);
    kmeans_ctx* ctx = nullptr;   // for CK
    cudaStream_t s = (cudaStream_t)stream;
    const int d = mix->d;
    double *dc = nullptr, *ds = nullptr;
    CK(cudaMallocAsync(&dc, sizeof(double) * mix->M * d, s));
    if (mix->n_sites > 0) CK(cudaMallocAsync(&ds, sizeof(double) * mix->n_sites * d, s));
    CK(cudaMemcpyAsync(dc, mix->centers, sizeof(double) * mix->M * d, cudaMemcpyHostToDevice, s));
    if (ds)
        CK(cudaMemcpyAsync(ds, mix->sites, sizeof(double) * mix->n_sites * d,
                           cudaMemcpyHostToDevice, s));
    // key = mix64(seed) on the host (the same finaliser as the kernel)
    uint64_t z = mix->seed;
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    const int blocks = (int)std::min<int64_t>((count + 255) / 256, 148 * 16);
    km::k_generate<<<blocks, 256, 0, s>>>(z, d, mix->M, dc, mix->sigma, mix->n_sites,
                                          mix->site_dups, ds, mix->N, start, count, out);
    CK(cudaGetLastError());
    CK(cudaFreeAsync(dc, s));
    if (ds) CK(cudaFreeAsync(ds, s));
    CK(cudaStreamSynchronize(s));   // the host spec arrays are copied by now
    return KMEANS_OK;
}

kmeans_status kmeans_release_memory(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n ||
        device >= kMaxDevices) {
        cudaGetLastError();
        set_error("kmeans_release_memory: bad device %d", device);
        return KMEANS_EINVAL;
    }
    DeviceGuard g(device);
    std::lock_guard<std::mutex> lk(g_mem_mu);
    flush_cache_locked(device);
    return KMEANS_OK;
}

const char* kmeans_last_error(void) { return g_last_error.c_str(); }

const char* kmeans_status_string(kmeans_status s) {
    switch (s) {
        case KMEANS_OK: return "KMEANS_OK";
        case KMEANS_EINVAL: return "KMEANS_EINVAL: invalid argument";
        case KMEANS_ENONFINITE: return "KMEANS_ENONFINITE: NaN or Inf in input";
        case KMEANS_ENOMEM: return "KMEANS_ENOMEM: allocation failed";
        case KMEANS_ECUDA: return "KMEANS_ECUDA: CUDA error";
        case KMEANS_ENCCL: return "KMEANS_ENCCL: NCCL error";
        case KMEANS_ESTATE: return "KMEANS_ESTATE: call out of order";
    }
    return "unknown kmeans_status";
}

void kmeans_opts_init(kmeans_opts* o) {
    if (!o) return;
    o->device = -1;
    o->stream = nullptr;
    o->layout = KMEANS_LAYOUT_AOS;
    o->nccl_comm = nullptr;
    o->global_offset = 0;
    o->global_N = 0;
    o->flags = 0;
    o->rank = 0;
    o->nranks = 0;
    o->expected_iters = 0;
    o->comm_timeout_s = 0.0;
}

void kmeans_destroy(kmeans_ctx* ctx) {
    if (!ctx) return;
    {
        DeviceGuard g(ctx->device);
        CreateTrace tr("kmeans_destroy");
        if (ctx->stream) cudaStreamSynchronize(ctx->stream);
        tr.mark(nullptr, "stream idle");
        if (ctx->graph) cudaGraphExecDestroy(ctx->graph);
        if (ctx->graph_u) cudaGraphExecDestroy(ctx->graph_u);
        tr.mark(nullptr, "graphs destroyed");
        pool_free(ctx, ctx->X);
        pool_free(ctx, ctx->mu);
        pool_free(ctx, ctx->cneg);
        pool_free(ctx, ctx->part);
        pool_free(ctx, ctx->red);
        pool_free(ctx, ctx->st);
        pinned_state_put(ctx->st_host);
        pool_free(ctx, ctx->trace_E);
        pool_free(ctx, ctx->trace_J);
        pool_free(ctx, ctx->labels);
        pool_free(ctx, ctx->idx_dev);
        pool_free(ctx, ctx->flag);
        pool_free(ctx, ctx->cpart);
        pool_free(ctx, ctx->sbox);
        pool_free(ctx, ctx->slist);
        pool_free(ctx, ctx->scl);
        pool_free(ctx, ctx->scount);
        pool_free(ctx, ctx->heavy);
        pool_free(ctx, ctx->heavy_count);
        pool_free(ctx, ctx->htile);
        pool_free(ctx, ctx->hctr);
        pool_free(ctx, ctx->perm);
        pool_free(ctx, ctx->init_pairs);
        pool_free(ctx, ctx->init_pos);
        pool_free(ctx, ctx->cbox);
        pool_free(ctx, ctx->cand_count);
        pool_free(ctx, ctx->labels_sorted);
        pool_free(ctx, ctx->brow);
        pool_free(ctx, ctx->psync);
        pool_free(ctx, ctx->pcol);
        for (void* p : ctx->xopened) cudaIpcCloseMemHandle(p);
        if (ctx->xown) cudaFree(ctx->xown);
        pool_free(ctx, ctx->xtab);
        tr.mark(nullptr, "buffers back to the cache");
        if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
        tr.mark(nullptr, "stream destroyed");
        cudaGetLastError();
    }
    delete ctx;
}

kmeans_status kmeans_create(kmeans_ctx** out, const float* points, int64_t N, int d, int K,
                            const kmeans_opts* opts_in) {
    CreateTrace tr;
    if (!out) {
        set_error("out is NULL");
        return KMEANS_EINVAL;
    }
    *out = nullptr;
    kmeans_opts opts;
    kmeans_opts_init(&opts);
    if (opts_in) opts = *opts_in;
    const int64_t gN = opts.global_N > 0 ? opts.global_N : N;
    if (!points || N < 1 || (d != 2 && d != 3) || K < 1 || K > KMEANS_MAX_K || K > gN ||
        (opts.layout != KMEANS_LAYOUT_AOS && opts.layout != KMEANS_LAYOUT_SOA) ||
        opts.global_offset < 0 || opts.global_offset + N > gN || opts.expected_iters < 0 ||
        !(opts.comm_timeout_s >= 0.0) ||
        (!opts.nccl_comm && (opts.nranks < 0 || (opts.nranks > 0 && (opts.rank < 0 ||
                                                                    opts.rank >= opts.nranks)))) ||
        (!opts.nccl_comm && opts.nranks == 0 && gN != N)) {
        set_error("invalid argument (N=%lld d=%d K=%d global_N=%lld offset=%lld)", (long long)N, d,
                  K, (long long)gN, (long long)opts.global_offset);
        return KMEANS_EINVAL;
    }
#ifndef KMEANS_WITH_NCCL
    if (opts.nccl_comm) {
        set_error("library built without NCCL");
        return KMEANS_ENCCL;
    }
#endif
    kmeans_ctx* ctx = new kmeans_ctx();
    int dev = opts.device;
    if (dev < 0) {
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) {
            delete ctx;
            set_error("cudaGetDevice: %s", cudaGetErrorString(e));
            return KMEANS_ECUDA;
        }
    }
    ctx->device = dev;
    DeviceGuard guard(dev);
    ctx->N = N;
    ctx->d = d;
    ctx->K = K;
    ctx->global_N = gN;
    ctx->global_offset = opts.global_offset;
    ctx->comm = opts.nccl_comm;
    ctx->group = opts.nccl_comm != nullptr || opts.nranks > 0;
    if (!opts.nccl_comm && opts.nranks > 0) {   // P2P-only group
        ctx->nranks = opts.nranks;
        ctx->rank = opts.rank;
    }
    if (opts.comm_timeout_s > 0.0) ctx->comm_timeout_s = opts.comm_timeout_s;
    // padded so every full 2048-point chunk (and every large-path tile) is in bounds
    ctx->ldx = round_up(N, km::kChunkPoints) + km::kChunkPoints;
#ifdef KMEANS_WITH_NCCL
    if (ctx->comm) {
        ncclCommCount((ncclComm_t)ctx->comm, &ctx->nranks);
        ncclCommUserRank((ncclComm_t)ctx->comm, &ctx->rank);
    }
#endif
    auto fail = [&](kmeans_status s) {
        kmeans_destroy(ctx);
        return s;
    };
    cudaError_t e;
    if (opts.stream) {
        ctx->stream = (cudaStream_t)opts.stream;
    } else {
        e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            cuda_fail(nullptr, e, "cudaStreamCreate");
            return fail(KMEANS_ECUDA);
        }
        ctx->own_stream = true;
    }
    if ((opts.flags & KMEANS_FLAG_NO_SORT) && (opts.flags & KMEANS_FLAG_FORCE_SORT)) {
        set_error("KMEANS_FLAG_NO_SORT and KMEANS_FLAG_FORCE_SORT together");
        return fail(KMEANS_EINVAL);
    }
    ctx->flags = opts.flags;
    if (opts.flags & KMEANS_FLAG_NO_SORT) ctx->sorted = false;
    else if (opts.flags & KMEANS_FLAG_FORCE_SORT) ctx->sorted = true;
    else {
        ctx->sorted = K > 16 || (double)N * K * d >= 3.84e8;   // see kmeans.h
        if (ctx->sorted && K <= 16 && opts.expected_iters > 0) {
            // the Morton sort must pay for itself over the expected iterations
            // (measured at N = 1e8, d = 3, K = 16: sort +
            // gather + keys ~0.098 ns per point; full scan at ~48% of the FP32
            // lanes; pruned pass at ~6.5 TB/s)
            const double t_sort = 0.098e-9 * (double)N;
            const double t_full = 2.0 * d * K * (double)N / (0.48 * 3.72e13);
            const double t_pruned = 4.0 * d * (double)N / 6.5e12;
            if ((double)opts.expected_iters * (t_full - t_pruned) < t_sort) ctx->sorted = false;
        }
    }
    if (ctx->sorted && N > INT32_MAX) {   // the sort's permutation is int32
        if (opts.flags & KMEANS_FLAG_FORCE_SORT) {
            set_error("KMEANS_FLAG_FORCE_SORT: the sorted path holds at most 2^31 - 1 points per shard");
            return fail(KMEANS_EINVAL);
        }
        ctx->sorted = false;
    }
    kmeans_status s = configure(ctx);
    if (s != KMEANS_OK) return fail(s);
    tr.mark(ctx->stream, "stream + configure");

    const int Kpad = K + 16;
    size_t bytesX = sizeof(float) * (size_t)d * ctx->ldx;
    if (pool_alloc(ctx, &ctx->X, bytesX) != cudaSuccess ||
        pool_alloc(ctx, &ctx->mu, sizeof(double) * 2 * Kpad * d) != cudaSuccess ||
        pool_alloc(ctx, &ctx->cneg, sizeof(float4) * 2 * Kpad) != cudaSuccess ||
        pool_alloc(ctx, &ctx->part, sizeof(double) * (size_t)ctx->nE * ctx->G) != cudaSuccess ||
        pool_alloc(ctx, &ctx->red, sizeof(double) * ctx->nE) != cudaSuccess ||
        pool_alloc(ctx, &ctx->st, sizeof(DevState)) != cudaSuccess ||
        pinned_state_get(reinterpret_cast<void**>(&ctx->st_host), sizeof(DevState)) != cudaSuccess ||
        pool_alloc(ctx, &ctx->idx_dev, sizeof(int64_t) * K) != cudaSuccess ||
        ((ctx->path == 0 || ctx->sorted) &&
         pool_alloc(ctx, &ctx->cpart, sizeof(double) * ctx->row_stride * (size_t)ctx->n_chunks) !=
             cudaSuccess) ||
        (ctx->sorted && ctx->path == 1 &&
         (pool_alloc(ctx, &ctx->sbox, sizeof(float) * 2 * d * (size_t)ctx->n_super) != cudaSuccess ||
          pool_alloc(ctx, &ctx->slist, sizeof(int) * (size_t)K * ctx->n_super) != cudaSuccess ||
          pool_alloc(ctx, &ctx->scl, sizeof(float4) * (size_t)K * ctx->n_super) != cudaSuccess ||
          pool_alloc(ctx, &ctx->scount, sizeof(int) * (size_t)ctx->n_super) != cudaSuccess ||
          pool_alloc(ctx, &ctx->heavy, sizeof(int) * (size_t)ctx->n_chunks) != cudaSuccess ||
          pool_alloc(ctx, &ctx->heavy_count, sizeof(int)) != cudaSuccess ||
          pool_alloc(ctx, &ctx->htile, sizeof(double2) * km::kHeavyWarps * (size_t)ctx->n_chunks) !=
              cudaSuccess ||
          pool_alloc(ctx, &ctx->hctr, sizeof(int) * (size_t)ctx->n_chunks) != cudaSuccess)) ||
        pool_alloc(ctx, &ctx->flag, sizeof(int)) != cudaSuccess ||
        (ctx->fused && pool_alloc(ctx, &ctx->brow, sizeof(double) * 2 * (size_t)ctx->nE *
                                                       ctx->fused_grid) != cudaSuccess) ||
        (ctx->persist &&
         (pool_alloc(ctx, &ctx->psync, sizeof(km::PersistSync)) != cudaSuccess ||
          pool_alloc(ctx, &ctx->pcol, sizeof(double) * ctx->nE *
                                          (size_t)(ctx->persist_grid + km::kMaxBlockGroups)) !=
              cudaSuccess))) {
        cudaGetLastError();
        set_error("device allocation failed (%zu bytes of points)", bytesX);
        return fail(KMEANS_ENOMEM);
    }
    tr.mark(ctx->stream, "pool allocations");
    if ((s = ensure_trace(ctx, 64)) != KMEANS_OK) return fail(s);
    if (cudaMemsetAsync(ctx->mu, 0, sizeof(double) * 2 * Kpad * d, ctx->stream) != cudaSuccess ||
        cudaMemsetAsync(ctx->flag, 0, sizeof(int), ctx->stream) != cudaSuccess ||
        ((ctx->path == 0 || ctx->sorted) &&
         cudaMemsetAsync(ctx->cpart, 0, sizeof(double) * ctx->row_stride * (size_t)ctx->n_chunks,
                         ctx->stream) != cudaSuccess) ||
        cudaMemsetAsync(ctx->st, 0, sizeof(DevState), ctx->stream) != cudaSuccess ||
        (ctx->hctr &&
         cudaMemsetAsync(ctx->hctr, 0, sizeof(int) * (size_t)ctx->n_chunks, ctx->stream) != cudaSuccess)) {
        cuda_fail(ctx, cudaGetLastError(), "cudaMemsetAsync");
        return fail(KMEANS_ECUDA);
    }

    // Ingest: host or device input -> padded SoA, with the non-finite check.
    cudaPointerAttributes attr;
    bool on_device = false;
    if (cudaPointerGetAttributes(&attr, points) == cudaSuccess)
        on_device = attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
    cudaGetLastError();
    const float* src = points;
    float* staging = nullptr;
    if (!on_device) {
        if (pool_alloc(ctx, &staging, sizeof(float) * (size_t)N * d) != cudaSuccess) {
            cudaGetLastError();
            set_error("staging allocation failed");
            return fail(KMEANS_ENOMEM);
        }
        e = cudaMemcpyAsync(staging, points, sizeof(float) * (size_t)N * d,
                            cudaMemcpyHostToDevice, ctx->stream);
        if (e != cudaSuccess) {
            pool_free(ctx, staging);
            cuda_fail(ctx, e, "H2D points");
            return fail(KMEANS_ECUDA);
        }
        src = staging;
    }
    tr.mark(ctx->stream, on_device ? "memsets" : "memsets + H2D");
    const int64_t si = opts.layout == KMEANS_LAYOUT_AOS ? d : 1;
    const int64_t sj = opts.layout == KMEANS_LAYOUT_AOS ? 1 : N;
    if (!ctx->sorted) {
        int blocks = (int)std::min<int64_t>((ctx->ldx + 255) / 256, 148 * 16);
        km::k_prep<<<blocks, 256, 0, ctx->stream>>>(src, N, d, si, sj, ctx->X, ctx->ldx,
                                                    ctx->flag);
        ctx->launches += 1;
    } else {
        s = sort_points(ctx, src, si, sj, tr);
        if (s != KMEANS_OK) {
            cudaStreamSynchronize(ctx->stream);
            if (staging) pool_free(ctx, staging);
            return fail(s);
        }
    }
    int hflag = 0;
    e = cudaMemcpyAsync(&hflag, ctx->flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (staging) pool_free(ctx, staging);
    if (e != cudaSuccess) {
        cuda_fail(ctx, e, "k_prep");
        return fail(KMEANS_ECUDA);
    }
    tr.mark(ctx->stream, "done");
    if (hflag) {
        set_error("points contain NaN or Inf");
        return fail(KMEANS_ENONFINITE);
    }
    *out = ctx;
    return KMEANS_OK;
}

kmeans_status kmeans_start(kmeans_ctx* ctx, const int64_t* init_idx, const double* centroids,
                           double tol, int max_iter) {
    CHECK_CTX(ctx);
    if ((!init_idx && !centroids) || !(tol >= 0.0) || max_iter < 1) {
        set_error("kmeans_start: need init_idx or centroids, tol >= 0, max_iter >= 1");
        return KMEANS_EINVAL;
    }
    if (ctx->group && !ctx->comm && !ctx->p2p) {
        set_error("P2P-only group: call kmeans_p2p_handle / kmeans_p2p_open first");
        return KMEANS_ESTATE;
    }
    DeviceGuard g(ctx->device);
    kmeans_status s;
    if (init_idx) {
        std::vector<int64_t> idx;
        if ((s = fetch_init_idx(ctx, init_idx, idx)) != KMEANS_OK) return s;
        CK(cudaMemcpyAsync(ctx->idx_dev, idx.data(), sizeof(int64_t) * ctx->K,
                           cudaMemcpyHostToDevice, ctx->stream));
        const int n = ctx->K * ctx->d;
        std::vector<int2> pairs;
        if (ctx->sorted) {
            // sorted positions of the local initial indices (one pass over perm)
            for (int k = 0; k < ctx->K; ++k) {
                const int64_t i = idx[k] - ctx->global_offset;
                if (i >= 0 && i < ctx->N) pairs.push_back(make_int2((int)i, k));
            }
            std::sort(pairs.begin(), pairs.end(),
                      [](const int2& a, const int2& b) { return a.x < b.x; });
            CK(cudaMemsetAsync(ctx->init_pos, 0xff, sizeof(int32_t) * ctx->K, ctx->stream));
            if (!pairs.empty()) {
                CK(cudaMemcpyAsync(ctx->init_pairs, pairs.data(), sizeof(int2) * pairs.size(),
                                   cudaMemcpyHostToDevice, ctx->stream));
                const int blocks = (int)std::min<int64_t>((ctx->N + 255) / 256, 148 * 8);
                km::k_find_pos<<<blocks, 256, 0, ctx->stream>>>(ctx->perm, ctx->N, ctx->init_pairs,
                                                                 (int)pairs.size(), ctx->init_pos);
                ctx->launches += 1;
            }
        }
        km::k_init_gather<<<(n + 255) / 256, 256, 0, ctx->stream>>>(
            ctx->X, ctx->d, ctx->K, ctx->idx_dev, ctx->global_offset, ctx->N,
            ctx->sorted ? ctx->init_pos : nullptr, ctx->mu);
        ctx->launches += 1;
        CK(cudaGetLastError());
        // CC1: assemble mu^0 from the owners (exact: one x plus zeros)
        if ((s = allreduce(ctx, ctx->mu, (size_t)n)) != KMEANS_OK) return s;
        DevState h;   // waits (idx vector lifetime) and reports a failed exchange
        if ((s = read_state(ctx, &h)) != KMEANS_OK) return s;
    } else {
        std::vector<double> c;
        if ((s = fetch_centroids(ctx, centroids, c)) != KMEANS_OK) return s;
        CK(cudaMemcpyAsync(ctx->mu, c.data(), sizeof(double) * c.size(), cudaMemcpyHostToDevice,
                           ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    if ((s = ensure_trace(ctx, std::min(max_iter, kTraceCap))) != KMEANS_OK) return s;
    if (ctx->persist) {   // the persistent kernel's counters start from zero
        CK(cudaMemsetAsync(ctx->psync, 0, sizeof(km::PersistSync), ctx->stream));
    }
    ctx->assigned = false;
    ctx->gen += 1;   // new epochs for the iteration exchanges of this run
    if ((s = write_state(ctx, 0, 0, max_iter, tol)) != KMEANS_OK) return s;
    return stage_centroids(ctx);
}

kmeans_status kmeans_iterate(kmeans_ctx* ctx, int n) {
    CHECK_CTX(ctx);
    if (n < 0) {
        set_error("n < 0");
        return KMEANS_EINVAL;
    }
    DeviceGuard g(ctx->device);
    kmeans_status s = ensure_graph(ctx);
    if (s != KMEANS_OK) return s;
    if (ctx->fused) {   // n iterations (or until the stop rule) in one cooperative launch
        if (n == 0) return KMEANS_OK;
        FusedFn ff = pick_fused(ctx->d, ctx->K);
        int n_iter = n;
        void* args[] = {(void*)&ctx->X,     (void*)&ctx->N,         (void*)&ctx->K,
                        (void*)&ctx->n_chunks, (void*)&ctx->mu,     (void*)&ctx->st,
                        (void*)&ctx->trace_E, (void*)&ctx->trace_J, (void*)&ctx->trace_cap,
                        (void*)&ctx->brow,  (void*)&ctx->red,       (void*)&n_iter};
        CK(cudaLaunchCooperativeKernel((const void*)ff, dim3(ctx->fused_grid),
                                       dim3(km::kFusedWarps * 32), args, ctx->fused_smem,
                                       ctx->stream));
        ctx->launches += 1;
        return KMEANS_OK;
    }
    if (persist_active(ctx)) {   // n iterations (or until the stop rule) in one launch
        if (n == 0) return KMEANS_OK;
        PersistFn pf = pick_persist(ctx->d, ctx->chunk_points);
        // the flag counts this launch's iterations from zero
        CK(cudaMemsetAsync(ctx->psync, 0, sizeof(unsigned long long), ctx->stream));
        km::P2PView pv{};
        if (ctx->p2p) pv = p2p_view(ctx);
        else pv.P = 1;
        int n_iter = n;
        const float* X = ctx->X;
        const float* cbox = ctx->cbox;
        double* gcol = ctx->pcol + (size_t)ctx->nE * ctx->persist_grid;
        void* args[] = {(void*)&X,           (void*)&ctx->N,        (void*)&ctx->K,
                        (void*)&ctx->n_chunks, (void*)&cbox,        (void*)&ctx->cneg,
                        (void*)&ctx->mu,     (void*)&ctx->st,       (void*)&ctx->trace_E,
                        (void*)&ctx->trace_J, (void*)&ctx->trace_cap, (void*)&ctx->pcol,
                        (void*)&gcol,        (void*)&ctx->red,      (void*)&ctx->psync,
                        (void*)&ctx->keep_n,
                        (void*)&n_iter,      (void*)&pv};
        const int W = ctx->d == 2 ? km::PersistCfg<2>::kWarps : km::PersistCfg<3>::kWarps;
        CK(cudaLaunchCooperativeKernel((const void*)pf, dim3(ctx->persist_grid), dim3(W * 32),
                                       args, ctx->persist_smem, ctx->stream));
        ctx->launches += 1;
        return KMEANS_OK;
    }
    int i = 0;
    for (; i + kGraphUnroll <= n; i += kGraphUnroll)
        CK(cudaGraphLaunch(ctx->graph_u, ctx->stream));
    for (; i < n; ++i) CK(cudaGraphLaunch(ctx->graph, ctx->stream));
    ctx->launches += (int64_t)n * kernels_per_iter(ctx);
    return KMEANS_OK;
}

kmeans_status kmeans_poll(kmeans_ctx* ctx, int* iters, int* done, double* E, double* J) {
    CHECK_CTX(ctx);
    DeviceGuard g(ctx->device);
    DevState h;
    kmeans_status s = read_state(ctx, &h);
    if (s != KMEANS_OK) return s;
    if (iters) *iters = h.t;
    if (done) *done = h.done;
    if (E) *E = h.E;
    if (J) *J = h.J;
    return KMEANS_OK;
}

kmeans_status kmeans_read_centroids(kmeans_ctx* ctx, double* centroids) {
    CHECK_CTX(ctx);
    if (!centroids) {
        set_error("centroids is NULL");
        return KMEANS_EINVAL;
    }
    DeviceGuard g(ctx->device);
    DevState h;
    kmeans_status s = read_state(ctx, &h);
    if (s != KMEANS_OK) return s;
    const size_t n = (size_t)ctx->K * ctx->d;
    CK(cudaMemcpyAsync(centroids, ctx->mu + (size_t)(h.t & 1) * n, sizeof(double) * n,
                       cudaMemcpyDefault, ctx->stream));
    return sync(ctx);
}

kmeans_status kmeans_final_labels(kmeans_ctx* ctx, int32_t* labels) {
    CHECK_CTX(ctx);
    if (!labels) {
        set_error("labels is NULL");
        return KMEANS_EINVAL;
    }
    DeviceGuard g(ctx->device);
    DevState h;
    kmeans_status s = read_state(ctx, &h);
    if (s != KMEANS_OK) return s;
    if (h.t < 1) {
        set_error("no completed iteration");
        return KMEANS_ESTATE;
    }
    // z^t = argmin over fl32(mu^{t-1}): mu_sel = 1 selects buffer (t-1) & 1.
    if ((s = launch_assign(ctx, km::kModeLabels, 1, 1)) != KMEANS_OK) return s;
    CK(cudaMemcpyAsync(labels, ctx->labels, sizeof(int32_t) * ctx->N, cudaMemcpyDefault,
                       ctx->stream));
    return sync(ctx);
}

kmeans_status kmeans_assign(kmeans_ctx* ctx, const double* centroids, int32_t* labels,
                            double* inertia, int64_t* counts, double* sums) {
    CHECK_CTX(ctx);
    if (!centroids) {
        set_error("centroids is NULL");
        return KMEANS_EINVAL;
    }
    if (ctx->group && !ctx->comm && !ctx->p2p) {
        set_error("P2P-only group: call kmeans_p2p_handle / kmeans_p2p_open first");
        return KMEANS_ESTATE;
    }
    DeviceGuard g(ctx->device);
    kmeans_status s;
    std::vector<double> c;
    if ((s = fetch_centroids(ctx, centroids, c)) != KMEANS_OK) return s;
    ctx->assigned = false;
    const size_t n = c.size();
    CK(cudaMemcpyAsync(ctx->mu, c.data(), sizeof(double) * n, cudaMemcpyHostToDevice,
                       ctx->stream));
    if ((s = write_state(ctx, 0, 0, 0x7fffffff, -1.0)) != KMEANS_OK) return s;
    if ((s = stage_centroids(ctx)) != KMEANS_OK) return s;
    const int mode = km::kModeReduce | (labels ? km::kModeLabels : 0);
    if ((s = launch_assign(ctx, mode, 0, 1)) != KMEANS_OK) return s;
    if ((s = launch_merge(ctx, 1)) != KMEANS_OK) return s;
    if ((s = allreduce(ctx, ctx->red, ctx->nE)) != KMEANS_OK) return s;
    std::vector<double> red(ctx->nE);
    CK(cudaMemcpyAsync(red.data(), ctx->red, sizeof(double) * ctx->nE, cudaMemcpyDeviceToHost,
                       ctx->stream));
    DevState h;   // the kernels (and the exchange) completed without error ...
    if ((s = read_state(ctx, &h)) != KMEANS_OK) return s;
    if (labels) {   // ... before any output is written
        CK(cudaMemcpyAsync(labels, ctx->labels, sizeof(int32_t) * ctx->N, cudaMemcpyDefault,
                           ctx->stream));
        if ((s = sync(ctx)) != KMEANS_OK) return s;
    }
    const int K = ctx->K, d = ctx->d;
    if (inertia) CK(cudaMemcpy(inertia, &red[(size_t)K * d + K], sizeof(double), cudaMemcpyDefault));
    if (counts) {
        std::vector<int64_t> cn(K);
        for (int k = 0; k < K; ++k) cn[k] = (int64_t)red[(size_t)K * d + k];
        CK(cudaMemcpy(counts, cn.data(), sizeof(int64_t) * K, cudaMemcpyDefault));
    }
    if (sums) CK(cudaMemcpy(sums, red.data(), sizeof(double) * K * d, cudaMemcpyDefault));
    ctx->mu_host = c;
    ctx->assigned = true;
    return KMEANS_OK;
}

kmeans_status kmeans_update(kmeans_ctx* ctx, double* centroids, double* shift_E) {
    CHECK_CTX(ctx);
    if (!ctx->assigned) {
        set_error("kmeans_update needs a preceding kmeans_assign");
        return KMEANS_ESTATE;
    }
    DeviceGuard g(ctx->device);
    kmeans_status s;
    if ((s = launch_update(ctx)) != KMEANS_OK) return s;
    DevState h;
    if ((s = read_state(ctx, &h)) != KMEANS_OK) return s;
    const size_t n = (size_t)ctx->K * ctx->d;
    if (centroids) {
        CK(cudaMemcpyAsync(centroids, ctx->mu + n /* buffer 1 = mu^{t+1} */, sizeof(double) * n,
                           cudaMemcpyDefault, ctx->stream));
        if ((s = sync(ctx)) != KMEANS_OK) return s;
    }
    if (shift_E) CK(cudaMemcpy(shift_E, &h.E, sizeof(double), cudaMemcpyDefault));
    ctx->assigned = false;
    return KMEANS_OK;
}

kmeans_status kmeans_fit_ctx(kmeans_ctx* ctx, const int64_t* init_idx, double tol, int max_iter,
                             int32_t* labels, double* centroids, int* iters, double* inertia,
                             double* E_trace, double* J_trace) {
    CHECK_CTX(ctx);
    if (!init_idx || !centroids || !iters || !inertia || !(tol >= 0.0) || max_iter < 1) {
        set_error("kmeans_fit_ctx: invalid argument");
        return KMEANS_EINVAL;
    }
    DeviceGuard g(ctx->device);
    kmeans_status s = kmeans_start(ctx, init_idx, nullptr, tol, max_iter);
    if (s != KMEANS_OK) return s;
    if ((E_trace || J_trace) && (s = ensure_trace(ctx, max_iter)) != KMEANS_OK) return s;
    // Graph replays in chunks; the device stop flag turns surplus iterations
    // into no-ops, the host polls once per chunk.
    int chunk = 4, t = 0, done = 0;
    while (!done) {
        const int n = std::min(chunk, max_iter - t);
        if ((s = kmeans_iterate(ctx, n)) != KMEANS_OK) return s;
        if ((s = kmeans_poll(ctx, &t, &done, nullptr, nullptr)) != KMEANS_OK) return s;
        chunk = std::min(chunk * 2, 64);
    }
    DevState h;
    if ((s = read_state(ctx, &h)) != KMEANS_OK) return s;
    if (labels && (s = kmeans_final_labels(ctx, labels)) != KMEANS_OK) return s;
    const size_t n = (size_t)ctx->K * ctx->d;
    CK(cudaMemcpyAsync(centroids, ctx->mu + (size_t)(h.t & 1) * n, sizeof(double) * n,
                       cudaMemcpyDefault, ctx->stream));
    if (E_trace)
        CK(cudaMemcpyAsync(E_trace, ctx->trace_E, sizeof(double) * h.t, cudaMemcpyDefault,
                           ctx->stream));
    if (J_trace)
        CK(cudaMemcpyAsync(J_trace, ctx->trace_J, sizeof(double) * h.t, cudaMemcpyDefault,
                           ctx->stream));
    if ((s = sync(ctx)) != KMEANS_OK) return s;
    CK(cudaMemcpy(iters, &h.t, sizeof(int), cudaMemcpyDefault));
    CK(cudaMemcpy(inertia, &h.J, sizeof(double), cudaMemcpyDefault));
    return KMEANS_OK;
}

kmeans_status kmeans_fit(const float* points, int64_t N, int d, int K, const int64_t* init_idx,
                         double tol, int max_iter, int32_t* labels, double* centroids, int* iters,
                         double* inertia) {
    if (!init_idx || !centroids || !iters || !inertia || !(tol >= 0.0) || max_iter < 1) {
        set_error("kmeans_fit: invalid argument");
        return KMEANS_EINVAL;
    }
    kmeans_ctx* ctx = nullptr;
    kmeans_opts o;
    kmeans_opts_init(&o);
    o.expected_iters = max_iter;   // the path choice weighs the sort against the run
    kmeans_status s = kmeans_create(&ctx, points, N, d, K, &o);
    if (s != KMEANS_OK) return s;
    s = kmeans_fit_ctx(ctx, init_idx, tol, max_iter, labels, centroids, iters, inertia, nullptr,
                       nullptr);
    kmeans_destroy(ctx);
    return s;
}

static kmeans_status enqueue_stage(kmeans_ctx* ctx, int n, int stage);

kmeans_status kmeans_profile_assign(kmeans_ctx* ctx, int n) {
    CHECK_CTX(ctx);
    if (n < 0) {
        set_error("n < 0");
        return KMEANS_EINVAL;
    }
    DeviceGuard g(ctx->device);
    return enqueue_stage(ctx, n, 0);
}

static kmeans_status enqueue_stage(kmeans_ctx* ctx, int n, int stage) {
    for (int i = 0; i < n; ++i) {
        kmeans_status s;
        if (stage == 0 || stage == 1)
            s = launch_assign(ctx, km::kModeReduce, 0, 1, stage == 0 ? 3 : 1);
        else if (stage == 2)
            s = launch_assign(ctx, km::kModeReduce, 0, 1, 2);
        else
            s = launch_merge(ctx, 1);
        if (s != KMEANS_OK) return s;
    }
    return KMEANS_OK;
}

kmeans_status kmeans_profile_stage(kmeans_ctx* ctx, int n, int stage, float* ms_per_launch) {
    CHECK_CTX(ctx);
    if (n < 0 || stage < 0 || stage > 3) {
        set_error("n < 0 or stage not in {0, 1, 2, 3}");
        return KMEANS_EINVAL;
    }
    DeviceGuard g(ctx->device);
    if (!ms_per_launch) return enqueue_stage(ctx, n, stage);
    // timed: the n launches captured in one graph (no host launch cost in the
    // measurement), run once untimed, then once between two events
    if (n == 0) {
        *ms_per_launch = 0.f;
        return KMEANS_OK;
    }
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    const int64_t launches0 = ctx->launches;
    CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    kmeans_status s = enqueue_stage(ctx, n, stage);
    cudaError_t ce = cudaStreamEndCapture(ctx->stream, &graph);
    if (s != KMEANS_OK) {
        if (graph) cudaGraphDestroy(graph);
        return s;
    }
    CK(ce);
    ctx->launches = launches0 + 2 * (ctx->launches - launches0);   // two graph runs
    ce = cudaGraphInstantiate(&exec, graph, 0);
    if (ce == cudaSuccess) ce = cudaEventCreate(&e0);
    if (ce == cudaSuccess) ce = cudaEventCreate(&e1);
    if (ce == cudaSuccess) ce = cudaGraphLaunch(exec, ctx->stream);
    if (ce == cudaSuccess) ce = cudaEventRecord(e0, ctx->stream);
    if (ce == cudaSuccess) ce = cudaGraphLaunch(exec, ctx->stream);
    if (ce == cudaSuccess) ce = cudaEventRecord(e1, ctx->stream);
    if (ce == cudaSuccess) ce = cudaEventSynchronize(e1);
    float ms = 0.f;
    if (ce == cudaSuccess) ce = cudaEventElapsedTime(&ms, e0, e1);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (exec) cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    CK(ce);
    *ms_per_launch = ms / n;
    return KMEANS_OK;
}

kmeans_status kmeans_candidate_stats(kmeans_ctx* ctx, double* mean, int* max, int64_t* single,
                                     int64_t* chunks) {
    CHECK_CTX(ctx);
    if (!ctx->sorted) {
        set_error("candidate statistics exist only on the sorted path");
        return KMEANS_ESTATE;
    }
    DeviceGuard g(ctx->device);
    std::vector<int> c(ctx->n_chunks);
    CK(cudaMemcpyAsync(c.data(), ctx->cand_count, sizeof(int) * c.size(), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    double sum = 0.0;
    int mx = 0;
    int64_t one = 0;
    for (int v : c) {
        sum += v;
        mx = std::max(mx, v);
        one += (v == 1);
    }
    if (getenv("KMEANS_TRACE") && *getenv("KMEANS_TRACE") && *getenv("KMEANS_TRACE") != '0') {
        std::map<int, int64_t> h;   // candidates per chunk -> chunks (tuning aid)
        for (int v : c) h[std::min(v, 65)] += 1;
        fprintf(stderr, "[kmeans_candidate_stats] chunks by candidate count:");
        for (auto& kv : h) fprintf(stderr, " %d:%lld", kv.first, (long long)kv.second);
        fprintf(stderr, "\n");
    }
    if (mean) *mean = c.empty() ? 0.0 : sum / c.size();
    if (max) *max = mx;
    if (single) *single = one;
    if (chunks) *chunks = (int64_t)c.size();
    return KMEANS_OK;
}

kmeans_status kmeans_get_stream(kmeans_ctx* ctx, void** stream) {
    CHECK_CTX(ctx);
    if (!stream) return KMEANS_EINVAL;
    *stream = (void*)ctx->stream;
    return KMEANS_OK;
}

kmeans_status kmeans_get_info(kmeans_ctx* ctx, kmeans_info* info) {
    if (!ctx || !info) {
        set_error("NULL argument");
        return KMEANS_EINVAL;
    }
    info->N = ctx->N;
    info->global_N = ctx->global_N;
    info->global_offset = ctx->global_offset;
    info->ldx = ctx->ldx;
    info->d = ctx->d;
    info->K = ctx->K;
    info->grid = (ctx->path == 0 || ctx->sorted) ? ctx->n_chunks : ctx->G;
    info->block = ctx->tpb;
    info->smem_bytes = ctx->smem;
    info->path = ctx->path;
    info->kernels_per_iter = kernels_per_iter(ctx);
    info->kernel_launches = ctx->launches;
    info->nranks = ctx->nranks;
    info->sorted = ctx->sorted ? 1 : 0;
    info->fused = ctx->fused ? 1 : 0;
    info->fused_grid = ctx->fused_grid;
    info->persistent = persist_active(ctx) ? 1 : 0;
    info->persist_grid = ctx->persist_grid;
    info->rank = ctx->rank;
    return KMEANS_OK;
}

kmeans_status kmeans_comm_unique_id(unsigned char id[128]) {
    if (!id) return KMEANS_EINVAL;
#ifdef KMEANS_WITH_NCCL
    ncclUniqueId u;
    ncclResult_t r = ncclGetUniqueId(&u);
    if (r != ncclSuccess) {
        set_error("ncclGetUniqueId: %s", ncclGetErrorString(r));
        return KMEANS_ENCCL;
    }
    memcpy(id, u.internal, 128);
    return KMEANS_OK;
#else
    set_error("library built without NCCL");
    return KMEANS_ENCCL;
#endif
}

kmeans_status kmeans_comm_init(void** comm, int nranks, const unsigned char id[128], int rank,
                               int device) {
    if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks) {
        set_error("kmeans_comm_init: invalid argument");
        return KMEANS_EINVAL;
    }
#ifdef KMEANS_WITH_NCCL
    if (device >= 0) cudaSetDevice(device);
    ncclUniqueId u;
    memcpy(u.internal, id, 128);
    ncclComm_t c = nullptr;
    ncclResult_t r = ncclCommInitRank(&c, nranks, u, rank);
    if (r != ncclSuccess) {
        set_error("ncclCommInitRank: %s", ncclGetErrorString(r));
        return KMEANS_ENCCL;
    }
    *comm = (void*)c;
    return KMEANS_OK;
#else
    (void)device;
    set_error("library built without NCCL");
    return KMEANS_ENCCL;
#endif
}

kmeans_status kmeans_comm_destroy(void* comm) {
    if (!comm) return KMEANS_OK;
#ifdef KMEANS_WITH_NCCL
    {   // already aborted (and freed) by a context that timed out on it
        std::lock_guard<std::mutex> lk(g_abort_mu);
        auto it = std::find(g_aborted.begin(), g_aborted.end(), comm);
        if (it != g_aborted.end()) {
            g_aborted.erase(it);
            return KMEANS_OK;
        }
    }
    ncclResult_t r = ncclCommDestroy((ncclComm_t)comm);
    if (r != ncclSuccess) {
        set_error("ncclCommDestroy: %s", ncclGetErrorString(r));
        return KMEANS_ENCCL;
    }
    return KMEANS_OK;
#else
    set_error("library built without NCCL");
    return KMEANS_ENCCL;
#endif
}

}  // extern "C"
