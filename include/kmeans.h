/*
 * kmeans.h -- C ABI of the B200-native Lloyd iteration (arXiv 2405.12052).
 *
 * The operation is one Lloyd iteration of PAPER.md (§THE LLOYD'S ALGORITHM,
 * lines 39-64, and §SERIAL LLOYD'S ALGORITHM, lines 65-70):
 *
 *   reassignment  z_i^{t+1} = argmin_k ||x_i - mu_k^t||_2^2
 *   mean          mu_k^{t+1} = sum_i 1(z_i^{t+1}=k) x_i
 *                              / sum_i 1(z_i^{t+1}=k)
 *   error         E = sum_k ||mu_k^{t+1} - mu_k^t||_2^2
 *   stop          E < tol, or t = max_iter
 *
 * with the numerical contract of DESIGN.md "Readings" (R1-R16): fp32 points,
 * centroids staged once per iteration fp64 -> fp32 (round to nearest even),
 * form-D distance e_j = x_j - c_j, s = e_0*e_0, s = fma(e_j, e_j, s), argmin
 * with the lowest index winning ties, fp64 sums / means / E / inertia, int64
 * counts, empty clusters keep mu^t, labels 0-based.
 *
 * Conventions for every function:
 *   - Returns a kmeans_status; nothing throws across the ABI.
 *   - Validation happens before any device work; outputs are written only on
 *     KMEANS_OK.
 *   - Every pointer argument may be host memory (pageable or pinned) or device
 *     memory of the context's device (CUDA unified addressing decides); the
 *     caller owns it, and the library never keeps it past the call.
 *   - After KMEANS_ECUDA or KMEANS_ENCCL a context is unusable (sticky error);
 *     only kmeans_destroy is valid.  (Exception: a failed kmeans_p2p_open
 *     leaves the context usable -- see there.)
 *   - A distributed context never waits forever for a peer: an exchange that
 *     a peer does not join within opts.comm_timeout_s fails the call with
 *     KMEANS_ENCCL (P2P exchange: a bounded spin in the kernel; NCCL: the
 *     host polls ncclCommGetAsyncError and aborts the communicator).
 *   - A context is not thread-safe; distinct contexts are independent.
 *   - kmeans_last_error() returns a thread-local message for the last failure.
 *
 * Supported shapes: d in {2, 3} (the paper's 2D and 3D datasets, PAPER.md:37,
 * 72); 1 <= K <= KMEANS_MAX_K; K <= N (global N when distributed).
 */
#ifndef KMEANS_H
#define KMEANS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KMEANS_ABI_VERSION 3   /* 3: kmeans_opts.rank / nranks / expected_iters / comm_timeout_s,
                                  bounded P2P waits, kmeans_p2p_selftest dead-rank arguments */
#define KMEANS_MAX_K 1024

typedef struct kmeans_ctx kmeans_ctx; /* opaque */

typedef enum kmeans_status {
    KMEANS_OK = 0,
    KMEANS_EINVAL = -1,     /* NULL where required; N < 1; d not in {2,3}; K < 1;
                               K > N or K > KMEANS_MAX_K; tol < 0 or NaN; max_iter < 1;
                               init_idx entry outside [0, N) or repeated */
    KMEANS_ENONFINITE = -2, /* NaN/Inf in points or centroids */
    KMEANS_ENOMEM = -3,     /* device or host allocation failed */
    KMEANS_ECUDA = -4,      /* CUDA error (sticky) */
    KMEANS_ENCCL = -5,      /* NCCL error, or library built without NCCL (sticky) */
    KMEANS_ESTATE = -6      /* call out of order, e.g. kmeans_update before kmeans_assign */
} kmeans_status;

typedef enum kmeans_layout {
    KMEANS_LAYOUT_AOS = 0,  /* N x d row-major (point-major), the default */
    KMEANS_LAYOUT_SOA = 1   /* d x N row-major, the paper's X in R^{d x N} */
} kmeans_layout;

typedef struct kmeans_opts {
    int device;             /* CUDA ordinal; -1 = current device */
    void* stream;           /* cudaStream_t to run on; NULL = a context-owned stream */
    int layout;             /* kmeans_layout of `points` */
    void* nccl_comm;        /* ncclComm_t (see kmeans_comm_init); NULL = single GPU.
                               When set, the context is one rank of a data-parallel
                               group: it owns the contiguous shard
                               [global_offset, global_offset + N) of global_N points,
                               and every compute call is collective over the group. */
    int64_t global_offset;  /* first global index of this rank's shard */
    int64_t global_N;       /* total points over all ranks; 0 = N */
    int flags;              /* KMEANS_FLAG_* bits */
    int rank;               /* without nccl_comm: this rank of a P2P-only group (0 <= rank < nranks) */
    int nranks;             /* without nccl_comm: group size; 0 = not distributed.  A P2P-only
                               group exchanges through kmeans_p2p_handle / kmeans_p2p_open
                               (no NCCL); the exchange must be opened before kmeans_start /
                               kmeans_assign (KMEANS_ESTATE otherwise).  With nccl_comm the
                               communicator's rank and size are used and these are ignored. */
    int expected_iters;     /* hint for the path choice: Lloyd iterations the caller will run on
                               this context (0 = unknown).  The sorted path costs a one-time
                               space-filling-curve sort at create (about 0.1 ms per million
                               points) that
                               pays off only over enough iterations; kmeans_fit passes
                               max_iter. */
    double comm_timeout_s;  /* distributed: seconds to wait for a peer in an exchange before
                               failing with KMEANS_ENCCL; 0 = 60 s */
} kmeans_opts;

/* kmeans_opts.flags */
#define KMEANS_FLAG_NO_SORT 1     /* keep the caller's point order: full-scan assign kernels */
#define KMEANS_FLAG_FORCE_SORT 2  /* always use the sorted (pruned) path */
#define KMEANS_FLAG_BIG_CHUNKS 8  /* sorted path, K <= 16: 2048-point chunks at any N
                                     (default: from 4e7 points per shard) */
#define KMEANS_FLAG_PERSIST 16    /* sorted path, K <= 16, shards of >= 256 x (SMs x warps per
                                     block) points: run kmeans_iterate's iterations inside ONE
                                     persistent kernel (k_persist_iterate: static unit ranges per
                                     warp, block / grid last-arriver merges, update and P2P
                                     exchange in the kernel, a device flag per iteration; SURVEY.md
                                     NEXT-1) instead of the per-iteration kernel graph.  Opt-in:
                                     measured slower than the graph */
#define KMEANS_FLAG_NO_FUSED 4    /* full-scan path: never use the one-launch
                                     multi-iteration kernel (k_fused_iterate) that
                                     kmeans_iterate / kmeans_fit_ctx use for small
                                     single-GPU shards (<= 4 x 8 x SMs chunks of 2048) */
/* Default (neither flag): the sorted path -- the shard is put in space-filling-
 * curve order (Hilbert in 3D and for 2D shards below 4e7 points, Z-curve
 * otherwise) once at create and each 1024-point chunk prunes the centroids that provably
 * cannot be its points' argmin (exact; labels are returned in the caller's
 * order) -- when K > 16 or N*K*d >= 3.84e8 (N >= 8e6 at K = 16, d = 3);
 * below that the full scan is faster (the pruned kernel has a fixed per-chunk
 * latency, measured in DESIGN.md section 5).  With opts.expected_iters > 0 and
 * K <= 16 the sort must also pay for itself over that many iterations
 * ("Path choice").  Shards of more than 2^31 - 1
 * points always take the full scan (KMEANS_EINVAL with FORCE_SORT).  Both
 * flags: KMEANS_EINVAL. */

/* Fills *opts with the defaults above. */
void kmeans_opts_init(kmeans_opts* opts);

/* Creates a context holding a device-resident copy of `points` (N points of
 * dimension d, layout per opts), laid out internally as SoA fp32.  K is the
 * number of clusters every later call uses.  Checks every coordinate for
 * NaN/Inf (KMEANS_ENONFINITE). */
kmeans_status kmeans_create(kmeans_ctx** out, const float* points, int64_t N, int d, int K,
                            const kmeans_opts* opts);

/* One reassignment step plus the fused per-cluster reduction at the given
 * centroids mu^t (K x d fp64, row-major).  Distributed: the
 * partials are summed over all ranks (collective), labels stay local.
 * Outputs (each may be NULL):
 *   labels  : N int32, z_i^{t+1} for this rank's points
 *   inertia : J(z^{t+1}, mu^t) = sum_i ||x_i - c_{z_i}||^2 (fp32 distances summed
 *             in fp64), global
 *   counts  : K int64, global
 *   sums    : K x d fp64, global per-cluster coordinate sums
 * Enables one following kmeans_update. */
kmeans_status kmeans_assign(kmeans_ctx* ctx, const double* centroids, int32_t* labels,
                            double* inertia, int64_t* counts, double* sums);

/* The mean step after kmeans_assign: writes
 * mu^{t+1} (K x d fp64) to `centroids` (empty clusters keep the mu^t given to
 * kmeans_assign) and E to *shift_E (either may be NULL).
 * KMEANS_ESTATE unless directly preceded by a successful kmeans_assign. */
kmeans_status kmeans_update(kmeans_ctx* ctx, double* centroids, double* shift_E);

/* The whole serial Lloyd run of PAPER.md:65-70 on one GPU:
 *   mu^0 = x[init_idx[k]] (K distinct indices in [0, N)),
 *   loop { assign; update } until E < tol or max_iter iterations.
 * points: N x d row-major fp32.  Outputs: labels z^{iters} (N, may be NULL),
 * centroids mu^{iters} (K x d), iters in [1, max_iter], inertia = J of the
 * last iteration.  Non-convergence at max_iter is KMEANS_OK. */
kmeans_status kmeans_fit(const float* points, int64_t N, int d, int K, const int64_t* init_idx,
                         double tol, int max_iter, int32_t* labels, double* centroids,
                         int* iters, double* inertia);

/* kmeans_fit on an existing context; collective when distributed (init_idx
 * are global indices; labels are this rank's N).  E_trace / J_trace (may be
 * NULL) receive E and J of every iteration (max_iter entries of room). */
kmeans_status kmeans_fit_ctx(kmeans_ctx* ctx, const int64_t* init_idx, double tol,
                             int max_iter, int32_t* labels, double* centroids, int* iters,
                             double* inertia, double* E_trace, double* J_trace);

/* ---- device-resident loop (asynchronous; used by kmeans_fit_ctx and bench) ---- */

/* Resets the iteration state: mu^0 from init_idx (K global indices) or, if
 * init_idx is NULL, from `centroids` (K x d fp64); t = 0; stop rule
 * (tol, max_iter).  Synchronous. */
kmeans_status kmeans_start(kmeans_ctx* ctx, const int64_t* init_idx, const double* centroids,
                           double tol, int max_iter);

/* Enqueues n Lloyd iterations on the context's stream (a captured CUDA graph
 * per iteration: assign+reduce, merge, [allreduce], update).  Iterations
 * after the stop rule fired are no-ops.  Returns without synchronising. */
kmeans_status kmeans_iterate(kmeans_ctx* ctx, int n);

/* Synchronises the stream and reads the state: completed iterations, stop
 * flag, last E and J (any may be NULL). */
kmeans_status kmeans_poll(kmeans_ctx* ctx, int* iters, int* done, double* E, double* J);

/* Copies the current centroids mu^t (K x d fp64).  Synchronous. */
kmeans_status kmeans_read_centroids(kmeans_ctx* ctx, double* centroids);

/* Writes z^{t} = argmin_k ||x_i - fl32(mu_k^{t-1})|| for this rank's points,
 * i.e. the labels of the last completed iteration (t >= 1).  Synchronous. */
kmeans_status kmeans_final_labels(kmeans_ctx* ctx, int32_t* labels);

/* Profiling aid (bench.py's roofline): enqueues n passes of the assignment
 * step with its fused per-chunk reduction at the current mu^t -- the assign
 * kernels plus the chunk-row merge, no group merge / update; the iteration
 * state is unchanged.  Returns without synchronising.  Same as
 * kmeans_profile_stage(ctx, n, 0). */
kmeans_status kmeans_profile_assign(kmeans_ctx* ctx, int n);

/* Profiling aid: n launches of one stage of the iteration, state unchanged:
 *   stage 0  assign kernels + chunk-row merge (= kmeans_profile_assign)
 *   stage 1  the assign kernels alone ([prune], assign+reduce, [heavy]) --
 *            the dominant kernel bench.py reports the roofline of
 *   stage 2  the chunk-row merge alone (k_merge_sparse16 / k_merge_rows /
 *            k_merge_sparse; nothing on the unsorted large-K path)
 *   stage 3  the group merge (k_merge) alone
 * ms_per_launch NULL: enqueues the launches and returns without synchronising.
 * ms_per_launch non-NULL: captures the n launches in a CUDA graph, runs it
 * once untimed and once between two CUDA events on the context's stream, and
 * writes the device time per launch (synchronous; excludes host launch cost).
 * KMEANS_EINVAL if n < 0 or stage is not 0..3. */
kmeans_status kmeans_profile_stage(kmeans_ctx* ctx, int n, int stage, float* ms_per_launch);

/* Sorted path: centroid candidates per chunk (1024 or 2048 points) in the last assign
 * pass -- mean, maximum, number of single-candidate chunks, number of chunks
 * (any may be NULL).  KMEANS_ESTATE on an unsorted context.  Synchronous. */
kmeans_status kmeans_candidate_stats(kmeans_ctx* ctx, double* mean, int* max, int64_t* single,
                                     int64_t* chunks);

/* The cudaStream_t the context runs on. */
kmeans_status kmeans_get_stream(kmeans_ctx* ctx, void** stream);

typedef struct kmeans_info {
    int64_t N, global_N, global_offset, ldx;
    int d, K;
    int grid;               /* blocks of the assign kernel: 1024/2048-point chunks (sorted),
                               2048-point chunks (full scan, K <= 16) or a persistent
                               multiple of the SM count (full scan, K > 16) */
    int block;              /* threads per block of the assign kernel */
    int smem_bytes;         /* dynamic shared memory of the assign kernel */
    int path;               /* 0 = chunked register-centroid path (K <= 16), 1 = shared-memory path */
    int kernels_per_iter;   /* kernels of this library launched per iteration */
    int64_t kernel_launches;/* kernels of this library launched so far by this context */
    int nranks, rank;
    int sorted;             /* 1 = curve-sorted shard with per-chunk pruning */
    int fused;              /* 1 = kmeans_iterate runs k_fused_iterate (grid = fused_grid) */
    int fused_grid;         /* its cooperative grid (blocks of 256 threads) */
    int persistent;         /* 1 = kmeans_iterate runs k_persist_iterate (KMEANS_FLAG_PERSIST) */
    int persist_grid;       /* its cooperative grid (one block per SM) */
} kmeans_info;

kmeans_status kmeans_get_info(kmeans_ctx* ctx, kmeans_info* info);

/* ---- multi-GPU plumbing (NCCL) ---- */

/* Writes a fresh NCCL unique id (128 bytes) to id; rank 0 calls it and the
 * caller broadcasts it (e.g. over torch.distributed). */
kmeans_status kmeans_comm_unique_id(unsigned char id[128]);

/* Creates an NCCL communicator for `rank` of `nranks` on CUDA device `device`
 * (collective over the ranks). *comm receives an ncclComm_t. */
kmeans_status kmeans_comm_init(void** comm, int nranks, const unsigned char id[128], int rank,
                               int device);

kmeans_status kmeans_comm_destroy(void* comm);

/* On-device synthetic input: the seeded Gaussian mixture
 * of DESIGN.md "Inputs", generated directly in HBM by the same
 * counter-based recipe as the host generator (datagen.py), so a rank can make
 * its shard [start, start + count) of an N-point dataset without host memory
 * or PCIe.  Box-Muller runs in fp64 with the device libm, whose log1p / cos /
 * sin may differ from the host's by an ulp: a value can move by one fp32 ulp
 * (rarely; bounded in the tests). */
typedef struct kmeans_mixture {
    uint64_t seed;          /* data seed (datagen Workload.data_seed) */
    int d;                  /* 2 or 3 */
    int M;                  /* blobs, >= 1 */
    const double* centers;  /* M x d, host */
    double sigma;           /* blob standard deviation */
    int n_sites;            /* planted outlier sites G (0 = none) */
    int site_dups;          /* duplicates per site r: points g (N / G) + q, q < r */
    const double* sites;    /* G x d, host (NULL if G = 0) */
    int64_t N;              /* points in the whole dataset */
} kmeans_mixture;

/* Writes points [start, start + count) as AoS fp32 (count x d) to `out`
 * (device memory) on `stream` (cudaStream_t, NULL = default stream) of CUDA
 * device `device`; synchronous.  KMEANS_EINVAL for a bad spec or range. */
kmeans_status kmeans_generate(const kmeans_mixture* mix, int64_t start, int64_t count, float* out,
                              int device, void* stream);

/* P2P exchange (multi-GPU).  On a context with an NCCL
 * communicator, the per-iteration allreduce of the K(d+1)+1 partials
 * ("local cluster means ... transferred to a global variable")
 * can run as one kernel over peer memory instead of ncclAllReduce: each rank
 * owns an exchange buffer in its HBM, every rank maps every peer's buffer
 * (CUDA IPC, NVLink), pushes its vector into all of them, publishes an epoch
 * flag, waits for all peers' flags and sums the P vectors in rank order (the
 * same bits on every rank), fused with the update (k_p2p_update).
 *   1. kmeans_p2p_handle: allocates this rank's buffer (once) and writes its
 *      64-byte cudaIpcMemHandle_t; the caller all-gathers the handles.
 *   2. kmeans_p2p_open: `handles` = nranks x 64 bytes in rank order; maps the
 *      peers' buffers; from then on the iteration, kmeans_start's mu^0
 *      assembly and kmeans_assign use the exchange.  Collective: every rank
 *      must open before any rank iterates.
 * The group is the NCCL communicator's, or opts.rank / opts.nranks of a
 * P2P-only context.  KMEANS_EINVAL on a single-GPU context or a second open;
 * KMEANS_ECUDA if IPC mapping fails (e.g. no peer access) -- NOT sticky: the
 * mappings made so far are closed and the context stays usable (a
 * communicator context can go on with the NCCL allreduce after
 * kmeans_p2p_disable; every rank must then disable). */
kmeans_status kmeans_p2p_handle(kmeans_ctx* ctx, unsigned char handle[64]);
kmeans_status kmeans_p2p_open(kmeans_ctx* ctx, const unsigned char* handles);
/* Diagnostic of an opened P2P group, run by ONE rank while the others are idle:
 * all nranks ranks of the exchange protocol emulated by the blocks of one
 * cooperative launch on this rank's GPU, over the REAL buffers -- this rank's
 * own and its peers' (mapped by CUDA IPC, possibly in other processes) --
 * with epochs no real exchange uses.  Round i: emulated rank r contributes
 * vals[i][r][0..n) (host, rounds x nranks x n doubles); out[i][r][0..n) (host)
 * receives what it computed, the rank-ordered sum over q of vals[i][q].
 * Checks that every mapping works both ways (remote stores and loads, system-
 * scope flags) without ranks waiting on one another across processes.
 * Synchronous.  KMEANS_EINVAL without an opened group, for rounds < 1, n < 1
 * or n > K (d + 1) + 1; KMEANS_ENCCL if an emulated rank timed out. */
kmeans_status kmeans_p2p_loopback(kmeans_ctx* ctx, int rounds, int n, const double* vals,
                                  double* out);

/* Back to the NCCL allreduce (e.g. when some rank could not map its peers;
 * every rank must then disable).  Synchronises the context's stream. */
kmeans_status kmeans_p2p_disable(kmeans_ctx* ctx);

/* Self-test of the exchange protocol on ONE GPU: P emulated ranks as P blocks
 * of one cooperative launch (ranks that wait on one another must not be
 * separate launches on one GPU), each with its own exchange buffer; in round
 * i rank r contributes vals[i][r][0..n) (host, rounds x P x n doubles) and
 * out[i][r][0..n) (host) receives what rank r computed -- the rank-ordered sum
 * over q of vals[i][q].  dead_rank in [0, P) never publishes (-1: none): the
 * other ranks must give up after timeout_s seconds (0 = 60 s); failed (host,
 * P ints, may be NULL) receives per rank the 1-based round whose exchange
 * failed, 0 if none (the dead rank itself: 0).  Synchronous.  Returns
 * KMEANS_ENCCL if any exchange failed; KMEANS_EINVAL for P not in [1, 64],
 * n < 1, rounds < 1, dead_rank >= P, timeout_s < 0 or NULL vals / out. */
kmeans_status kmeans_p2p_selftest(int device, int P, int n, int rounds, const double* vals,
                                  double* out, int dead_rank, double timeout_s, int* failed);

/* NULL-safe; frees all device memory of the context (not the caller's stream
 * or communicator).  Freed blocks go to a library-owned cache per device that
 * the next kmeans_create reuses (no cudaMalloc / cudaFree of the point arrays
 * on every create / destroy); a failing cudaMalloc empties the cache first. */
void kmeans_destroy(kmeans_ctx* ctx);

/* Returns the blocks the library cache of CUDA device `device` holds (memory
 * of destroyed contexts) to the driver.  KMEANS_EINVAL for a bad device. */
kmeans_status kmeans_release_memory(int device);

const char* kmeans_status_string(kmeans_status s);
const char* kmeans_last_error(void);
int kmeans_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* KMEANS_H */
