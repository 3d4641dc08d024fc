// kernels.cuh -- sm_100a kernels of one Lloyd iteration (arXiv 2405.12052).
//
// Step map:
//   k_prep          AoS/SoA fp32 input -> padded SoA fp32, non-finite check (create only)
//   k_init_gather   mu^0_k = (double) x[init_idx[k]]
//   k_assign_small  K <= 16: centroids in registers, form-D distances with packed
//                   f32x2 FADD2/FMUL2/FFMA2, exact argmin (lowest index on ties),
//                   per-thread private fp64 smem accumulators, per-block partials
//                                                                        PAPER.md:45-52
//   k_assign_large  16 < K <= 1024: centroids in smem, per-warp fp64 accumulators
//                   updated in lane order (conflicting lanes serialised by
//                   __match_any_sync rounds), per-block partials
//   k_merge         per-GPU sum of the per-block partials in a fixed order
//                   (the OpenMP "global variable" merge of PAPER.md:97, without
//                   the critical section)
//   k_update        mu^{t+1} = S/n (empty cluster keeps mu^t), E, J, stop flag
//                                                                        PAPER.md:50-70
// No global float atomics anywhere; every reduction has a fixed order, so results
// are bit-reproducible run to run for a fixed grid.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace km {

// Device-resident loop state (E compared with tol "at the end of each
// iteration").  t = completed iterations; mu^t lives in mu_buf[t & 1].
struct DevState {
    int t;
    int done;
    int max_iter;
    int pad0;
    double tol;
    double E;
    double J;
};

constexpr int kSmallTPB = 256;     // threads per block, small-K path
constexpr int kLargeTPBMax = 256;  // threads per block (max), large-K path
constexpr int kPadPoints = 1024;   // SoA arrays padded so any tile start < N is in bounds

__device__ __forceinline__ float pos_inf() { return __int_as_float(0x7f800000); }

// Read of 2 consecutive fp32 coordinates (8-byte aligned), read-only path.
__device__ __forceinline__ float2 ld_stream2(const float* p) {
    return __ldg(reinterpret_cast<const float2*>(p));
}

// ---------------------------------------------------------------------------
// k_prep: out[j * ldx + i] = in[i * si + j * sj] for i < N, 0 for N <= i < ldx.
// Any non-finite coordinate sets *flag (integer atomic, order-free).
// ---------------------------------------------------------------------------
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
            out[(int64_t)j * ldx + i] = v;
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// mu^0_k = (double) x_{idx_k} for the indices this rank owns, 0 elsewhere (the
// allreduce over ranks then assembles mu^0 exactly: one x plus zeros).
__global__ void k_init_gather(const float* __restrict__ X, int64_t ldx, int d, int K,
                              const int64_t* __restrict__ idx, int64_t offset, int64_t n_local,
                              double* __restrict__ mu0) {
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= K * d) return;
    int k = q / d, j = q % d;
    int64_t i = idx[k] - offset;
    mu0[q] = (i >= 0 && i < n_local) ? (double)X[(int64_t)j * ldx + i] : 0.0;
}

// Per-block partial layout: part[e * G + b], e in [0, K*D + K + 1):
//   e <  K*D          : S_k,j  (k-major)
//   K*D <= e < K*D+K  : n_k    (exact integer in fp64)
//   e == K*D + K      : J
// Merged / allreduced vector red[e] has the same e order.

enum : int { kModeReduce = 1, kModeLabels = 2 };

// ---------------------------------------------------------------------------
// Small-K path.  KP = compile-time padded K (4, 8 or 16); padded slots have
// c = +inf so their distance is +inf and never wins (strict <).
// Each thread handles 2 consecutive points per tile (float2 loads, packed math).
// ---------------------------------------------------------------------------
template <int D, int KP, int MODE>
__global__ void __launch_bounds__(kSmallTPB, 2)
k_assign_small(const float* __restrict__ X, int64_t ldx, int64_t n, int K,
               const double* __restrict__ mu_buf, const DevState* __restrict__ st,
               int mu_sel, int ignore_done, double* __restrict__ part,
               int32_t* __restrict__ labels) {
    if (!ignore_done && st->done) return;
    const int t_it = st->t;
    const double* mu = mu_buf + (size_t)((t_it - mu_sel) & 1) * K * D;

    // Stage: c_k = fl32(mu_k^t) (RN), kept negated so that x + (-c) == x - c.
    float nc[KP][D];
#pragma unroll
    for (int k = 0; k < KP; ++k) {
#pragma unroll
        for (int j = 0; j < D; ++j)
            nc[k][j] = (k < K) ? -__double2float_rn(__ldg(&mu[k * D + j])) : -pos_inf();
    }

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x;
    double2* accA = reinterpret_cast<double2*>(smem_raw);                 // [KP][TPB] (sx, sy)
    double* accZ = reinterpret_cast<double*>(accA + KP * kSmallTPB);       // [KP][TPB] sz (D==3)
    int* accN = reinterpret_cast<int*>(accZ + (D == 3 ? KP * kSmallTPB : 0));  // [KP][TPB]
    double* warpJ = reinterpret_cast<double*>(accN + KP * kSmallTPB);      // [TPB/32]

    if (MODE & kModeReduce) {
#pragma unroll
        for (int k = 0; k < KP; ++k) {
            accA[k * kSmallTPB + tid] = make_double2(0.0, 0.0);
            if (D == 3) accZ[k * kSmallTPB + tid] = 0.0;
            accN[k * kSmallTPB + tid] = 0;
        }
    }
    double J = 0.0;

    const float* X0 = X;
    const float* X1 = X + ldx;
    const float* X2 = X + 2 * ldx;
    constexpr int kTile = 2 * kSmallTPB;
    const int64_t n_tiles = (n + kTile - 1) / kTile;

    int64_t tile = blockIdx.x;
    float2 px, py, pz = make_float2(0.f, 0.f);
    if (tile < n_tiles) {
        int64_t p = tile * kTile + 2 * tid;
        px = ld_stream2(X0 + p);
        py = ld_stream2(X1 + p);
        if (D == 3) pz = ld_stream2(X2 + p);
    }
    for (; tile < n_tiles; tile += gridDim.x) {
        const int64_t p = tile * kTile + 2 * tid;
        const float2 x = px, y = py, z = pz;
        // prefetch the next tile of this block (1-deep register pipeline)
        const int64_t nt = tile + gridDim.x;
        if (nt < n_tiles) {
            int64_t q = nt * kTile + 2 * tid;
            px = ld_stream2(X0 + q);
            py = ld_stream2(X1 + q);
            if (D == 3) pz = ld_stream2(X2 + q);
        }

        // Reassignment, form D, both points at once.
        float b0, b1;
        int l0 = 0, l1 = 0;
        {
            float2 e0 = __fadd2_rn(x, make_float2(nc[0][0], nc[0][0]));
            float2 e1 = __fadd2_rn(y, make_float2(nc[0][1], nc[0][1]));
            float2 s = __fmul2_rn(e0, e0);
            s = __ffma2_rn(e1, e1, s);
            if (D == 3) {
                float2 e2 = __fadd2_rn(z, make_float2(nc[0][2], nc[0][2]));
                s = __ffma2_rn(e2, e2, s);
            }
            b0 = s.x;
            b1 = s.y;
        }
#pragma unroll
        for (int k = 1; k < KP; ++k) {
            float2 e0 = __fadd2_rn(x, make_float2(nc[k][0], nc[k][0]));
            float2 e1 = __fadd2_rn(y, make_float2(nc[k][1], nc[k][1]));
            float2 s = __fmul2_rn(e0, e0);
            s = __ffma2_rn(e1, e1, s);
            if (D == 3) {
                float2 e2 = __fadd2_rn(z, make_float2(nc[k][2], nc[k][2]));
                s = __ffma2_rn(e2, e2, s);
            }
            if (s.x < b0) { b0 = s.x; l0 = k; }
            if (s.y < b1) { b1 = s.y; l1 = k; }
        }

        const bool v0 = p < n, v1 = p + 1 < n;
        if (MODE & kModeLabels) {
            // labels buffer is padded like X: the pair store is always in bounds
            *reinterpret_cast<int2*>(labels + p) = make_int2(l0, l1);
        }
        if (MODE & kModeReduce) {
            // Fused mean numerator/denominator, private column.
            if (v0) {
                int a = l0 * kSmallTPB + tid;
                double2 sxy = accA[a];
                sxy.x += (double)x.x;
                sxy.y += (double)y.x;
                accA[a] = sxy;
                if (D == 3) accZ[a] += (double)z.x;
                accN[a] += 1;
                J += (double)b0;
            }
            if (v1) {
                int a = l1 * kSmallTPB + tid;
                double2 sxy = accA[a];
                sxy.x += (double)x.y;
                sxy.y += (double)y.y;
                accA[a] = sxy;
                if (D == 3) accZ[a] += (double)z.y;
                accN[a] += 1;
                J += (double)b1;
            }
        }
    }

    if (!(MODE & kModeReduce)) return;

    // Block reduction in a fixed order: lane l sums threads l, l+32, ... in
    // ascending order, then a butterfly over the 32 lanes.
    const int lane = tid & 31, warp = tid >> 5;
    constexpr int W = kSmallTPB / 32;
    {
        double j = J;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) j += __shfl_xor_sync(0xffffffffu, j, o);
        if (lane == 0) warpJ[warp] = j;
    }
    __syncthreads();
    const int G = gridDim.x;
    const int nE = K * D + K + 1;
    for (int e = warp; e < nE; e += W) {
        double v = 0.0;
        if (e < K * D) {
            const int k = e / D, j = e % D;
#pragma unroll
            for (int r = 0; r < kSmallTPB / 32; ++r) {
                const int a = k * kSmallTPB + r * 32 + lane;
                v += (j == 0) ? accA[a].x : (j == 1) ? accA[a].y : accZ[a];
            }
        } else if (e < K * D + K) {
            const int k = e - K * D;
            long long c = 0;
#pragma unroll
            for (int r = 0; r < kSmallTPB / 32; ++r) c += accN[k * kSmallTPB + r * 32 + lane];
            v = (double)c;
        } else {
            v = (lane < W) ? warpJ[lane] : 0.0;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) part[(size_t)e * G + blockIdx.x] = v;
    }
}

// ---------------------------------------------------------------------------
// Large-K path (16 < K <= 1024).  Centroids staged in smem as float4
// {-cx, -cy, -cz, 0}; each warp owns fp64 accumulators accS[w][k][D] and int
// counts accN[w][k]; the 32 lanes of a warp update them in ascending lane order
// (lanes with equal labels are serialised in rounds; distinct labels update in
// parallel), so the sums are deterministic.
// ---------------------------------------------------------------------------
template <int D, int MODE>
__global__ void __launch_bounds__(kLargeTPBMax)
k_assign_large(const float* __restrict__ X, int64_t ldx, int64_t n, int K,
               const double* __restrict__ mu_buf, const DevState* __restrict__ st,
               int mu_sel, int ignore_done, double* __restrict__ part,
               int32_t* __restrict__ labels) {
    if (!ignore_done && st->done) return;
    const int t_it = st->t;
    const double* mu = mu_buf + (size_t)((t_it - mu_sel) & 1) * K * D;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x;
    const int nthr = blockDim.x;
    const int W = nthr >> 5;
    const int lane = tid & 31, warp = tid >> 5;
    float4* cen = reinterpret_cast<float4*>(smem_raw);                  // [K]
    double* accS = reinterpret_cast<double*>(cen + K);                  // [W][K][D]
    int* accN = reinterpret_cast<int*>(accS + (size_t)W * K * D);        // [W][K]
    double* warpJ = reinterpret_cast<double*>(accN + W * K + ((W * K) & 1));  // [W]

    for (int k = tid; k < K; k += nthr) {
        float4 c;
        c.x = -__double2float_rn(mu[k * D + 0]);
        c.y = -__double2float_rn(mu[k * D + 1]);
        c.z = (D == 3) ? -__double2float_rn(mu[k * D + 2]) : 0.0f;
        c.w = 0.0f;
        cen[k] = c;
    }
    if (MODE & kModeReduce) {
        for (int q = tid; q < W * K * D; q += nthr) accS[q] = 0.0;
        for (int q = tid; q < W * K; q += nthr) accN[q] = 0;
    }
    __syncthreads();

    double* myS = accS + (size_t)warp * K * D;
    int* myN = accN + warp * K;
    double J = 0.0;

    const float* X0 = X;
    const float* X1 = X + ldx;
    const float* X2 = X + 2 * ldx;
    const int tileN = 2 * nthr;
    const int64_t n_tiles = (n + tileN - 1) / tileN;

    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int64_t p = tile * tileN + 2 * tid;
        const float2 x = ld_stream2(X0 + p);
        const float2 y = ld_stream2(X1 + p);
        const float2 z = (D == 3) ? ld_stream2(X2 + p) : make_float2(0.f, 0.f);

        float b0 = pos_inf(), b1 = pos_inf();
        int l0 = 0, l1 = 0;
        // k = 0 sets the initial best (a +inf distance must still yield label 0)
        {
            const float4 c = cen[0];
            float2 e0 = __fadd2_rn(x, make_float2(c.x, c.x));
            float2 e1 = __fadd2_rn(y, make_float2(c.y, c.y));
            float2 s = __fmul2_rn(e0, e0);
            s = __ffma2_rn(e1, e1, s);
            if (D == 3) {
                float2 e2 = __fadd2_rn(z, make_float2(c.z, c.z));
                s = __ffma2_rn(e2, e2, s);
            }
            b0 = s.x;
            b1 = s.y;
        }
#pragma unroll 4
        for (int k = 1; k < K; ++k) {
            const float4 c = cen[k];
            float2 e0 = __fadd2_rn(x, make_float2(c.x, c.x));
            float2 e1 = __fadd2_rn(y, make_float2(c.y, c.y));
            float2 s = __fmul2_rn(e0, e0);
            s = __ffma2_rn(e1, e1, s);
            if (D == 3) {
                float2 e2 = __fadd2_rn(z, make_float2(c.z, c.z));
                s = __ffma2_rn(e2, e2, s);
            }
            if (s.x < b0) { b0 = s.x; l0 = k; }
            if (s.y < b1) { b1 = s.y; l1 = k; }
        }

        const bool v0 = p < n, v1 = p + 1 < n;
        if (MODE & kModeLabels) *reinterpret_cast<int2*>(labels + p) = make_int2(l0, l1);
        if (MODE & kModeReduce) {
            if (v0) J += (double)b0;
            if (v1) J += (double)b1;
            // point 0 of every lane, then point 1 of every lane (fixed order)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const bool v = h ? v1 : v0;
                const int lab = h ? l1 : l0;
                const float cx = h ? x.y : x.x, cy = h ? y.y : y.x, cz = h ? z.y : z.x;
                unsigned pending = __ballot_sync(0xffffffffu, v);
                while (pending) {
                    // lanes still pending with my label
                    const unsigned peers = __match_any_sync(0xffffffffu, v ? lab : -1 - lane) & pending;
                    const bool mine = v && (pending >> lane & 1u) && ((peers & ((1u << lane) - 1u)) == 0u);
                    if (mine) {
                        double* s = myS + (size_t)lab * D;
                        s[0] += (double)cx;
                        s[1] += (double)cy;
                        if (D == 3) s[2] += (double)cz;
                        myN[lab] += 1;
                    }
                    __syncwarp();
                    pending &= ~__ballot_sync(0xffffffffu, mine);
                }
            }
        }
    }

    if (!(MODE & kModeReduce)) return;
    {
        double j = J;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) j += __shfl_xor_sync(0xffffffffu, j, o);
        if (lane == 0) warpJ[warp] = j;
    }
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
    for (int b = lane; b < G; b += 32) v += row[b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[e] = v;
}

// ---------------------------------------------------------------------------
// k_update (one block): the mean step of PAPER.md:50-62 and the error term of
// PAPER.md:66-69; then t += 1 and the stop decision of PAPER.md:70.
// ---------------------------------------------------------------------------
template <int D>
__global__ void k_update(double* __restrict__ mu_buf, int K, const double* __restrict__ red,
                         DevState* __restrict__ st, double* __restrict__ trace_E,
                         double* __restrict__ trace_J, int trace_cap) {
    if (st->done) return;
    __shared__ double red_sm[32];
    const int t = st->t;
    const double* mu_old = mu_buf + (size_t)(t & 1) * K * D;
    double* mu_new = mu_buf + (size_t)((t + 1) & 1) * K * D;
    const int tid = threadIdx.x;
    double e_acc = 0.0;
    for (int q = tid; q < K * D; q += blockDim.x) {
        const int k = q / D;
        const double nk = red[K * D + k];
        const double old = mu_old[q];
        const double nw = (nk > 0.0) ? red[q] / nk : old;   // empty cluster keeps mu^t
        mu_new[q] = nw;
        const double diff = nw - old;
        e_acc += diff * diff;
    }
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e_acc += __shfl_xor_sync(0xffffffffu, e_acc, o);
    if (lane == 0) red_sm[warp] = e_acc;
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        double v = (lane < nw) ? red_sm[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) {
            const double E = v;
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
}

}  // namespace km
