// lk_icp.cu -- ICP point-to-plane refinement on sm_100a (north-star item 4,
// config D). The reference has no ICP; the specification is the
// builder's, frozen in oracle/lk_oracle.cpp "ICP point-to-plane" and
// DESIGN.md "ICP", and this file reproduces it bit for bit:
//
//   k_icp_accum   thread per source point, CTA per 256-point chunk: y = T p,
//                 the exact EvalGrid NN through the ring grid (lk_ring.cuh:
//                 FP32 shell scan, FP64 decisions, the reference's +-1 window
//                 and (d2, index) order), r and J = (y x n, n); the 28
//                 products reduced by 32-lane butterflies and an in-order sum
//                 of the CTA's 8 warps.
//   k_icp_solve   one CTA: 32-chunk butterflies summed in order, the LDL^T
//                 solve of H delta = -g and the Cayley update of T, the
//                 convergence test; writes T and its FP32 image for the next
//                 iteration. All iterations are enqueued back to back; a
//                 finished run turns the remaining launches into no-ops.
#include <cmath>
#include <cstdint>

#include "lk_device_math.cuh"
#include "lk_kernels.cuh"
#include "lk_ring.cuh"

namespace lkk {

using namespace lkd;

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kIcpVals = 28;  // 21 H (upper, row-major) + 6 g + e
constexpr int kIcpThreads = 256;

struct IcpState {
    double R[9], t[3];
    int32_t done;         // 1 once converged or singular
    int32_t iterations;   // updates applied
    int32_t converged;
    int32_t status;       // 0, or 6 (fewer than 6 correspondences in the first iteration)
    int64_t count;        // correspondences of the last accumulation
    double rmse;
};

__device__ __forceinline__ double butterfly(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

// The nearest neighbours of one iteration, queries in the source's Morton
// order (perm) so that a warp's walks share cells; nn[i] = -1 for no match.
// nn holds the previous iteration's matches on entry (seeds of the walks).
__global__ void __launch_bounds__(kIcpThreads) k_icp_nn(const double4* __restrict__ pos4,
                                                        const int32_t* __restrict__ perm, int64_t n,
                                                        const __grid_constant__ RingGrid rg, double d2_max,
                                                        const IcpState* __restrict__ st, int32_t* __restrict__ nn) {
    if (st->done) return;
    __shared__ double s_R[12];
    __shared__ float4 s_buf[kIcpThreads / 32][32];
    if (threadIdx.x < 12) s_R[threadIdx.x] = threadIdx.x < 9 ? st->R[threadIdx.x] : st->t[threadIdx.x - 9];
    __syncthreads();
    const int64_t t = blockIdx.x * static_cast<int64_t>(kIcpThreads) + threadIdx.x;
    const bool act = t < n;
    const int32_t i = act ? __ldg(perm + t) : 0;
    const V3 y = act ? xform(s_R, s_R + 9, ld4(pos4, i)) : mk(0.0, 0.0, 0.0);
    // seeded with the previous iteration's match (nn starts at -1)
    const int32_t prev = act ? __ldg(nn + i) : -1;
    const int32_t j = ring_nn_warp(rg, y, d2_max, act, s_buf[threadIdx.x >> 5], prev);  // warp-uniform call
    if (act) nn[i] = j;
}

__global__ void __launch_bounds__(kIcpThreads) k_icp_accum(const double4* __restrict__ pos4, int64_t n,
                                                           const __grid_constant__ RingGrid rg,
                                                           const double* __restrict__ tnrm,
                                                           const int32_t* __restrict__ nn,
                                                           const IcpState* __restrict__ st,
                                                           double* __restrict__ partial,
                                                           unsigned long long* __restrict__ count) {
    if (st->done) return;
    __shared__ double s_R[12];
    __shared__ double s_w[kIcpThreads / 32][kIcpVals];
    if (threadIdx.x < 12) s_R[threadIdx.x] = threadIdx.x < 9 ? st->R[threadIdx.x] : st->t[threadIdx.x - 9];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n_chunks = (n + kIcpThreads - 1) / kIcpThreads;
    unsigned long long cnt = 0;
    for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        const int64_t i = c * kIcpThreads + threadIdx.x;
        double J[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        double r = 0.0;
        if (i < n) {
            const int32_t j = __ldg(nn + i);
            if (j >= 0) {
                const V3 y = xform(s_R, s_R + 9, ld4(pos4, i));
                const V3 nt = ld3(tnrm, j);
                if (!is_zero(nt)) {
                    const V3 q = ld4(rg.pos4, j);
                    r = dot(sub(y, q), nt);
                    J[0] = y.y * nt.z - y.z * nt.y;
                    J[1] = y.z * nt.x - y.x * nt.z;
                    J[2] = y.x * nt.y - y.y * nt.x;
                    J[3] = nt.x;
                    J[4] = nt.y;
                    J[5] = nt.z;
                    cnt += 1;
                }
            }
        }
        int k = 0;
#pragma unroll
        for (int u = 0; u < 6; ++u)
#pragma unroll
            for (int w = u; w < 6; ++w) {
                const double v = butterfly(J[u] * J[w]);
                if (lane == 0) s_w[warp][k] = v;
                ++k;
            }
#pragma unroll
        for (int u = 0; u < 6; ++u) {
            const double v = butterfly(J[u] * r);
            if (lane == 0) s_w[warp][21 + u] = v;
        }
        {
            const double v = butterfly(r * r);
            if (lane == 0) s_w[warp][27] = v;
        }
        __syncthreads();
        if (threadIdx.x < kIcpVals) {
            double acc = s_w[0][threadIdx.x];
#pragma unroll
            for (int w = 1; w < kIcpThreads / 32; ++w) acc = acc + s_w[w][threadIdx.x];
            partial[c * kIcpVals + threadIdx.x] = acc;
        }
        __syncthreads();
    }
    cnt = __reduce_add_sync(kFull, static_cast<unsigned>(cnt));
    if (lane == 0 && cnt) atomicAdd(count, cnt);
}

// LDL^T solve of H x = -g, operation for operation oracle/lk_oracle.cpp icp_solve.
__device__ bool icp_solve(const double* h21, const double* g6, double* x6) {
    double H[6][6];
    int k = 0;
    for (int u = 0; u < 6; ++u)
        for (int w = u; w < 6; ++w) {
            H[u][w] = h21[k];
            H[w][u] = h21[k];
            ++k;
        }
    double L[6][6], D[6];
    for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) L[i][j] = 0.0;
    for (int j = 0; j < 6; ++j) {
        double dj = H[j][j];
        for (int q = 0; q < j; ++q) dj = dj - (L[j][q] * L[j][q]) * D[q];
        if (!(dj > 0.0)) return false;
        D[j] = dj;
        for (int i = j + 1; i < 6; ++i) {
            double v = H[i][j];
            for (int q = 0; q < j; ++q) v = v - (L[i][q] * L[j][q]) * D[q];
            L[i][j] = v / dj;
        }
    }
    double z[6];
    for (int i = 0; i < 6; ++i) {
        double v = -g6[i];
        for (int q = 0; q < i; ++q) v = v - L[i][q] * z[q];
        z[i] = v;
    }
    for (int i = 5; i >= 0; --i) {
        double v = z[i] / D[i];
        for (int q = i + 1; q < 6; ++q) v = v - L[q][i] * x6[q];
        x6[i] = v;
    }
    return true;
}

// Matrix3d * Matrix3d in Eigen's order (rows 0-1 packet, row 2 scalar), row-major
__device__ void mat_mul(const double* a, const double* b, double* out) {
    for (int j = 0; j < 3; ++j) {
        for (int i = 0; i < 2; ++i)
            out[3 * i + j] = (a[3 * i] * b[j] + a[3 * i + 1] * b[3 + j]) + a[3 * i + 2] * b[6 + j];
        out[6 + j] = a[6] * b[j] + (a[7] * b[3 + j] + a[8] * b[6 + j]);
    }
}

__global__ void __launch_bounds__(kIcpVals * 32) k_icp_solve(const double* __restrict__ partial, int64_t n_chunks,
                                                             const unsigned long long* __restrict__ count,
                                                             IcpState* __restrict__ st,
                                                             double* __restrict__ history, int32_t iteration,
                                                             double eps2) {
    if (st->done) return;
    __shared__ double s_tot[kIcpVals];
    const int lane = threadIdx.x & 31, v = threadIdx.x >> 5;
    // 32-chunk butterflies summed in order; eight groups' loads and
    // butterflies in flight at once (the in-order sum is unchanged)
    double acc = 0.0;
    constexpr int kU = 8;
    for (int64_t s0 = 0; s0 < n_chunks; s0 += 32 * kU) {
        double x[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t c = s0 + 32 * u + lane;
            x[u] = c < n_chunks ? partial[c * kIcpVals + v] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) x[u] = butterfly(x[u]);
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (s0 + 32 * u < n_chunks) acc = acc + x[u];
    }
    if (lane == 0) s_tot[v] = acc;
    __syncthreads();
    if (threadIdx.x != 0) return;
    const int64_t cnt = static_cast<int64_t>(*count);
    st->count = cnt;
    st->rmse = cnt > 0 ? sqrt(s_tot[27] / static_cast<double>(cnt)) : 0.0;
    double x[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    const bool ok = cnt >= 6 && icp_solve(s_tot, s_tot + 21, x);
    double dd = 0.0;
    if (ok)
        for (int k = 0; k < 6; ++k) dd = dd + x[k] * x[k];
    if (history) {
        history[3 * iteration] = static_cast<double>(cnt);
        history[3 * iteration + 1] = st->rmse;
        history[3 * iteration + 2] = dd;
    }
    if (!ok) {
        if (iteration == 0 && cnt < 6) st->status = 6;
        st->done = 1;
        return;
    }
    // Cayley update, operation for operation oracle/lk_oracle.cpp icp_update
    const double wx = x[0] * 0.5, wy = x[1] * 0.5, wz = x[2] * 0.5;
    const double s = 2.0 / (1.0 + ((wx * wx + wy * wy) + wz * wz));
    const double K[9] = {0.0, -wz, wy, wz, 0.0, -wx, -wy, wx, 0.0};
    double K2[9], Rd[9], Rn[9];
    mat_mul(K, K, K2);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) Rd[3 * i + j] = (i == j ? 1.0 : 0.0) + s * (K[3 * i + j] + K2[3 * i + j]);
    mat_mul(Rd, st->R, Rn);
    const V3 tn = rot(Rd, mk(st->t[0], st->t[1], st->t[2]));
    for (int k = 0; k < 9; ++k) st->R[k] = Rn[k];
    st->t[0] = tn.x + x[3];
    st->t[1] = tn.y + x[4];
    st->t[2] = tn.z + x[5];
    st->iterations = iteration + 1;
    if (dd < eps2) {
        st->converged = 1;
        st->done = 1;
    }
}

}  // namespace

cudaError_t icp_point_to_plane(const double* d_src, int64_t n, const RingStorage& ring, const double* d_tnrm,
                               double max_dist, int32_t max_iter, double eps, const double* R0, const double* t0,
                               double* R9, double* t3, IcpOutcome* out, double* d_history, cudaStream_t stream,
                               int sm_count) {
    double4* pos4 = nullptr;
    int32_t *perm = nullptr, *nn = nullptr;
    double* partial = nullptr;
    unsigned long long* counts = nullptr;
    IcpState* st = nullptr;
    const int64_t n_chunks = (n + kIcpThreads - 1) / kIcpThreads;
    cudaError_t e;
    auto cleanup = [&] {
        pool_free(pos4, stream);
        pool_free(perm, stream);
        pool_free(nn, stream);
        pool_free(partial, stream);
        pool_free(counts, stream);
        pool_free(st, stream);
    };
#define ICP_TRY(x)              \
    do {                        \
        e = (x);                \
        if (e != cudaSuccess) { \
            cleanup();          \
            return e;           \
        }                       \
    } while (0)
    const int32_t iters = max_iter > 0 ? max_iter : 0;
    ICP_TRY(pool_alloc(&pos4, n * sizeof(double4), stream));
    ICP_TRY(pool_alloc(&partial, n_chunks * kIcpVals * sizeof(double), stream));
    ICP_TRY(pool_alloc(&counts, (iters + 1) * sizeof(unsigned long long), stream));
    ICP_TRY(pool_alloc(&st, sizeof(IcpState), stream));
    ICP_TRY(pool_alloc(&perm, n * sizeof(int32_t), stream));
    ICP_TRY(pool_alloc(&nn, n * sizeof(int32_t), stream));
    ICP_TRY(cudaMemsetAsync(nn, 0xff, n * sizeof(int32_t), stream));  // no seeds in the first iteration
    ICP_TRY(make_records(d_src, nullptr, n, pos4, nullptr, stream));
    ICP_TRY(spatial_order(d_src, n, perm, stream));
    ICP_TRY(cudaMemsetAsync(counts, 0, (iters + 1) * sizeof(unsigned long long), stream));
    IcpState h{};
    for (int k = 0; k < 9; ++k) h.R[k] = R0[k];
    for (int k = 0; k < 3; ++k) h.t[k] = t0[k];
    ICP_TRY(cudaMemcpyAsync(st, &h, sizeof(h), cudaMemcpyHostToDevice, stream));
    const int blocks = static_cast<int>(n_chunks < sm_count * 8 ? n_chunks : sm_count * 8);
    const double d2_max = max_dist * max_dist;
    for (int32_t it = 0; it < iters; ++it) {
        k_icp_nn<<<static_cast<unsigned>(n_chunks), kIcpThreads, 0, stream>>>(pos4, perm, n, ring.view, d2_max, st, nn);
        k_icp_accum<<<blocks, kIcpThreads, 0, stream>>>(pos4, n, ring.view, d_tnrm, nn, st, partial, counts + it);
        k_icp_solve<<<1, kIcpVals * 32, 0, stream>>>(partial, n_chunks, counts + it, st, d_history, it, eps * eps);
    }
    ICP_TRY(cudaGetLastError());
    ICP_TRY(cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, stream));
    ICP_TRY(cudaStreamSynchronize(stream));
#undef ICP_TRY
    cleanup();
    for (int k = 0; k < 9; ++k) R9[k] = h.R[k];
    for (int k = 0; k < 3; ++k) t3[k] = h.t[k];
    out->iterations = h.iterations;
    out->converged = h.converged;
    out->status = h.status;
    out->correspondences = h.count;
    out->rmse = h.rmse;
    out->fitness = n > 0 ? static_cast<double>(h.count) / static_cast<double>(n) : 0.0;
    return cudaSuccess;
}

}  // namespace lkk
