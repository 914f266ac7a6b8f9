// lk_icp.cu -- ICP point-to-plane refinement on sm_100a (north-star item 4,
// config D). The reference has no ICP; the specification is the
// builder's, frozen in oracle/lk_oracle.cpp "ICP point-to-plane" and
// DESIGN.md "ICP", and this file reproduces it bit for bit:
//
//   k_icp_accum   thread per source point, CTA per 256-point chunk: y = T p,
//                 the exact EvalGrid NN (FP32 fine-list scan, FP64 decisions,
//                 the reference's +-1 window and (d2, index) order), r and
//                 J = (y x n, n); the 28 products reduced by 32-lane
//                 butterflies and an in-order sum of the CTA's 8 warps.
//   k_icp_solve   one CTA: 32-chunk butterflies summed in order, the LDL^T
//                 solve of H delta = -g and the Cayley update of T, the
//                 convergence test; writes T and its FP32 image for the next
//                 iteration. All iterations are enqueued back to back; a
//                 finished run turns the remaining launches into no-ops.
#include <cmath>
#include <cstdint>

#include "lk_device_math.cuh"
#include "lk_kernels.cuh"
#include "lk_score_common.cuh"

namespace lkk {

using namespace lkd;

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kIcpVals = 28;  // 21 H (upper, row-major) + 6 g + e
constexpr int kIcpThreads = 256;

struct IcpState {
    double R[9], t[3];
    FastRT F;             // FP32 image of (R, t) in fine-cell units
    int32_t done;         // 1 once converged or singular
    int32_t iterations;   // updates applied
    int32_t converged;
    int32_t status;       // 0, or 6 (fewer than 6 correspondences in the first iteration)
    int64_t count;        // correspondences of the last accumulation
    double rmse;
};

// exact NN of y within d_max over the block list of y's EvalGrid cell
// (registration.cpp:165-199 semantics); returns the original index or -1
__device__ int32_t nn_coarse(const GridView& g, V3 y, double d2_max, double& best_d2) {
    const double fx = floor((y.x - g.ox) / g.cell) - static_cast<double>(g.offx);
    const double fy = floor((y.y - g.oy) / g.cell) - static_cast<double>(g.offy);
    const double fz = floor((y.z - g.oz) / g.cell) - static_cast<double>(g.offz);
    if (!(fx >= 0.0 && fy >= 0.0 && fz >= 0.0 && fx < g.nx && fy < g.ny && fz < g.nz)) return -1;
    const int64_t c = (static_cast<int64_t>(fx) * g.ny + static_cast<int64_t>(fy)) * g.nz + static_cast<int64_t>(fz);
    const int2 bi = __ldg(g.block_info + c);
    best_d2 = __longlong_as_double(0x7ff0000000000000ll);
    int32_t best = INT32_MAX;
    for (int32_t e = bi.x; e < bi.x + bi.y; ++e) {
        const double2* bp = reinterpret_cast<const double2*>(g.block_pts + e);
        const double2 qa = __ldg(bp), qb = __ldg(bp + 1);
        const double dx = qa.x - y.x, dy = qa.y - y.y, dz = qb.x - y.z;
        const double d2 = (dx * dx + dy * dy) + dz * dz;
        if (d2 > d2_max) continue;
        const int32_t orig = static_cast<int32_t>(qb.y);
        if (d2 < best_d2 || (d2 == best_d2 && orig < best)) {
            best_d2 = d2;
            best = orig;
        }
    }
    return best == INT32_MAX ? -1 : best;
}

// The same NN through the fine lists: FP32 location and top-3 scan, FP64
// decisions (as resolve_fine in lk_hypotheses.cu, without the normal gate).
__device__ int32_t nn_fine(const GridView& g, const FastRT& F, const double* R, const double* t, float4 P, V3 p,
                           double d2_max, V3& y) {
    y = xform(R, t, p);
    if (F.ok == 0.0f) {
        double d2;
        return nn_coarse(g, y, d2_max, d2);
    }
    const float qx = fmaf(F.r[0], P.x, fmaf(F.r[1], P.y, fmaf(F.r[2], P.z, F.t[0])));
    const float qy = fmaf(F.r[3], P.x, fmaf(F.r[4], P.y, fmaf(F.r[5], P.z, F.t[1])));
    const float qz = fmaf(F.r[6], P.x, fmaf(F.r[7], P.y, fmaf(F.r[8], P.z, F.t[2])));
    const float eps = F.eps;
    if (qx < -eps || qy < -eps || qz < -eps || qx >= g.fnx + eps || qy >= g.fny + eps || qz >= g.fnz + eps)
        return -1;  // certainly outside the grid box
    const float fx = floorf(qx), fy = floorf(qy), fz = floorf(qz);
    const float rx = qx - fx, ry = qy - fy, rz = qz - fz;
    if (rx < eps || rx > 1.0f - eps || ry < eps || ry > 1.0f - eps || rz < eps || rz > 1.0f - eps) {
        double d2;
        return nn_coarse(g, y, d2_max, d2);
    }
    const int ix = static_cast<int>(fx), iy = static_cast<int>(fy), iz = static_cast<int>(fz);
    if (ix < 0 || iy < 0 || iz < 0 || ix >= g.fnx || iy >= g.fny || iz >= g.fnz) return -1;
    const int2 bi = __ldg(g.fine_info + (static_cast<int64_t>(ix) * g.fny + iy) * g.fnz + iz);
    if (bi.y == 0) return -1;
    const float inf = __int_as_float(0x7f800000);
    float f1 = inf, f2 = inf, f3 = inf;
    int32_t o1 = -1, o2 = -1;
    const int32_t end = bi.x + bi.y;
    int32_t e = bi.x;
    for (; e + 1 < end; e += 2) {
        const float4 A = __ldg(g.fine_pts + e), B = __ldg(g.fine_pts + e + 1);
        float x = qx - A.x, yy = qy - A.y, z = qz - A.z;
        top3(fmaf(x, x, fmaf(yy, yy, z * z)), __float_as_int(A.w), f1, f2, f3, o1, o2);
        x = qx - B.x; yy = qy - B.y; z = qz - B.z;
        top3(fmaf(x, x, fmaf(yy, yy, z * z)), __float_as_int(B.w), f1, f2, f3, o1, o2);
    }
    if (e < end) {
        const float4 A = __ldg(g.fine_pts + e);
        const float x = qx - A.x, yy = qy - A.y, z = qz - A.z;
        top3(fmaf(x, x, fmaf(yy, yy, z * z)), __float_as_int(A.w), f1, f2, f3, o1, o2);
    }
    const float band = F.band;
    if (f1 > F.pad + band) return -1;
    double best_d2 = __longlong_as_double(0x7ff0000000000000ll);
    int32_t best = INT32_MAX;
    auto consider = [&](int32_t o) {
        const V3 q = ld4(g.pos4_orig, o);
        const double d2 = sqnorm(sub(q, y));
        if (d2 > d2_max) return;
        if (d2 < best_d2 || (d2 == best_d2 && o < best)) {
            best_d2 = d2;
            best = o;
        }
    };
    const float lim = f1 + 2.0f * band;
    if (f3 <= lim) {
        for (int32_t k = bi.x; k < end; ++k) {
            const float4 E = __ldg(g.fine_pts + k);
            const float dx = qx - E.x, dy = qy - E.y, dz = qz - E.z;
            if (fmaf(dx, dx, fmaf(dy, dy, dz * dz)) <= lim) consider(__float_as_int(E.w));
        }
    } else {
        consider(o1);
        if (f2 <= lim) consider(o2);
    }
    return best == INT32_MAX ? -1 : best;
}

__device__ __forceinline__ double butterfly(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

__global__ void __launch_bounds__(kIcpThreads) k_icp_accum(const float4* __restrict__ pos32,
                                                           const double4* __restrict__ pos4, int64_t n,
                                                           const __grid_constant__ GridView g, double d2_max,
                                                           const IcpState* __restrict__ st,
                                                           double* __restrict__ partial,
                                                           unsigned long long* __restrict__ count) {
    if (st->done) return;
    __shared__ double s_R[12];
    __shared__ FastRT s_F;
    __shared__ double s_w[kIcpThreads / 32][kIcpVals];
    if (threadIdx.x < 12) s_R[threadIdx.x] = threadIdx.x < 9 ? st->R[threadIdx.x] : st->t[threadIdx.x - 9];
    if (threadIdx.x == 0) s_F = st->F;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n_chunks = (n + kIcpThreads - 1) / kIcpThreads;
    unsigned long long cnt = 0;
    for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        const int64_t i = c * kIcpThreads + threadIdx.x;
        double J[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        double r = 0.0;
        if (i < n) {
            V3 y;
            const int32_t j = nn_fine(g, s_F, s_R, s_R + 9, __ldg(pos32 + i), ld4(pos4, i), d2_max, y);
            if (j >= 0) {
                const V3 nn = ld3(g.nrm_orig, j);
                if (!is_zero(nn)) {
                    const V3 q = ld4(g.pos4_orig, j);
                    r = dot(sub(y, q), nn);
                    J[0] = y.y * nn.z - y.z * nn.y;
                    J[1] = y.z * nn.x - y.x * nn.z;
                    J[2] = y.x * nn.y - y.y * nn.x;
                    J[3] = nn.x;
                    J[4] = nn.y;
                    J[5] = nn.z;
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
                                                             int64_t n_source, const __grid_constant__ GridView g,
                                                             ScoreParams sp, IcpState* __restrict__ st,
                                                             double* __restrict__ history, int32_t iteration,
                                                             double eps2) {
    if (st->done) return;
    __shared__ double s_tot[kIcpVals];
    const int lane = threadIdx.x & 31, v = threadIdx.x >> 5;
    double acc = 0.0;
    for (int64_t s0 = 0; s0 < n_chunks; s0 += 32) {
        const double x = s0 + lane < n_chunks ? partial[(s0 + lane) * kIcpVals + v] : 0.0;
        acc = acc + butterfly(x);
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
    st->F = make_fast_fine(st->R, st->t, g, sp);
    if (dd < eps2) {
        st->converged = 1;
        st->done = 1;
    }
}

__global__ void k_icp_init(IcpState* st, const __grid_constant__ GridView g, ScoreParams sp) {
    st->F = make_fast_fine(st->R, st->t, g, sp);
}

__global__ void k_max_norm(const double* __restrict__ p, int64_t n, unsigned long long* out) {
    double m = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double x = p[3 * i], y = p[3 * i + 1], z = p[3 * i + 2];
        m = fmax(m, sqrt(x * x + y * y + z * z));
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(kFull, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(m)));
}

}  // namespace

cudaError_t icp_point_to_plane(const double* d_src, int64_t n, const GridStorage& grid, double max_dist,
                               int32_t max_iter, double eps, const double* R0, const double* t0, double* R9,
                               double* t3, IcpOutcome* out, double* d_history, cudaStream_t stream, int sm_count,
                               bool fast) {
    const GridView& g = grid.view;
    float4* pos32 = nullptr;
    double4* pos4 = nullptr;
    double* partial = nullptr;
    unsigned long long* counts = nullptr;
    IcpState* st = nullptr;
    const int64_t n_chunks = (n + kIcpThreads - 1) / kIcpThreads;
    cudaError_t e;
    auto cleanup = [&] {
        pool_free(pos32, stream);
        pool_free(pos4, stream);
        pool_free(partial, stream);
        pool_free(counts, stream);
        pool_free(st, stream);
    };
#define ICP_TRY(x)            \
    do {                      \
        e = (x);              \
        if (e != cudaSuccess) { \
            cleanup();        \
            return e;         \
        }                     \
    } while (0)
    ICP_TRY(pool_alloc(&pos32, n * sizeof(float4), stream));
    ICP_TRY(pool_alloc(&pos4, n * sizeof(double4), stream));
    ICP_TRY(pool_alloc(&partial, n_chunks * kIcpVals * sizeof(double), stream));
    const int32_t iters = max_iter > 0 ? max_iter : 0;
    ICP_TRY(pool_alloc(&counts, (iters + 1) * sizeof(unsigned long long), stream));
    ICP_TRY(pool_alloc(&st, sizeof(IcpState), stream));
    ICP_TRY(make_source32(d_src, n, pos32, stream));
    ICP_TRY(make_records(d_src, nullptr, n, pos4, nullptr, stream));
    // |p|max for the FP32 guard bands (ScoreParams::pmax_cells)
    ICP_TRY(cudaMemsetAsync(counts, 0, (iters + 1) * sizeof(unsigned long long), stream));
    k_max_norm<<<sm_count * 2, 256, 0, stream>>>(d_src, n, counts + iters);
    unsigned long long mbits = 0;
    ICP_TRY(cudaMemcpyAsync(&mbits, counts + iters, sizeof(mbits), cudaMemcpyDeviceToHost, stream));
    ICP_TRY(cudaStreamSynchronize(stream));
    double pmax;
    static_assert(sizeof(pmax) == sizeof(mbits), "bits");
    __builtin_memcpy(&pmax, &mbits, sizeof(pmax));
    ScoreParams sp{};
    sp.d_max = max_dist;
    sp.d2_max = max_dist * max_dist;
    if (fast) configure_fast_path(sp, g, pmax);  // else sp.fast = 0: exact FP64 NN for every point
    IcpState h{};
    for (int k = 0; k < 9; ++k) h.R[k] = R0[k];
    for (int k = 0; k < 3; ++k) h.t[k] = t0[k];
    ICP_TRY(cudaMemcpyAsync(st, &h, sizeof(h), cudaMemcpyHostToDevice, stream));
    k_icp_init<<<1, 1, 0, stream>>>(st, g, sp);
    const int blocks = static_cast<int>(n_chunks < sm_count * 8 ? n_chunks : sm_count * 8);
    for (int32_t it = 0; it < iters; ++it) {
        k_icp_accum<<<blocks, kIcpThreads, 0, stream>>>(pos32, pos4, n, g, sp.d2_max, st, partial, counts + it);
        k_icp_solve<<<1, kIcpVals * 32, 0, stream>>>(partial, n_chunks, counts + it, n, g, sp, st, d_history, it,
                                                     eps * eps);
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
