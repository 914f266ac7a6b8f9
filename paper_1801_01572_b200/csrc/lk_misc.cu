// lk_misc.cu -- feature pre-match (K1, the reference binary's float matcher), edge_info (K8), point transforms.
#include <cstdint>
#include <algorithm>
#include <cstdlib>

#include "lk_device_math.cuh"
#include "lk_kernels.cuh"

namespace lkk {

using namespace lkd;

namespace {

constexpr int kFeatDim = 33;
constexpr int kFeatThreads = 128;

// ---- feature pre-match (K1): the reference binary's float matcher ---------
// proj/src/grid.cpp:176-213: score_j = |q_j|^2 - 2 (Q^T f)_j in FP32 through
// Eigen (x86-64 SSE2, no FMA), argmin with strict < over ascending j (ties ->
// lowest j). Every score is reproduced bit for bit (the order below is Eigen
// 3.4's, restated in oracle/lk_oracle.cpp and oracle/ref_shim/Eigen/Dense and
// checked against the reference build there), so the argmin needs no
// tie-band rescan:
//   |q|^2 (colwise().squaredNorm(), redux_impl LinearVectorized): 4-lane
//     accumulators r0 = packets 0,2,4,6 and r1 = packets 1,3,5,7 (adds in
//     order), r0 + r1, predux (l0 + l2) + (l1 + l3), + q32^2;
//   (Q^T f)_j (row-major general_matrix_vector_product): lanes
//     c_l = (((0 + a_l b_l) + a_{4+l} b_{4+l}) + ...) over the 8 whole
//     packets, predux (c0 + c2) + (c1 + c3), + a32 b32, times alpha 2 (exact).
// Products and sums are separately rounded (mul/add .rn, packed FP32x2 where
// two lanes run the same chain), never fused.
constexpr int kFnnThreads = 128;
constexpr int kFnnTile = 64;
constexpr int kFnnPad = 36;  // 33 bins padded to 9 float4

struct BestF {
    float s;
    int32_t j;
};

// Products as scalar FMUL, lane sums as packed FADD2 (.x = first lane, .y =
// second). A packed product is not usable: ptxas contracts mul.rn.f32x2 ->
// add.rn.f32x2 (also through __fmul2_rn / __fadd2_rn and with -fmad=false)
// into FFMA2, which rounds once instead of twice. Scalar __fmul_rn feeding
// __fadd2_rn stays two roundings (checked in the SASS: FMUL + FADD2, no FFMA2).
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul_pair(float a0, float b0, float a1, float b1) {
    return make_float2(__fmul_rn(a0, b0), __fmul_rn(a1, b1));
}

// colwise().squaredNorm() of one 33-bin feature, Eigen's order
__device__ __forceinline__ float eigen_qnorm33(const float* q) {
    float r0[4], r1[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
        r0[l] = __fmul_rn(q[l], q[l]);
        r1[l] = __fmul_rn(q[4 + l], q[4 + l]);
    }
#pragma unroll
    for (int idx = 8; idx < 32; idx += 8)
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            r0[l] = __fadd_rn(r0[l], __fmul_rn(q[idx + l], q[idx + l]));
            r1[l] = __fadd_rn(r1[l], __fmul_rn(q[idx + 4 + l], q[idx + 4 + l]));
        }
#pragma unroll
    for (int l = 0; l < 4; ++l) r0[l] = __fadd_rn(r0[l], r1[l]);
    const float res = __fadd_rn(__fadd_rn(r0[0], r0[2]), __fadd_rn(r0[1], r0[3]));
    return __fadd_rn(res, __fmul_rn(q[32], q[32]));
}

// one score, scalar: the exhaustive path (LK_FP64_ONLY=1) and the reference
// for the packed kernel below
__device__ __forceinline__ float eigen_score(float q2, const float* a, const float* b) {
    float c[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int k = 0; k < 32; k += 4)
#pragma unroll
        for (int l = 0; l < 4; ++l) c[l] = __fadd_rn(__fmul_rn(a[k + l], b[k + l]), c[l]);
    float cc = __fadd_rn(__fadd_rn(c[0], c[2]), __fadd_rn(c[1], c[3]));
    cc = __fadd_rn(cc, __fmul_rn(a[32], b[32]));
    return __fsub_rn(q2, __fmul_rn(2.0f, cc));
}

// exhaustive: one thread per source over every target in order
__global__ void __launch_bounds__(kFeatThreads) k_feature_nn_exact(const float* __restrict__ sf, int64_t ns,
                                                                   const float* __restrict__ tf, int64_t nt,
                                                                   const float* __restrict__ q2,
                                                                   int32_t* __restrict__ out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= ns) return;
    float f[kFeatDim];
    for (int b = 0; b < kFeatDim; ++b) f[b] = sf[i * kFeatDim + b];
    int32_t best = 0;
    float best_s = eigen_score(q2[0], tf, f);
    for (int64_t j = 1; j < nt; ++j) {
        const float s = eigen_score(q2[j], tf + j * kFeatDim, f);
        if (s < best_s) {
            best_s = s;
            best = static_cast<int32_t>(j);
        }
    }
    out[i] = best;
}

// q2 (optional): |q|^2 per feature, by the thread of its first float4
__global__ void k_pad_features(const float* __restrict__ f, int64_t n, float4* __restrict__ out,
                               float* __restrict__ q2) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= n * (kFnnPad / 4)) return;
    const int64_t i = t / (kFnnPad / 4), q = t % (kFnnPad / 4);
    if (q2 && q == 0) q2[i] = eigen_qnorm33(f + i * kFeatDim);
    float v[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int b = static_cast<int>(4 * q + c);
        v[c] = b < kFeatDim ? f[i * kFeatDim + b] : 0.0f;
    }
    out[t] = make_float4(v[0], v[1], v[2], v[3]);
}

// grid (source blocks, target chunks): the chunk's best (score, lowest j) per
// source. Target tiles staged in shared memory and read as broadcasts; four
// targets at a time, the lane pairs (0,1) and (2,3) of Eigen's 4-lane
// accumulators as packed FP32x2 chains (two FMUL + one FADD2 per two bins).
// Two source points per thread (i and i + kFnnThreads of the block's
// 2 * kFnnThreads): every staged target bin read from shared memory feeds
// both, halving the loads per score.
__global__ void __launch_bounds__(kFnnThreads) k_fnn_partial(const float4* __restrict__ sf, int64_t ns,
                                                             const float4* __restrict__ tf,
                                                             const float* __restrict__ q2, int64_t nt,
                                                             int64_t chunk, BestF* __restrict__ partial) {
    __shared__ float4 s_t[kFnnTile * (kFnnPad / 4)];
    __shared__ float s_q2[kFnnTile];
    const int64_t i0 = blockIdx.x * static_cast<int64_t>(2 * kFnnThreads) + threadIdx.x;
    const int64_t i1 = i0 + kFnnThreads;
    float2 xa01[8], xa23[8], xb01[8], xb23[8];
    float xa32, xb32;
    {
        float4 s[kFnnPad / 4];
#pragma unroll
        for (int q = 0; q < kFnnPad / 4; ++q) s[q] = i0 < ns ? sf[i0 * (kFnnPad / 4) + q] : make_float4(0, 0, 0, 0);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            xa01[q] = make_float2(s[q].x, s[q].y);
            xa23[q] = make_float2(s[q].z, s[q].w);
        }
        xa32 = s[8].x;
#pragma unroll
        for (int q = 0; q < kFnnPad / 4; ++q) s[q] = i1 < ns ? sf[i1 * (kFnnPad / 4) + q] : make_float4(0, 0, 0, 0);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            xb01[q] = make_float2(s[q].x, s[q].y);
            xb23[q] = make_float2(s[q].z, s[q].w);
        }
        xb32 = s[8].x;
    }
    const int64_t j_begin = blockIdx.y * chunk;
    const int64_t j_end = j_begin + chunk < nt ? j_begin + chunk : nt;
    float best_a = __int_as_float(0x7f800000), best_b = best_a;
    int32_t ja = -1, jb = -1;
    for (int64_t j0 = j_begin; j0 < j_end; j0 += kFnnTile) {
        const int tile = static_cast<int>(j_end - j0 < kFnnTile ? j_end - j0 : kFnnTile);
        __syncthreads();
        for (int q = threadIdx.x; q < tile * (kFnnPad / 4); q += kFnnThreads) s_t[q] = tf[j0 * (kFnnPad / 4) + q];
        for (int q = threadIdx.x; q < tile; q += kFnnThreads) s_q2[q] = q2[j0 + q];
        __syncthreads();
        auto take = [&](float sc, int jj, float& bs, int32_t& bj) {
            if (sc < bs || bj < 0) {
                bs = sc;
                bj = static_cast<int32_t>(j0 + jj);
            }
        };
        int jj = 0;
        for (; jj + 2 <= tile; jj += 2) {
            float2 a01[2], a23[2], b01[2], b23[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const float4 y = s_t[(jj + u) * (kFnnPad / 4)];
                a01[u] = mul_pair(y.x, xa01[0].x, y.y, xa01[0].y);  // 0 + a b == a b (features are >= 0)
                a23[u] = mul_pair(y.z, xa23[0].x, y.w, xa23[0].y);
                b01[u] = mul_pair(y.x, xb01[0].x, y.y, xb01[0].y);
                b23[u] = mul_pair(y.z, xb23[0].x, y.w, xb23[0].y);
            }
#pragma unroll
            for (int q = 1; q < 8; ++q)
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const float4 y = s_t[(jj + u) * (kFnnPad / 4) + q];
                    a01[u] = add2(mul_pair(y.x, xa01[q].x, y.y, xa01[q].y), a01[u]);
                    a23[u] = add2(mul_pair(y.z, xa23[q].x, y.w, xa23[q].y), a23[u]);
                    b01[u] = add2(mul_pair(y.x, xb01[q].x, y.y, xb01[q].y), b01[u]);
                    b23[u] = add2(mul_pair(y.z, xb23[q].x, y.w, xb23[q].y), b23[u]);
                }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const float y32 = s_t[(jj + u) * (kFnnPad / 4) + 8].x, qq = s_q2[jj + u];
                const float2 pa = add2(a01[u], a23[u]), pb = add2(b01[u], b23[u]);  // (c0 + c2, c1 + c3)
                float ca = __fadd_rn(pa.x, pa.y), cb = __fadd_rn(pb.x, pb.y);
                ca = __fadd_rn(ca, __fmul_rn(y32, xa32));
                cb = __fadd_rn(cb, __fmul_rn(y32, xb32));
                take(__fsub_rn(qq, __fmul_rn(2.0f, ca)), jj + u, best_a, ja);
                take(__fsub_rn(qq, __fmul_rn(2.0f, cb)), jj + u, best_b, jb);
            }
        }
        for (; jj < tile; ++jj) {
            const float* t = reinterpret_cast<const float*>(s_t + jj * (kFnnPad / 4));
            float fa[kFnnPad], fb[kFnnPad];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                fa[4 * q] = xa01[q].x, fa[4 * q + 1] = xa01[q].y, fa[4 * q + 2] = xa23[q].x, fa[4 * q + 3] = xa23[q].y;
                fb[4 * q] = xb01[q].x, fb[4 * q + 1] = xb01[q].y, fb[4 * q + 2] = xb23[q].x, fb[4 * q + 3] = xb23[q].y;
            }
            fa[32] = xa32;
            fb[32] = xb32;
            take(eigen_score(s_q2[jj], t, fa), jj, best_a, ja);
            take(eigen_score(s_q2[jj], t, fb), jj, best_b, jb);
        }
    }
    if (i0 < ns) partial[blockIdx.y * ns + i0] = BestF{best_a, ja};
    if (i1 < ns) partial[blockIdx.y * ns + i1] = BestF{best_b, jb};
}

// chunks in ascending j order, strict <: the lowest index wins ties
__global__ void k_fnn_merge(int64_t ns, const BestF* __restrict__ partial, int n_chunks, int32_t* __restrict__ out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= ns) return;
    BestF b = partial[i];
    for (int c = 1; c < n_chunks; ++c) {
        const BestF p = partial[c * ns + i];
        if (p.s < b.s) b = p;
    }
    out[i] = b.j;
}

struct Xf {
    double r[9], t[3];
};

__global__ void k_transform(const double* __restrict__ in, int64_t n, Xf T, double* __restrict__ out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    V3 y = xform(T.r, T.t, ld3(in, i));
    out[3 * i] = y.x;
    out[3 * i + 1] = y.y;
    out[3 * i + 2] = y.z;
}

constexpr int kInfoThreads = 256;

// edge_info (proj/src/line_process.cpp:11-33): per point of cloud_i whose
// posed position has any posed cloud_j point within eps (nn_within existence),
// accumulate G^T G with G = [-[p]x | I] (p local). Per-CTA partial sums are
// reduced in a fixed order by k_info_final (deterministic).
__global__ void __launch_bounds__(kInfoThreads) k_edge_info(const double* __restrict__ ci, int64_t ni, Xf Ti,
                                                            GridView g, double eps2,
                                                            double* __restrict__ partials,
                                                            unsigned long long* __restrict__ count) {
    __shared__ double s_acc[kInfoThreads / 32][21];
    double acc[21];
#pragma unroll
    for (int q = 0; q < 21; ++q) acc[q] = 0.0;
    unsigned long long hits = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < ni;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        V3 p = ld3(ci, i);
        V3 y = xform(Ti.r, Ti.t, p);
        double fx = floor((y.x - g.ox) / g.cell) - static_cast<double>(g.offx);
        double fy = floor((y.y - g.oy) / g.cell) - static_cast<double>(g.offy);
        double fz = floor((y.z - g.oz) / g.cell) - static_cast<double>(g.offz);
        if (!(fx >= 0.0 && fy >= 0.0 && fz >= 0.0 && fx < g.nx && fy < g.ny && fz < g.nz)) continue;
        const int ix = static_cast<int>(fx), iy = static_cast<int>(fy), iz = static_cast<int>(fz);
        if (!g.near[(static_cast<int64_t>(ix) * g.ny + iy) * g.nz + iz]) continue;
        const int r = g.radius;
        bool found = false;
        for (int x = max(ix - r, 0); x <= min(ix + r, g.nx - 1) && !found; ++x)
            for (int yy = max(iy - r, 0); yy <= min(iy + r, g.ny - 1) && !found; ++yy) {
                const int64_t row = (static_cast<int64_t>(x) * g.ny + yy) * g.nz;
                const int32_t s0 = g.start[row + max(iz - r, 0)];
                const int32_t s1 = g.start[row + min(iz + r, g.nz - 1) + 1];
                for (int32_t s = s0; s < s1; ++s)
                    if (sqnorm(sub(ld3(g.slot_pos, s), y)) <= eps2) {
                        found = true;
                        break;
                    }
            }
        if (!found) continue;
        hits += 1;
        // a = -[p]x ; TL += a^T a (6 unique), TR += a^T, BL += a, BR += I
        const double a[3][3] = {{-0.0, p.z, -p.y}, {-p.z, -0.0, p.x}, {p.y, -p.x, -0.0}};
        int q = 0;
#pragma unroll
        for (int rr = 0; rr < 3; ++rr)
#pragma unroll
            for (int cc = rr; cc < 3; ++cc)
                acc[q++] += (a[0][rr] * a[0][cc] + a[1][rr] * a[1][cc]) + a[2][rr] * a[2][cc];
        acc[6] += p.x;
        acc[7] += p.y;
        acc[8] += p.z;
    }
    // block reduction of the 9 accumulated sums (rest unused)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < 9; ++q) {
        double v = acc[q];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) s_acc[warp][q] = v;
    }
    for (int o = 16; o > 0; o >>= 1) hits += __shfl_xor_sync(0xffffffffu, hits, o);
    __syncthreads();
    if (threadIdx.x < 9) {
        double v = 0.0;
        for (int w = 0; w < kInfoThreads / 32; ++w) v += s_acc[w][threadIdx.x];
        partials[blockIdx.x * 9 + threadIdx.x] = v;
    }
    if (lane == 0 && hits) atomicAdd(count, hits);
}

// Assemble the 6x6 from the fixed-order sum of the per-CTA partials:
// TL = sum a^T a, TR = sum a^T = sum [p]x, BL = sum a = -sum [p]x, BR = n I.
__global__ void k_info_final(const double* __restrict__ partials, int nb, const unsigned long long* __restrict__ count,
                             double* __restrict__ info) {
    __shared__ double s[9];
    if (threadIdx.x < 9) {
        double v = 0.0;
        for (int b = 0; b < nb; ++b) v += partials[b * 9 + threadIdx.x];
        s[threadIdx.x] = v;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    double L[6][6];
    for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c) L[r][c] = 0.0;
    int q = 0;
    for (int r = 0; r < 3; ++r)
        for (int c = r; c < 3; ++c) {
            L[r][c] = s[q];
            L[c][r] = s[q];
            ++q;
        }
    const double px = s[6], py = s[7], pz = s[8];
    // a = -[p]x = [[0, pz, -py], [-pz, 0, px], [py, -px, 0]] (summed)
    const double A[3][3] = {{0.0, pz, -py}, {-pz, 0.0, px}, {py, -px, 0.0}};
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            L[r][3 + c] = A[c][r];
            L[3 + r][c] = A[r][c];
        }
    const double n = static_cast<double>(*count);
    for (int r = 0; r < 3; ++r) L[3 + r][3 + r] = n;
    for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c) info[6 * r + c] = L[r][c];
}

}  // namespace

size_t fnn_padded_bytes(int64_t n) { return static_cast<size_t>(n > 0 ? n : 1) * kFnnPad * sizeof(float); }

cudaError_t fnn_prepare(const float* d_f, int64_t n, float4* d_padded, float* d_q2, cudaStream_t stream) {
    if (n > 0)
        k_pad_features<<<static_cast<unsigned>((n * (kFnnPad / 4) + 255) / 256), 256, 0, stream>>>(d_f, n, d_padded,
                                                                                                 d_q2);
    return cudaGetLastError();
}

cudaError_t feature_nn_prepared(const float* d_sf, const float4* d_sp, int64_t ns, const float* d_tf,
                                const float4* d_tp, const float* d_q2, int64_t nt, int32_t* d_out,
                                cudaStream_t stream) {
    if (const char* v = std::getenv("LK_FP64_ONLY"); v && v[0] == '1') {
        const unsigned blocks = static_cast<unsigned>((ns + kFeatThreads - 1) / kFeatThreads);
        k_feature_nn_exact<<<blocks, kFeatThreads, 0, stream>>>(d_sf, ns, d_tf, nt, d_q2, d_out);
        return cudaGetLastError();
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t src_blocks = (ns + 2 * kFnnThreads - 1) / (2 * kFnnThreads);
    int64_t n_chunks = (8 * sms + src_blocks - 1) / src_blocks;
    if (n_chunks < 1) n_chunks = 1;
    if (n_chunks > (nt + kFnnTile - 1) / kFnnTile) n_chunks = (nt + kFnnTile - 1) / kFnnTile;
    const int64_t chunk = (nt + n_chunks - 1) / n_chunks;
    n_chunks = (nt + chunk - 1) / chunk;
    Scratch sc(stream, Scratch::round(n_chunks * ns * sizeof(BestF)));
    BestF* partial = sc.take<BestF>(n_chunks * ns);
    cudaError_t e = sc.status();
    if (e != cudaSuccess) return e;
    k_fnn_partial<<<dim3(static_cast<unsigned>(src_blocks), static_cast<unsigned>(n_chunks)), kFnnThreads, 0,
                    stream>>>(d_sp, ns, d_tp, d_q2, nt, chunk, partial);
    k_fnn_merge<<<static_cast<unsigned>((ns + 255) / 256), 256, 0, stream>>>(ns, partial, static_cast<int>(n_chunks),
                                                                            d_out);
    return cudaGetLastError();
}

cudaError_t feature_nn(const float* d_sf, int64_t ns, const float* d_tf, int64_t nt, int32_t* d_out,
                       cudaStream_t stream) {
    float* q2 = nullptr;
    float4 *sp = nullptr, *tp = nullptr;
    cudaError_t e;
    if ((e = pool_alloc(&q2, std::max<int64_t>(nt, 1) * sizeof(float), stream)) != cudaSuccess) return e;
    if ((e = pool_alloc(&sp, fnn_padded_bytes(ns), stream)) != cudaSuccess) return e;
    if ((e = pool_alloc(&tp, fnn_padded_bytes(nt), stream)) != cudaSuccess) return e;
    if ((e = fnn_prepare(d_sf, ns, sp, nullptr, stream)) == cudaSuccess &&
        (e = fnn_prepare(d_tf, nt, tp, q2, stream)) == cudaSuccess)
        e = feature_nn_prepared(d_sf, sp, ns, d_tf, tp, q2, nt, d_out, stream);
    pool_free(sp, stream);
    pool_free(tp, stream);
    pool_free(q2, stream);
    return e;
}

cudaError_t transform_points(const double* d_in, int64_t n, const double* T12, double* d_out, cudaStream_t stream) {
    Xf T;
    for (int k = 0; k < 9; ++k) T.r[k] = T12[k];
    for (int k = 0; k < 3; ++k) T.t[k] = T12[9 + k];
    k_transform<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(d_in, n, T, d_out);
    return cudaGetLastError();
}

cudaError_t edge_info(const double* d_ci, int64_t ni, const double* Ti12, const GridView& grid, double eps,
                      double* d_partials, int n_partial_blocks, double* d_info, unsigned long long* d_count,
                      cudaStream_t stream) {
    Xf T;
    for (int k = 0; k < 9; ++k) T.r[k] = Ti12[k];
    for (int k = 0; k < 3; ++k) T.t[k] = Ti12[9 + k];
    cudaError_t e = cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), stream);
    if (e != cudaSuccess) return e;
    k_edge_info<<<n_partial_blocks, kInfoThreads, 0, stream>>>(d_ci, ni, T, grid, eps * eps, d_partials, d_count);
    k_info_final<<<1, 32, 0, stream>>>(d_partials, n_partial_blocks, d_count, d_info);
    return cudaGetLastError();
}

}  // namespace lkk
