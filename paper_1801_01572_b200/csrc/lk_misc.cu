// lk_misc.cu -- feature pre-match (K1), edge_info (K8), point transforms.
#include <cstdint>
#include <cstdlib>

#include "lk_device_math.cuh"
#include "lk_kernels.cuh"

namespace lkk {

using namespace lkd;

namespace {

constexpr int kFeatDim = 33;
constexpr int kFeatThreads = 128;
constexpr int kFeatTile = 128;

// argmin_j sum_b (double(s_b) - double(t_b))^2, strict < over ascending j
// (proj/include/loopkit/reference.hpp:56-76). One thread per source feature;
// target features are staged through shared memory tile by tile and read as
// broadcasts.
__global__ void __launch_bounds__(kFeatThreads) k_feature_nn(const float* __restrict__ sf, int64_t ns,
                                                             const float* __restrict__ tf, int64_t nt,
                                                             int32_t* __restrict__ out) {
    __shared__ float s_t[kFeatTile * kFeatDim];
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    float f[kFeatDim];
#pragma unroll
    for (int b = 0; b < kFeatDim; ++b) f[b] = i < ns ? sf[i * kFeatDim + b] : 0.0f;
    double best_d2 = __longlong_as_double(0x7ff0000000000000ll);
    int32_t best = -1;
    for (int64_t j0 = 0; j0 < nt; j0 += kFeatTile) {
        const int64_t tile = nt - j0 < kFeatTile ? nt - j0 : kFeatTile;
        __syncthreads();
        for (int64_t q = threadIdx.x; q < tile * kFeatDim; q += blockDim.x) s_t[q] = tf[j0 * kFeatDim + q];
        __syncthreads();
        for (int jj = 0; jj < tile; ++jj) {
            const float* t = s_t + jj * kFeatDim;
            double d2 = 0.0;
#pragma unroll
            for (int b = 0; b < kFeatDim; ++b) {
                double diff = static_cast<double>(f[b]) - static_cast<double>(t[b]);
                d2 += diff * diff;
            }
            if (d2 < best_d2) {
                best_d2 = d2;
                best = static_cast<int32_t>(j0 + jj);
            }
        }
    }
    if (i < ns) out[i] = best;
}

// ---- FP32 pre-match with exact FP64 resolution of near-ties ---------------
// d2f = sum_b fl(s_b - t_b)^2 via fmaf is within (2 + 33 + 1) * 2^-24 < 2.2e-6
// relative of the exact d2 (all terms are non-negative). Every (source,
// target-chunk) keeps its FP32 best (value, lowest index) and runner-up;
// chunks merge in ascending order. A source whose runner-up lies within
// kTieRel of the best is resolved exactly in FP64 over all targets within
// that band (ties -> lowest index, as reference.hpp:56-76). d2f == 0 implies
// identical features, hence an exact zero: no resolution needed.
constexpr int kFnnThreads = 128;
constexpr int kFnnTile = 64;
constexpr int kFnnPad = 36;  // 33 bins padded to 9 float4
constexpr float kTieRel = 1e-5f;

struct Best3 {
    float f1;
    int32_t j1;
    float f2;
};

// packed FP32 pairs (sm_100a FADD2 / FFMA2): lo = first, hi = second
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
    return (static_cast<unsigned long long>(__float_as_uint(hi)) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ float2 unpack2(unsigned long long v) {
    return make_float2(__uint_as_float(static_cast<unsigned>(v)), __uint_as_float(static_cast<unsigned>(v >> 32)));
}
__device__ __forceinline__ unsigned long long sub2(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

__device__ __forceinline__ float feat_d2f(const float4* a, const float4* b) {
    float acc = 0.0f;
#pragma unroll
    for (int q = 0; q < kFnnPad / 4; ++q) {
        const float4 x = a[q], y = b[q];
        float d;
        d = x.x - y.x; acc = fmaf(d, d, acc);
        d = x.y - y.y; acc = fmaf(d, d, acc);
        d = x.z - y.z; acc = fmaf(d, d, acc);
        d = x.w - y.w; acc = fmaf(d, d, acc);
    }
    return acc;
}

__global__ void k_pad_features(const float* __restrict__ f, int64_t n, float4* __restrict__ out) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= n * (kFnnPad / 4)) return;
    const int64_t i = t / (kFnnPad / 4), q = t % (kFnnPad / 4);
    float v[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int b = static_cast<int>(4 * q + c);
        v[c] = b < kFeatDim ? f[i * kFeatDim + b] : 0.0f;
    }
    out[t] = make_float4(v[0], v[1], v[2], v[3]);
}

// grid (source blocks, target chunks): FP32 best / runner-up per pair
__global__ void __launch_bounds__(kFnnThreads) k_fnn_partial(const float4* __restrict__ sf, int64_t ns,
                                                             const float4* __restrict__ tf, int64_t nt,
                                                             int64_t chunk, Best3* __restrict__ partial) {
    __shared__ float4 s_t[kFnnTile * (kFnnPad / 4)];
    const int64_t i = blockIdx.x * static_cast<int64_t>(kFnnThreads) + threadIdx.x;
    float4 s[kFnnPad / 4];
#pragma unroll
    for (int q = 0; q < kFnnPad / 4; ++q) s[q] = i < ns ? sf[i * (kFnnPad / 4) + q] : make_float4(0, 0, 0, 0);
    const int64_t j_begin = blockIdx.y * chunk;
    const int64_t j_end = j_begin + chunk < nt ? j_begin + chunk : nt;
    float f1 = __int_as_float(0x7f800000), f2 = f1;
    int32_t j1 = -1;
    for (int64_t j0 = j_begin; j0 < j_end; j0 += kFnnTile) {
        const int tile = static_cast<int>(j_end - j0 < kFnnTile ? j_end - j0 : kFnnTile);
        __syncthreads();
        for (int q = threadIdx.x; q < tile * (kFnnPad / 4); q += kFnnThreads) s_t[q] = tf[j0 * (kFnnPad / 4) + q];
        __syncthreads();
        auto take = [&](float d2, int64_t j) {
            if (d2 < f1) {
                f2 = f1;
                f1 = d2;
                j1 = static_cast<int32_t>(j);
            } else if (d2 < f2) {
                f2 = d2;
            }
        };
        int jj = 0;
        // four targets at a time, two partial sums each (bins x, z and y, w of
        // every float4): eight independent FMA chains, run as packed FP32x2
        // pairs (FADD2 / FFMA2: one instruction per two bins). Any summation
        // order stays within the 2.2e-6 bound the near-tie rescan assumes.
        for (; jj + 4 <= tile; jj += 4) {
            unsigned long long a[4] = {0ull, 0ull, 0ull, 0ull};  // (even, odd) partial sums
#pragma unroll
            for (int q = 0; q < kFnnPad / 4; ++q) {
                const float4 x = s[q];
                const unsigned long long xlo = pack2(x.x, x.y), xhi = pack2(x.z, x.w);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float4 y = s_t[(jj + u) * (kFnnPad / 4) + q];
                    const unsigned long long dlo = sub2(xlo, pack2(y.x, y.y));
                    a[u] = fma2(dlo, dlo, a[u]);
                    const unsigned long long dhi = sub2(xhi, pack2(y.z, y.w));
                    a[u] = fma2(dhi, dhi, a[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float2 v = unpack2(a[u]);
                take(v.x + v.y, j0 + jj + u);
            }
        }
        for (; jj < tile; ++jj) take(feat_d2f(s, s_t + jj * (kFnnPad / 4)), j0 + jj);
    }
    if (i < ns) partial[blockIdx.y * ns + i] = Best3{f1, j1, f2};
}

__global__ void k_fnn_merge(const float4* __restrict__ sf, const float* __restrict__ sraw, int64_t ns,
                            const float4* __restrict__ tf, const float* __restrict__ traw, int64_t nt,
                            const Best3* __restrict__ partial, int n_chunks, int32_t* __restrict__ out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= ns) return;
    Best3 b = partial[i];
    for (int c = 1; c < n_chunks; ++c) {
        const Best3 p = partial[c * ns + i];
        if (p.f1 < b.f1) {
            b.f2 = fminf(b.f1, p.f2);
            b.f1 = p.f1;
            b.j1 = p.j1;
        } else {
            b.f2 = fminf(b.f2, p.f1);  // equal values keep the earlier (lower) index
        }
    }
    int32_t best = b.j1;
    if (b.f1 > 0.0f && b.f2 <= b.f1 * (1.0f + kTieRel)) {
        // near-tie: exact FP64 distances for every target within the band
        const float lim = b.f1 * (1.0f + kTieRel);
        float4 s[kFnnPad / 4];
#pragma unroll
        for (int q = 0; q < kFnnPad / 4; ++q) s[q] = sf[i * (kFnnPad / 4) + q];
        double best_d2 = __longlong_as_double(0x7ff0000000000000ll);
        best = -1;
        for (int64_t j = 0; j < nt; ++j) {
            if (feat_d2f(s, tf + j * (kFnnPad / 4)) > lim) continue;
            double d2 = 0.0;
            for (int q = 0; q < kFeatDim; ++q) {
                const double diff = static_cast<double>(sraw[i * kFeatDim + q]) - static_cast<double>(traw[j * kFeatDim + q]);
                d2 += diff * diff;
            }
            if (d2 < best_d2) {
                best_d2 = d2;
                best = static_cast<int32_t>(j);
            }
        }
    }
    out[i] = best;
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

cudaError_t feature_nn(const float* d_sf, int64_t ns, const float* d_tf, int64_t nt, int32_t* d_out,
                       cudaStream_t stream) {
    if (const char* v = std::getenv("LK_FP64_ONLY"); v && v[0] == '1') {
        const unsigned blocks = static_cast<unsigned>((ns + kFeatThreads - 1) / kFeatThreads);
        k_feature_nn<<<blocks, kFeatThreads, 0, stream>>>(d_sf, ns, d_tf, nt, d_out);
        return cudaGetLastError();
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t src_blocks = (ns + kFnnThreads - 1) / kFnnThreads;
    int64_t n_chunks = (8 * sms + src_blocks - 1) / src_blocks;
    if (n_chunks < 1) n_chunks = 1;
    if (n_chunks > (nt + kFnnTile - 1) / kFnnTile) n_chunks = (nt + kFnnTile - 1) / kFnnTile;
    const int64_t chunk = (nt + n_chunks - 1) / n_chunks;
    n_chunks = (nt + chunk - 1) / chunk;
    float4 *sp = nullptr, *tp = nullptr;
    Best3* partial = nullptr;
    cudaError_t e;
    if ((e = pool_alloc(&sp, ns * kFnnPad * sizeof(float), stream)) != cudaSuccess) return e;
    if ((e = pool_alloc(&tp, nt * kFnnPad * sizeof(float), stream)) != cudaSuccess) return e;
    if ((e = pool_alloc(&partial, n_chunks * ns * sizeof(Best3), stream)) != cudaSuccess) return e;
    k_pad_features<<<static_cast<unsigned>((ns * 9 + 255) / 256), 256, 0, stream>>>(d_sf, ns, sp);
    k_pad_features<<<static_cast<unsigned>((nt * 9 + 255) / 256), 256, 0, stream>>>(d_tf, nt, tp);
    k_fnn_partial<<<dim3(static_cast<unsigned>(src_blocks), static_cast<unsigned>(n_chunks)), kFnnThreads, 0,
                    stream>>>(sp, ns, tp, nt, chunk, partial);
    k_fnn_merge<<<static_cast<unsigned>((ns + 255) / 256), 256, 0, stream>>>(sp, d_sf, ns, tp, d_tf, nt, partial,
                                                                            static_cast<int>(n_chunks), d_out);
    pool_free(sp, stream);
    pool_free(tp, stream);
    pool_free(partial, stream);
    return cudaGetLastError();
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
