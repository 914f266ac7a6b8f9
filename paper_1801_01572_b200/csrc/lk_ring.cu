// lk_ring.cu -- exact nearest neighbour for dense targets (ICP, config D).
//
// The EvalGrid's 3x3x3 block lists grow with the square of the target density
// (a 640x480-rendered submap puts ~150 points in a 5 cm cell, ~4000 in its
// block). The ring grid instead bins the target into small cells (dense CSR
// over the bounding box, cell d_max / 5 coarsened for sparse targets, within a
// memory cap) and answers a query by scanning cube shells of cells around it
// in FP32, stopping as soon
// as no unscanned entry can be nearer (or tie), then deciding in FP64:
//   * FP32 keeps the three smallest d2; the stop test and the FP64 re-check
//     use guard bands sized from the conversion error of both coordinates;
//   * the winner (and every entry within the band) is re-evaluated with the
//     FP64 d2 and the (d2, original index) order;
//   * the result is the reference's EvalGrid neighbour
//     (registration.cpp:165-199): the query's EvalGrid cell must be inside the
//     grid, and a global nearest point outside the query's +-1 EvalGrid
//     window (possible only when a division rounds across a cell face) sends
//     the query to an exact scan of that window.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "lk_device_math.cuh"
#include "lk_kernels.cuh"

namespace lkk {

using namespace lkd;

namespace {

inline unsigned nblocks(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

__device__ __forceinline__ unsigned long long order_key(double d) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(d));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ inline double from_key(unsigned long long k) {
    const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    double d;
    memcpy(&d, &b, sizeof(d));
    return d;
}

// keys[0..2] = min, keys[3..5] = max (orderable encodings)
__global__ void k_ring_bbox(const double* __restrict__ p, int64_t n, unsigned long long* keys) {
    unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0ull, 0ull, 0ull};
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        for (int a = 0; a < 3; ++a) {
            const unsigned long long k = order_key(p[3 * i + a]);
            lo[a] = k < lo[a] ? k : lo[a];
            hi[a] = k > hi[a] ? k : hi[a];
        }
    for (int a = 0; a < 3; ++a) {
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long x = __shfl_xor_sync(0xffffffffu, lo[a], o);
            const unsigned long long y = __shfl_xor_sync(0xffffffffu, hi[a], o);
            lo[a] = x < lo[a] ? x : lo[a];
            hi[a] = y > hi[a] ? y : hi[a];
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(keys + a, lo[a]);
            atomicMax(keys + 3 + a, hi[a]);
        }
    }
}

__device__ __forceinline__ int ring_cell_axis(double v, double o, double cell, int n) {
    int c = static_cast<int>(floor((v - o) / cell));
    return c < 0 ? 0 : (c >= n ? n - 1 : c);
}

__global__ void k_ring_count(const double* __restrict__ p, int64_t n, RingGrid rg, int32_t* __restrict__ cell_of,
                             int32_t* __restrict__ counts) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int cx = ring_cell_axis(p[3 * i], rg.ox, rg.cell, rg.nx);
    const int cy = ring_cell_axis(p[3 * i + 1], rg.oy, rg.cell, rg.ny);
    const int cz = ring_cell_axis(p[3 * i + 2], rg.oz, rg.cell, rg.nz);
    const int64_t c = (static_cast<int64_t>(cx) * rg.ny + cy) * rg.nz + cz;
    cell_of[i] = static_cast<int32_t>(c);
    atomicAdd(counts + c, 1);
}

// sum over points of their cell's count (= sum over cells of count^2)
__global__ void k_ring_occupancy(const int32_t* __restrict__ cell_of, int64_t n, const int32_t* __restrict__ counts,
                                 unsigned long long* __restrict__ out) {
    unsigned long long acc = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        acc += static_cast<unsigned long long>(counts[cell_of[i]]);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

__global__ void k_ring_scatter(const double* __restrict__ p, int64_t n, RingGrid rg,
                               const int32_t* __restrict__ cell_of, int32_t* __restrict__ cursor,
                               float4* __restrict__ pts) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int32_t s = rg.start[cell_of[i]] + atomicAdd(cursor + cell_of[i], 1);
    pts[s] = make_float4(static_cast<float>((p[3 * i] - rg.ox) / rg.cell),
                         static_cast<float>((p[3 * i + 1] - rg.oy) / rg.cell),
                         static_cast<float>((p[3 * i + 2] - rg.oz) / rg.cell), __int_as_float(static_cast<int>(i)));
}


// Chebyshev distance transform of the cell occupancy, one axis per pass
// (the max-norm distance is separable): out = min over |d| <= K along the
// axis of max(|d|, in[c + d]), with in = 0 / K + 1 for occupied / empty cells
// on the first pass. Values saturate at K + 1 ("farther than K").
template <int AX, bool FIRST>
__global__ void k_ring_dt(const int32_t* __restrict__ start, const uint8_t* __restrict__ in, RingGrid rg, int K,
                          uint8_t* __restrict__ out) {
    const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (c >= rg.ncells) return;
    const int64_t plane = static_cast<int64_t>(rg.ny) * rg.nz;
    const int64_t stride = AX == 0 ? plane : (AX == 1 ? rg.nz : 1);
    const int n = AX == 0 ? rg.nx : (AX == 1 ? rg.ny : rg.nz);
    const int a = AX == 0 ? static_cast<int>(c / plane)
                          : (AX == 1 ? static_cast<int>((c / rg.nz) % rg.ny) : static_cast<int>(c % rg.nz));
    const int lo = a - K < 0 ? -a : -K, hi = a + K >= n ? n - 1 - a : K;
    int best = K + 1;
    for (int d = lo; d <= hi; ++d) {
        const int64_t o = c + d * stride;
        const int v = FIRST ? (__ldg(start + o + 1) > __ldg(start + o) ? 0 : K + 1) : static_cast<int>(__ldg(in + o));
        const int ad = d < 0 ? -d : d;
        const int m = v > ad ? v : ad;
        best = m < best ? m : best;
    }
    out[c] = static_cast<uint8_t>(best);
}

cudaError_t ring_distance_transform(RingGrid& v, uint8_t** dt, cudaStream_t stream) {
    const int K = std::min(v.rmax + 1, 254);
    uint8_t* tmp = nullptr;
    cudaError_t e = pool_alloc(dt, v.ncells, stream);
    if (e != cudaSuccess) return e;
    if ((e = cudaMallocAsync(&tmp, v.ncells, stream)) != cudaSuccess) return e;
    const unsigned b = nblocks(v.ncells, 256);
    k_ring_dt<0, true><<<b, 256, 0, stream>>>(v.start, nullptr, v, K, *dt);
    k_ring_dt<1, false><<<b, 256, 0, stream>>>(nullptr, *dt, v, K, tmp);
    k_ring_dt<2, false><<<b, 256, 0, stream>>>(nullptr, tmp, v, K, *dt);
    cudaFreeAsync(tmp, stream);
    v.dt = *dt;
    return cudaGetLastError();
}

// 30-bit Morton code of a point in the cube of side `ext` at `lo` (10 bits per axis)
__device__ __forceinline__ uint32_t spread10(uint32_t v) {
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000ffu;
    v = (v | (v << 8)) & 0x0300f00fu;
    v = (v | (v << 4)) & 0x030c30c3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

__global__ void k_morton(const double* __restrict__ p, int64_t n, int64_t block,
                         const unsigned long long* __restrict__ keys, unsigned long long* __restrict__ code,
                         int32_t* __restrict__ idx) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    double lo[3], ext = 0.0;
    for (int a = 0; a < 3; ++a) {
        lo[a] = from_key(keys[a]);
        ext = fmax(ext, from_key(keys[3 + a]) - lo[a]);
    }
    const double s = ext > 0.0 ? 1023.0 / ext : 0.0;
    uint32_t c = 0;
    for (int a = 0; a < 3; ++a) {
        const double q = (p[3 * i + a] - lo[a]) * s;
        const uint32_t v = q > 0.0 ? (q < 1023.0 ? static_cast<uint32_t>(q) : 1023u) : 0u;
        c |= spread10(v) << a;
    }
    code[i] = (static_cast<unsigned long long>(i / block) << 30) | c;
    idx[i] = static_cast<int32_t>(i);
}

// ring cells of d_max / LK_RING_DIV for single dense grids; unset (0): d_max
// / 5, coarsened to the occupancy target (build_ring_grid)
double ring_divisor() {
    static double cached = -1.0;
    if (cached < 0.0) {
        const char* e = std::getenv("LK_RING_DIV");
        const double v = e ? std::atof(e) : 0.0;
        cached = v >= 1.0 && v <= 64.0 ? v : 0.0;
    }
    return cached;
}

// LK_RING_DT=0 disables the distance-transform shell skip (comparison runs)
bool ring_dt_enabled() {
    static int cached = -1;
    if (cached < 0) {
        const char* e = std::getenv("LK_RING_DT");
        cached = (e && e[0] == '0') ? 0 : 1;
    }
    return cached == 1;
}

// ---- batched build (K clouds concatenated) ---------------------------------
__device__ __forceinline__ int cloud_of(const int64_t* __restrict__ off, int K, int64_t i) {
    int lo = 0, hi = K;  // off[lo] <= i < off[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(off + mid) <= i) lo = mid;
        else hi = mid;
    }
    return lo;
}

// CTA per cloud: keys[6k..6k+2] = min, [6k+3..6k+5] = max
__global__ void k_ring_bbox_batched(const double* __restrict__ p, const int64_t* __restrict__ off,
                                    unsigned long long* __restrict__ keys) {
    const int k = blockIdx.x;
    unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0ull, 0ull, 0ull};
    for (int64_t i = off[k] + threadIdx.x; i < off[k + 1]; i += blockDim.x)
        for (int a = 0; a < 3; ++a) {
            const unsigned long long q = order_key(p[3 * i + a]);
            lo[a] = q < lo[a] ? q : lo[a];
            hi[a] = q > hi[a] ? q : hi[a];
        }
    for (int a = 0; a < 3; ++a) {
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long x = __shfl_xor_sync(0xffffffffu, lo[a], o);
            const unsigned long long y = __shfl_xor_sync(0xffffffffu, hi[a], o);
            lo[a] = x < lo[a] ? x : lo[a];
            hi[a] = y > hi[a] ? y : hi[a];
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(keys + 6 * k + a, lo[a]);
            atomicMax(keys + 6 * k + 3 + a, hi[a]);
        }
    }
}

__global__ void k_ring_count_batched(const double* __restrict__ p, int64_t n, const int64_t* __restrict__ off,
                                     int K, const RingGrid* __restrict__ views, const int64_t* __restrict__ cell_off,
                                     int64_t* __restrict__ cell_of, int32_t* __restrict__ counts) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int k = cloud_of(off, K, i);
    const RingGrid& rg = views[k];
    const int cx = ring_cell_axis(p[3 * i], rg.ox, rg.cell, rg.nx);
    const int cy = ring_cell_axis(p[3 * i + 1], rg.oy, rg.cell, rg.ny);
    const int cz = ring_cell_axis(p[3 * i + 2], rg.oz, rg.cell, rg.nz);
    const int64_t c = cell_off[k] + (static_cast<int64_t>(cx) * rg.ny + cy) * rg.nz + cz;
    cell_of[i] = c;
    atomicAdd(counts + c, 1);
}

__global__ void k_ring_scatter_batched(const double* __restrict__ p, int64_t n, const int64_t* __restrict__ off,
                                       int K, const RingGrid* __restrict__ views, const int32_t* __restrict__ start,
                                       const int64_t* __restrict__ cell_of, int32_t* __restrict__ cursor,
                                       float4* __restrict__ pts) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int k = cloud_of(off, K, i);
    const RingGrid& rg = views[k];
    const int64_t c = cell_of[i];
    const int32_t s = start[c] + atomicAdd(cursor + c, 1);
    pts[s] = make_float4(static_cast<float>((p[3 * i] - rg.ox) / rg.cell),
                         static_cast<float>((p[3 * i + 1] - rg.oy) / rg.cell),
                         static_cast<float>((p[3 * i + 2] - rg.oz) / rg.cell),
                         __int_as_float(static_cast<int>(i - off[k])));
}

}  // namespace

// Frame of one ring grid over a cloud with bounding box [lo, hi] answering
// radius d_max: ring cells of d_max / 6 (coarsened under max_cells), guard
// bands, and the reference window -- the EvalGrid at cell d_max when
// search_cell <= 0, else a SearchGrid of that cell length.
RingGrid ring_frame(const double* lo, const double* hi, double d_max, double search_cell, int64_t max_cells,
                    bool fast, double divisor) {
    RingGrid v{};
    if (search_cell <= 0.0) {
        // the reference's EvalGrid over the same cloud (registration.cpp:82-97)
        v.ecell = d_max;
        v.eox = lo[0] - d_max;
        v.eoy = lo[1] - d_max;
        v.eoz = lo[2] - d_max;
        v.enx = static_cast<int>(std::floor(((hi[0] - v.eox) + d_max) / d_max)) + 2;
        v.eny = static_cast<int>(std::floor(((hi[1] - v.eoy) + d_max) / d_max)) + 2;
        v.enz = static_cast<int>(std::floor(((hi[2] - v.eoz) + d_max) / d_max)) + 2;
        v.ewin = 1;
        v.ebounded = 1;
    } else {
        // SearchGrid (grid.cpp:26-30, 101-109): center 0, block radius ceil(d / cell)
        v.ecell = search_cell;
        v.eox = v.eoy = v.eoz = 0.0;
        v.ewin = static_cast<int>(std::ceil(d_max / search_cell));
        v.ebounded = 0;
    }
    double cell = d_max / divisor;
    int dims[3] = {1, 1, 1};
    int64_t nc = 1;
    for (int guard = 0; guard < 200; ++guard) {
        for (int a = 0; a < 3; ++a) dims[a] = static_cast<int>(std::floor((hi[a] - lo[a]) / cell)) + 1;
        nc = static_cast<int64_t>(dims[0]) * dims[1] * dims[2];
        if (nc <= max_cells) break;
        cell *= 1.25;
    }
    v.ox = lo[0];
    v.oy = lo[1];
    v.oz = lo[2];
    v.cell = cell;
    v.nx = dims[0];
    v.ny = dims[1];
    v.nz = dims[2];
    v.ncells = nc;
    v.rmax = static_cast<int>(std::ceil(d_max / cell)) + 2;
    // FP32 conversion error of a coordinate (cells), both sides, plus slack
    const double nmax = std::max(v.nx, std::max(v.ny, v.nz)) + v.rmax + 2.0;
    v.delta = static_cast<float>(2.0 * nmax * 5.9604644775390625e-8 + 1e-6);
    const double thr = (d_max / cell) * (d_max / cell);
    v.thr = static_cast<float>(thr);
    // |d2_fp32 - d2| <= 2 sqrt3 |d| delta + 3 delta^2 + 4 u d2 over |d| <= rmax cells; 4x margin
    const double R = v.rmax + 1.0;
    v.band = static_cast<float>(4.0 * (2.0 * 1.7320508 * R * v.delta + 3.0 * v.delta * v.delta +
                                       4.0 * 5.9604644775390625e-8 * R * R) + 1e-6);
    // FP64-only mode: an infinite band scans every shell within d_max and
    // decides every entry in FP64 (the tests' exhaustive reference path)
    if (!fast) v.band = 1e30f;
    return v;
}

void RingStorage::release() {
    pool_free(start, stream);
    pool_free(pts, stream);
    pool_free(pos4, stream);
    pool_free(dt, stream);
    start = nullptr;
    pts = nullptr;
    pos4 = nullptr;
    dt = nullptr;
    view = RingGrid{};
}

// A spatially coherent order of a cloud (Morton order of its own bounding
// cube, 10 bits per axis): consecutive entries of perm lie close together,
// and stay close under any rigid transform, so a warp walking queries in this
// order visits the same ring cells (shared loop trip counts, L1 reuse).
// spatial_order_blocks: the same inside each run of `block` consecutive
// points (perm[b * block ...] is block b's points in Morton order).
cudaError_t spatial_order_blocks(const double* d_pos, int64_t n, int64_t block, int32_t* d_perm,
                                 cudaStream_t stream) {
    if (n <= 0 || n > INT32_MAX || block <= 0) return cudaErrorInvalidValue;
    int end_bit = 30;
    for (int64_t nb = (n + block - 1) / block; nb > 1; nb = (nb + 1) / 2) ++end_bit;
    unsigned long long* keys = nullptr;
    unsigned long long *code = nullptr, *code_out = nullptr;
    int32_t* idx = nullptr;
    void* temp = nullptr;
    size_t temp_bytes = 0;
    cudaError_t e = cudaSuccess;
    auto done = [&](cudaError_t r) {
        cudaFreeAsync(keys, stream);
        cudaFreeAsync(code, stream);
        cudaFreeAsync(code_out, stream);
        cudaFreeAsync(idx, stream);
        if (temp) cudaFreeAsync(temp, stream);
        return r;
    };
    if ((e = cudaMallocAsync(&keys, 6 * sizeof(unsigned long long), stream)) != cudaSuccess) return done(e);
    if ((e = cudaMallocAsync(&code, n * sizeof(unsigned long long), stream)) != cudaSuccess) return done(e);
    if ((e = cudaMallocAsync(&code_out, n * sizeof(unsigned long long), stream)) != cudaSuccess) return done(e);
    if ((e = cudaMallocAsync(&idx, n * sizeof(int32_t), stream)) != cudaSuccess) return done(e);
    // min keys start at all-ones, max keys at zero
    if ((e = cudaMemsetAsync(keys, 0xff, 3 * sizeof(unsigned long long), stream)) != cudaSuccess) return done(e);
    if ((e = cudaMemsetAsync(keys + 3, 0, 3 * sizeof(unsigned long long), stream)) != cudaSuccess) return done(e);
    k_ring_bbox<<<std::min<unsigned>(nblocks(n, 256), 296), 256, 0, stream>>>(d_pos, n, keys);
    k_morton<<<nblocks(n, 256), 256, 0, stream>>>(d_pos, n, block, keys, code, idx);
    if ((e = cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, code, code_out, idx, d_perm, static_cast<int>(n), 0,
                                             end_bit, stream)) != cudaSuccess)
        return done(e);
    if ((e = cudaMallocAsync(&temp, temp_bytes > 0 ? temp_bytes : 1, stream)) != cudaSuccess) return done(e);
    if ((e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, code, code_out, idx, d_perm, static_cast<int>(n), 0,
                                             end_bit, stream)) != cudaSuccess)
        return done(e);
    return done(cudaGetLastError());
}

cudaError_t spatial_order(const double* d_pos, int64_t n, int32_t* d_perm, cudaStream_t stream) {
    return spatial_order_blocks(d_pos, n, n, d_perm, stream);
}

cudaError_t build_ring_grid(RingStorage& rs, const double* d_pos, int64_t n, double d_max, cudaStream_t stream,
                            bool fast) {
#define RG_TRY(x)                         \
    do {                                  \
        cudaError_t e_ = (x);             \
        if (e_ != cudaSuccess) return e_; \
    } while (0)
    rs.stream = stream;
    if (n <= 0 || n > INT32_MAX || !(d_max > 0.0)) return cudaErrorInvalidValue;
    unsigned long long* keys = nullptr;
    RG_TRY(cudaMallocAsync(&keys, 6 * sizeof(unsigned long long), stream));
    const unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull};
    RG_TRY(cudaMemcpyAsync(keys, init, sizeof(init), cudaMemcpyHostToDevice, stream));
    k_ring_bbox<<<std::min<unsigned>(nblocks(n, 256), 296), 256, 0, stream>>>(d_pos, n, keys);
    unsigned long long* hk = static_cast<unsigned long long*>(host_scratch(6 * sizeof(unsigned long long)));
    if (!hk) return cudaErrorMemoryAllocation;
    RG_TRY(cudaMemcpyAsync(hk, keys, 6 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream));
    RG_TRY(cudaStreamSynchronize(stream));
    cudaFreeAsync(keys, stream);
    double lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
        lo[a] = from_key(hk[a]);
        hi[a] = from_key(hk[3 + a]);
    }
    // at most 64 cells per point (and 2^28 overall)
    const int64_t cap = std::min<int64_t>(std::max<int64_t>(64 * n, 4096), int64_t(1) << 28);
    const double fixed_div = ring_divisor();
    RingGrid v = ring_frame(lo, hi, d_max, -1.0, cap, fast, fixed_div > 0.0 ? fixed_div : 5.0);
    int64_t nc = v.ncells;
    int32_t *cell_of = nullptr, *counts = nullptr;
    RG_TRY(cudaMallocAsync(&cell_of, n * sizeof(int32_t), stream));
    RG_TRY(cudaMallocAsync(&counts, nc * sizeof(int32_t), stream));
    RG_TRY(cudaMemsetAsync(counts, 0, nc * sizeof(int32_t), stream));
    k_ring_count<<<nblocks(n, 256), 256, 0, stream>>>(d_pos, n, v, cell_of, counts);
    if (fixed_div <= 0.0) {
        // The walk's cost is a fixed cost per (x, y) row plus a cost per
        // entry; sparse targets (few points per occupied cell) pay mostly
        // rows. Coarsen until a point's cell holds ~kRingOccupancy entries
        // (point-weighted mean, measured; surfaces scale it with the cell
        // area), never beyond d_max / 2.5. Measured on B200: the B2 frame
        // (13.7 at d_max / 5) runs 1.4x faster at d_max / 3 (43); the 2.4M
        // submap of config D (51 at d_max / 5) is left alone.
        constexpr double kRingOccupancy = 40.0;
        unsigned long long* d_occ = nullptr;
        RG_TRY(cudaMallocAsync(&d_occ, sizeof(unsigned long long), stream));
        RG_TRY(cudaMemsetAsync(d_occ, 0, sizeof(unsigned long long), stream));
        k_ring_occupancy<<<std::min<unsigned>(nblocks(n, 256), 592), 256, 0, stream>>>(cell_of, n, counts, d_occ);
        auto* h_occ = static_cast<unsigned long long*>(host_scratch(sizeof(unsigned long long)));
        if (!h_occ) return cudaErrorMemoryAllocation;
        RG_TRY(cudaMemcpyAsync(h_occ, d_occ, sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream));
        RG_TRY(cudaStreamSynchronize(stream));
        cudaFreeAsync(d_occ, stream);
        const double occ = static_cast<double>(*h_occ) / static_cast<double>(n);
        if (occ < kRingOccupancy) {
            const double div = std::max(2.5, (d_max / v.cell) / std::sqrt(kRingOccupancy / occ));
            if (d_max / v.cell - div > 0.25) {
                v = ring_frame(lo, hi, d_max, -1.0, cap, fast, div);
                if (v.ncells > nc) return cudaErrorInvalidValue;  // coarser never has more cells
                nc = v.ncells;
                RG_TRY(cudaMemsetAsync(counts, 0, nc * sizeof(int32_t), stream));
                k_ring_count<<<nblocks(n, 256), 256, 0, stream>>>(d_pos, n, v, cell_of, counts);
            }
        }
    }
    RG_TRY(pool_alloc(&rs.start, (nc + 1) * sizeof(int32_t), stream));
    RG_TRY(pool_alloc(&rs.pts, n * sizeof(float4), stream));
    RG_TRY(exclusive_scan(counts, nc, rs.start, stream));
    RG_TRY(cudaMemsetAsync(counts, 0, nc * sizeof(int32_t), stream));
    v.start = rs.start;
    k_ring_scatter<<<nblocks(n, 256), 256, 0, stream>>>(d_pos, n, v, cell_of, counts, rs.pts);
    RG_TRY(pool_alloc(&rs.pos4, n * sizeof(double4), stream));
    RG_TRY(make_records(d_pos, nullptr, n, rs.pos4, nullptr, stream));
    cudaFreeAsync(cell_of, stream);
    cudaFreeAsync(counts, stream);
    if (ring_dt_enabled()) RG_TRY(ring_distance_transform(v, &rs.dt, stream));
    v.pts = rs.pts;
    v.pos4 = rs.pos4;
    v.npoints = n;
    rs.view = v;
    return cudaGetLastError();
#undef RG_TRY
}

void RingBatch::release() {
    pool_free(start, stream);
    pool_free(pts, stream);
    pool_free(pos4, stream);
    pool_free(d_views, stream);
    start = nullptr;
    pts = nullptr;
    pos4 = nullptr;
    d_views = nullptr;
}

cudaError_t build_ring_grids(RingBatch& rb, const double* d_pos, const int64_t* h_offsets, int32_t K,
                             const double* h_dmax, const double* h_cell, cudaStream_t stream) {
#define RG_TRY(x)                         \
    do {                                  \
        cudaError_t e_ = (x);             \
        if (e_ != cudaSuccess) return e_; \
    } while (0)
    rb.stream = stream;
    if (K <= 0) return cudaErrorInvalidValue;
    const int64_t n = h_offsets[K];
    if (n <= 0 || n > INT32_MAX) return cudaErrorInvalidValue;
    for (int k = 0; k < K; ++k)
        if (h_offsets[k + 1] <= h_offsets[k] || !(h_dmax[k] > 0.0)) return cudaErrorInvalidValue;
    int64_t* d_off = nullptr;
    unsigned long long* keys = nullptr;
    RG_TRY(cudaMallocAsync(&d_off, (K + 1) * sizeof(int64_t), stream));
    RG_TRY(cudaMallocAsync(&keys, 6 * static_cast<size_t>(K) * sizeof(unsigned long long), stream));
    std::vector<unsigned long long> hk(6 * static_cast<size_t>(K));
    for (int k = 0; k < K; ++k)
        for (int a = 0; a < 3; ++a) {
            hk[6 * k + a] = ~0ull;
            hk[6 * k + 3 + a] = 0ull;
        }
    RG_TRY(cudaMemcpyAsync(d_off, h_offsets, (K + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, stream));
    RG_TRY(cudaMemcpyAsync(keys, hk.data(), hk.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice, stream));
    k_ring_bbox_batched<<<K, 256, 0, stream>>>(d_pos, d_off, keys);
    RG_TRY(cudaMemcpyAsync(hk.data(), keys, hk.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream));
    RG_TRY(cudaStreamSynchronize(stream));
    cudaFreeAsync(keys, stream);
    std::vector<RingGrid> views(static_cast<size_t>(K));
    std::vector<int64_t> cell_off(static_cast<size_t>(K) + 1, 0);
    for (int k = 0; k < K; ++k) {
        double lo[3], hi[3];
        for (int a = 0; a < 3; ++a) {
            lo[a] = from_key(hk[6 * k + a]);
            hi[a] = from_key(hk[6 * k + 3 + a]);
        }
        // the dense CSR is sized to the cloud: at most 16 cells per point
        const int64_t npk = h_offsets[k + 1] - h_offsets[k];
        const int64_t cap = std::min<int64_t>(std::max<int64_t>(16 * npk, 4096), int64_t(1) << 24);
        views[k] = ring_frame(lo, hi, h_dmax[k], h_cell ? h_cell[k] : -1.0, cap, true, 6.0);
        cell_off[k + 1] = cell_off[k] + views[k].ncells;
    }
    const int64_t nc = cell_off[K];
    if (nc > INT32_MAX) return cudaErrorInvalidValue;
    int64_t *d_cell_off = nullptr, *cell_of = nullptr;
    int32_t* counts = nullptr;
    RG_TRY(cudaMallocAsync(&d_cell_off, (K + 1) * sizeof(int64_t), stream));
    RG_TRY(cudaMallocAsync(&cell_of, n * sizeof(int64_t), stream));
    RG_TRY(cudaMallocAsync(&counts, nc * sizeof(int32_t), stream));
    RG_TRY(pool_alloc(&rb.start, (nc + 1) * sizeof(int32_t), stream));
    RG_TRY(pool_alloc(&rb.pts, n * sizeof(float4), stream));
    RG_TRY(pool_alloc(&rb.pos4, n * sizeof(double4), stream));
    RG_TRY(pool_alloc(&rb.d_views, K * sizeof(RingGrid), stream));
    for (int k = 0; k < K; ++k) {
        views[k].start = rb.start + cell_off[k];
        views[k].pts = rb.pts;
        views[k].pos4 = rb.pos4 + h_offsets[k];
        views[k].npoints = h_offsets[k + 1] - h_offsets[k];
    }
    RG_TRY(cudaMemcpyAsync(d_cell_off, cell_off.data(), (K + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, stream));
    RG_TRY(cudaMemcpyAsync(rb.d_views, views.data(), K * sizeof(RingGrid), cudaMemcpyHostToDevice, stream));
    RG_TRY(cudaMemsetAsync(counts, 0, nc * sizeof(int32_t), stream));
    k_ring_count_batched<<<nblocks(n, 256), 256, 0, stream>>>(d_pos, n, d_off, K, rb.d_views, d_cell_off, cell_of,
                                                              counts);
    RG_TRY(exclusive_scan(counts, nc, rb.start, stream));
    RG_TRY(cudaMemsetAsync(counts, 0, nc * sizeof(int32_t), stream));
    k_ring_scatter_batched<<<nblocks(n, 256), 256, 0, stream>>>(d_pos, n, d_off, K, rb.d_views, rb.start, cell_of,
                                                                counts, rb.pts);
    RG_TRY(make_records(d_pos, nullptr, n, rb.pos4, nullptr, stream));
    // the host vectors above are read by async copies: finish before returning
    RG_TRY(cudaStreamSynchronize(stream));
    cudaFreeAsync(d_off, stream);
    cudaFreeAsync(d_cell_off, stream);
    cudaFreeAsync(cell_of, stream);
    cudaFreeAsync(counts, stream);
    return cudaGetLastError();
#undef RG_TRY
}

}  // namespace lkk
