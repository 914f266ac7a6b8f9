// lk_grid.cu -- device construction of the target cell grid (K6 in SURVEY.md 2.2).
//
// EvalGrid (proj/src/registration.cpp:80-148) and the SearchGrid cell
// convention (proj/src/grid.cpp:26-66) built on the device as a dense CSR:
// bbox / cell-bounds reduction -> per-point cell -> count -> exclusive scan ->
// scatter -> per-cell sort by original index (the reference's CSR order) ->
// slot payload gather -> occupancy dilation.
#include <algorithm>
#include <cmath>
#include <cstdint>

#include <mutex>
#include <unordered_map>
#include <cub/device/device_scan.cuh>
#include <vector>

#include "lk_kernels.cuh"

namespace lkk {

namespace {

__global__ void k_bbox(const double* __restrict__ pos, int64_t n, double* __restrict__ out6) {
    __shared__ double s_lo[3][32], s_hi[3][32];
    double lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
        lo[a] = pos[a];
        hi[a] = pos[a];
    }
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        for (int a = 0; a < 3; ++a) {
            double v = pos[3 * i + a];
            lo[a] = v < lo[a] ? v : lo[a];
            hi[a] = hi[a] < v ? v : hi[a];
        }
    }
    for (int a = 0; a < 3; ++a) {
        for (int o = 16; o > 0; o >>= 1) {
            double l = __shfl_xor_sync(0xffffffffu, lo[a], o);
            double h = __shfl_xor_sync(0xffffffffu, hi[a], o);
            lo[a] = l < lo[a] ? l : lo[a];
            hi[a] = hi[a] < h ? h : hi[a];
        }
    }
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (lane == 0)
        for (int a = 0; a < 3; ++a) {
            s_lo[a][warp] = lo[a];
            s_hi[a][warp] = hi[a];
        }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int a = 0; a < 3; ++a) {
            double l = s_lo[a][0], h = s_hi[a][0];
            for (int w = 1; w < nw; ++w) {
                l = s_lo[a][w] < l ? s_lo[a][w] : l;
                h = h < s_hi[a][w] ? s_hi[a][w] : h;
            }
            out6[a] = l;
            out6[3 + a] = h;
        }
    }
}

__device__ __forceinline__ int floor_cell(double q) {
    double f = floor(q);
    if (!(f >= -2147483648.0 && f < 2147483648.0)) return INT32_MIN;
    return static_cast<int>(f);
}

// SearchGrid cells of every point: min / max over floor((p - 0) / cell)
__global__ void k_cell_bounds(const double* __restrict__ pos, int64_t n, double cell, int* __restrict__ out6) {
    __shared__ int s[6];
    if (threadIdx.x < 3) {
        s[threadIdx.x] = INT32_MAX;
        s[3 + threadIdx.x] = INT32_MIN;
    }
    __syncthreads();
    int lo[3] = {INT32_MAX, INT32_MAX, INT32_MAX}, hi[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        for (int a = 0; a < 3; ++a) {
            int c = floor_cell((pos[3 * i + a] - 0.0) / cell);
            lo[a] = min(lo[a], c);
            hi[a] = max(hi[a], c);
        }
    }
    for (int a = 0; a < 3; ++a) {
        atomicMin(&s[a], lo[a]);
        atomicMax(&s[3 + a], hi[a]);
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        atomicMin(&out6[threadIdx.x], s[threadIdx.x]);
        atomicMax(&out6[3 + threadIdx.x], s[3 + threadIdx.x]);
    }
}

__global__ void k_cell_of(const double* __restrict__ pos, int64_t n, GridView g, int32_t* __restrict__ cell_of,
                          int32_t* __restrict__ counts) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int kx = floor_cell((pos[3 * i + 0] - g.ox) / g.cell) - g.offx;
    int ky = floor_cell((pos[3 * i + 1] - g.oy) / g.cell) - g.offy;
    int kz = floor_cell((pos[3 * i + 2] - g.oz) / g.cell) - g.offz;
    int32_t c = (kx * g.ny + ky) * g.nz + kz;
    cell_of[i] = c;
    atomicAdd(&counts[c], 1);
}

__global__ void k_scatter(const int32_t* __restrict__ cell_of, int64_t n, const int32_t* __restrict__ start,
                          int32_t* __restrict__ cursor, int32_t* __restrict__ index) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t c = cell_of[i];
    int32_t slot = start[c] + atomicAdd(&cursor[c], 1);
    index[slot] = static_cast<int32_t>(i);
}

// Restores the reference's ascending-index order within every cell.
// Warp per cell: slots ascending by original index. Indices are distinct, so
// each value's rank (how many values of the cell are smaller) is its slot.
// Cells of up to 32 * kSortQ points are ranked in registers; larger cells
// (not seen at the reference's densities) are insertion-sorted by lane 0.
constexpr int kSortQ = 16;
__global__ void __launch_bounds__(256) k_sort_cells(const int32_t* __restrict__ start, int64_t ncells,
                                                    int32_t* __restrict__ index) {
    const int64_t c = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (c >= ncells) return;
    const int32_t s0 = start[c], s1 = start[c + 1];
    const int k = s1 - s0;
    if (k <= 1) return;
    if (k <= 32 * kSortQ) {
        const int q_used = (k + 31) >> 5;
        int32_t v[kSortQ], rank[kSortQ];
#pragma unroll
        for (int q = 0; q < kSortQ; ++q) {
            const int e = 32 * q + lane;
            v[q] = (q < q_used && e < k) ? index[s0 + e] : INT32_MAX;
            rank[q] = 0;
        }
#pragma unroll
        for (int q2 = 0; q2 < kSortQ; ++q2) {
            if (q2 >= q_used) break;
            for (int t = 0; t < 32; ++t) {
                const int32_t u = __shfl_sync(0xffffffffu, v[q2], t);
#pragma unroll
                for (int q = 0; q < kSortQ; ++q) rank[q] += (q < q_used && u < v[q]) ? 1 : 0;
            }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < kSortQ; ++q) {
            const int e = 32 * q + lane;
            if (q < q_used && e < k) index[s0 + rank[q]] = v[q];
        }
        return;
    }
    if (lane == 0) {
        for (int32_t a = s0 + 1; a < s1; ++a) {
            int32_t val = index[a];
            int32_t b = a - 1;
            while (b >= s0 && index[b] > val) {
                index[b + 1] = index[b];
                --b;
            }
            index[b + 1] = val;
        }
    }
}

__global__ void k_gather_slots(const int32_t* __restrict__ index, int64_t n, const double* __restrict__ pos,
                               const double* __restrict__ nrm, double* __restrict__ slot_pos,
                               double* __restrict__ slot_nrm) {
    int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= n) return;
    int64_t i = index[s];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        slot_pos[3 * s + a] = pos[3 * i + a];
        slot_nrm[3 * s + a] = nrm ? nrm[3 * i + a] : 0.0;
    }
}

__global__ void k_dilate(const int32_t* __restrict__ cell_of, int64_t n, GridView g, uint8_t* __restrict__ near) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t c = cell_of[i];
    int kz = c % g.nz;
    int ky = (c / g.nz) % g.ny;
    int kx = c / (g.nz * g.ny);
    int r = g.radius;
    for (int x = max(kx - r, 0); x <= min(kx + r, g.nx - 1); ++x)
        for (int y = max(ky - r, 0); y <= min(ky + r, g.ny - 1); ++y)
            for (int z = max(kz - r, 0); z <= min(kz + r, g.nz - 1); ++z) near[(x * g.ny + y) * g.nz + z] = 1;
}

__device__ __forceinline__ void cell_coords(int64_t c, const GridView& g, int& kx, int& ky, int& kz) {
    kz = static_cast<int>(c % g.nz);
    ky = static_cast<int>((c / g.nz) % g.ny);
    kx = static_cast<int>(c / (static_cast<int64_t>(g.nz) * g.ny));
}

// points in the 3x3x3 block of every cell (rows are contiguous in z)
__global__ void k_block_count(const int32_t* __restrict__ start, int64_t ncells, GridView g,
                              int32_t* __restrict__ counts) {
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= ncells) return;
    int kx, ky, kz;
    cell_coords(c, g, kx, ky, kz);
    const int z0 = max(kz - 1, 0), z1 = min(kz + 1, g.nz - 1);
    int32_t n = 0;
    for (int x = max(kx - 1, 0); x <= min(kx + 1, g.nx - 1); ++x)
        for (int y = max(ky - 1, 0); y <= min(ky + 1, g.ny - 1); ++y) {
            const int64_t row = (static_cast<int64_t>(x) * g.ny + y) * g.nz;
            n += start[row + z1 + 1] - start[row + z0];
        }
    counts[c] = n;
}

__global__ void k_block_fill(const int32_t* __restrict__ start, const int32_t* __restrict__ index,
                             const double* __restrict__ slot_pos, const int32_t* __restrict__ offsets, int64_t ncells,
                             GridView g, int2* __restrict__ info, double4* __restrict__ pts,
                             float4* __restrict__ pts32) {
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= ncells) return;
    int kx, ky, kz;
    cell_coords(c, g, kx, ky, kz);
    const int z0 = max(kz - 1, 0), z1 = min(kz + 1, g.nz - 1);
    const int32_t off0 = offsets[c];
    int32_t off = off0;
    for (int x = max(kx - 1, 0); x <= min(kx + 1, g.nx - 1); ++x)
        for (int y = max(ky - 1, 0); y <= min(ky + 1, g.ny - 1); ++y) {
            const int64_t row = (static_cast<int64_t>(x) * g.ny + y) * g.nz;
            for (int32_t s = start[row + z0]; s < start[row + z1 + 1]; ++s) {
                const double px = slot_pos[3 * s], py = slot_pos[3 * s + 1], pz = slot_pos[3 * s + 2];
                pts[off] = make_double4(px, py, pz, static_cast<double>(index[s]));
                // local cell coordinates for the FP32 guard-band scan
                pts32[off] = make_float4(static_cast<float>((px - g.ox) / g.cell - g.offx),
                                         static_cast<float>((py - g.oy) / g.cell - g.offy),
                                         static_cast<float>((pz - g.oz) / g.cell - g.offz),
                                         __int_as_float(index[s]));
                ++off;
            }
        }
    info[c] = make_int2(off0, off - off0);
}

// ---- fine lists ----------------------------------------------------------
// Fine lists, warp per coarse cell C and its 8 half-size cells. The
// candidates of a fine box are the entries of C's 3x3x3 block list within
// fine_dmax of the box (+ a relative 1e-9 and an absolute 1e-12 margin) --
// every point the reference's window can hold within d_max of a query in
// the box. They are then Voronoi-pruned: entry j is dropped when some entry k
// is strictly closer than j to EVERY point of the (slightly expanded) box, so
// j can never be a query's nearest neighbour there (a dominating k is itself
// within d_max whenever j is; the resolve pass checks the reference window and
// falls back to the exact coarse scan when the winner lies outside it).
// |x-j|^2 - |x-k|^2 is separable per axis, so its minimum over the box is the
// sum of per-axis minima over the two faces; the margin (1e-9 fcell^2) dwarfs
// FP64 rounding of d2, so the reference's computed d2 orders k before j too.
// Storage: the 8 fine lists of C are packed from 8 * (C's block-list offset),
// which bounds them (each block entry is listed at most once per fine cell),
// so one pass writes them with no count pass, scan or host round trip.
constexpr int kFineWarps = 4;
constexpr int kFineCap = 256;

__device__ __forceinline__ bool box_within(double px, double py, double pz, const double* lo, double h, double r2) {
    const double dx = fmax(0.0, fmax(lo[0] - px, px - (lo[0] + h)));
    const double dy = fmax(0.0, fmax(lo[1] - py, py - (lo[1] + h)));
    const double dz = fmax(0.0, fmax(lo[2] - pz, pz - (lo[2] + h)));
    return (dx * dx + dy * dy) + dz * dz <= r2;
}

__global__ void __launch_bounds__(32 * kFineWarps) k_fine_build(GridView g, int64_t ncells, double r2,
                                                                 int2* __restrict__ info, float4* __restrict__ out) {
    __shared__ int32_t s_cand[kFineWarps][kFineCap];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t c = blockIdx.x * static_cast<int64_t>(kFineWarps) + warp;
    if (c >= ncells) return;
    const int2 bi = __ldg(g.block_info + c);
    if (bi.y == 0) return;  // info stays (0, 0)
    const int ix = static_cast<int>(c / (static_cast<int64_t>(g.ny) * g.nz));
    const int iy = static_cast<int>((c / g.nz) % g.ny);
    const int iz = static_cast<int>(c % g.nz);
    const double mexp = 1e-7 * g.fcell;
    const double hexp = g.fcell + 2 * mexp;
    const double margin = 1e-9 * g.fcell * g.fcell;
    int32_t* cand = s_cand[warp];
    int32_t w = 8 * bi.x;  // next free entry of C's fine storage
    for (int sub = 0; sub < 8; ++sub) {
        const int fx = 2 * ix + (sub >> 2), fy = 2 * iy + ((sub >> 1) & 1), fz = 2 * iz + (sub & 1);
        const int64_t fc = (static_cast<int64_t>(fx) * g.fny + fy) * g.fnz + fz;
        const double lo[3] = {g.ox + (fx + 2 * g.offx) * g.fcell, g.oy + (fy + 2 * g.offy) * g.fcell,
                              g.oz + (fz + 2 * g.offz) * g.fcell};
        const double le[3] = {lo[0] - mexp, lo[1] - mexp, lo[2] - mexp};
        // candidates within fine_dmax of the box
        int L = 0;
        for (int32_t b = 0; b < bi.y; b += 32) {
            const int32_t e = b + lane;
            bool in = false;
            if (e < bi.y) {
                const double4 P = g.block_pts[bi.x + e];
                in = box_within(P.x, P.y, P.z, lo, g.fcell, r2);
            }
            const unsigned m = __ballot_sync(0xffffffffu, in);
            const int at = L + __popc(m & ((1u << lane) - 1u));
            if (in && at < kFineCap) cand[at] = bi.x + e;
            L += __popc(m);
        }
        __syncwarp();
        if (L > kFineCap) {
            // (not seen at the reference's densities) no pruning: keep every candidate
            const int32_t w0 = w;
            for (int32_t b = 0; b < bi.y; b += 32) {
                const int32_t e = b + lane;
                bool in = false;
                double4 P = make_double4(0, 0, 0, 0);
                if (e < bi.y) {
                    P = g.block_pts[bi.x + e];
                    in = box_within(P.x, P.y, P.z, lo, g.fcell, r2);
                }
                const unsigned m = __ballot_sync(0xffffffffu, in);
                if (in)
                    out[w + __popc(m & ((1u << lane) - 1u))] =
                        make_float4(static_cast<float>((P.x - g.ox) / g.fcell - 2 * g.offx),
                                    static_cast<float>((P.y - g.oy) / g.fcell - 2 * g.offy),
                                    static_cast<float>((P.z - g.oz) / g.fcell - 2 * g.offz),
                                    __int_as_float(static_cast<int32_t>(P.w)));
                w += __popc(m);
            }
            if (lane == 0) info[fc] = make_int2(w0, w - w0);
            __syncwarp();
            continue;
        }
        // dominance pruning, lane-parallel over the candidates
        int K = 0;
        const int32_t w0 = w;
        for (int a0 = 0; a0 < L; a0 += 32) {
            const int a = a0 + lane;
            bool keep = false;
            double4 J = make_double4(0, 0, 0, 0);
            if (a < L) {
                J = g.block_pts[cand[a]];
                keep = true;
                for (int k = 0; k < L && keep; ++k) {
                    if (k == a) continue;
                    const double4 Q = g.block_pts[cand[k]];
                    const double jv[3] = {J.x, J.y, J.z}, kv[3] = {Q.x, Q.y, Q.z};
                    double fmin = 0.0;
#pragma unroll
                    for (int ax = 0; ax < 3; ++ax) {
                        const double c0 = le[ax], c1 = le[ax] + hexp;
                        const double f0 = (c0 - jv[ax]) * (c0 - jv[ax]) - (c0 - kv[ax]) * (c0 - kv[ax]);
                        const double f1 = (c1 - jv[ax]) * (c1 - jv[ax]) - (c1 - kv[ax]) * (c1 - kv[ax]);
                        fmin += f0 < f1 ? f0 : f1;
                    }
                    if (fmin > margin) keep = false;
                }
            }
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep)
                out[w0 + K + __popc(m & ((1u << lane) - 1u))] =
                    make_float4(static_cast<float>((J.x - g.ox) / g.fcell - 2 * g.offx),
                                static_cast<float>((J.y - g.oy) / g.fcell - 2 * g.offy),
                                static_cast<float>((J.z - g.oz) / g.fcell - 2 * g.offz),
                                __int_as_float(static_cast<int32_t>(J.w)));
            K += __popc(m);
        }
        if (lane == 0) info[fc] = make_int2(w0, K);
        w += K;
        __syncwarp();
    }
}

__global__ void k_to_float4(const double* __restrict__ pos, int64_t n, float4* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n)
        out[i] = make_float4(static_cast<float>(pos[3 * i]), static_cast<float>(pos[3 * i + 1]),
                             static_cast<float>(pos[3 * i + 2]), 0.0f);
}

__global__ void k_copy_normals(const double* __restrict__ nrm, int64_t n, double* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < 3 * n) out[i] = nrm ? nrm[i] : 0.0;
}

inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

// exclusive scan of n int32 into out[0..n] (out[n] = total)
// out[0..n] = exclusive prefix sums of in[0..n-1], out[n] = the total: one
// single-pass (decoupled look-back) inclusive scan into out + 1
cudaError_t exclusive_scan(const int32_t* in, int64_t n, int32_t* out, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(int32_t), stream);
    if (e != cudaSuccess || n <= 0) return e;
    if (n > INT32_MAX) return cudaErrorInvalidValue;
    size_t temp_bytes = 0;
    e = cub::DeviceScan::InclusiveSum(nullptr, temp_bytes, in, out + 1, static_cast<int>(n), stream);
    if (e != cudaSuccess) return e;
    void* temp = nullptr;
    e = cudaMallocAsync(&temp, temp_bytes > 0 ? temp_bytes : 1, stream);
    if (e != cudaSuccess) return e;
    e = cub::DeviceScan::InclusiveSum(temp, temp_bytes, in, out + 1, static_cast<int>(n), stream);
    cudaFreeAsync(temp, stream);
    return e != cudaSuccess ? e : cudaGetLastError();
}

size_t scan_temp_bytes(int64_t n) {
    size_t temp_bytes = 0;
    if (n > 0 && n <= INT32_MAX)
        cub::DeviceScan::InclusiveSum(nullptr, temp_bytes, static_cast<const int32_t*>(nullptr),
                                      static_cast<int32_t*>(nullptr), static_cast<int>(n));
    return temp_bytes > 0 ? temp_bytes : 1;
}

cudaError_t exclusive_scan(const int32_t* in, int64_t n, int32_t* out, cudaStream_t stream, void* temp,
                           size_t temp_bytes, bool zero_first) {
    if (zero_first) {
        const cudaError_t e = cudaMemsetAsync(out, 0, sizeof(int32_t), stream);
        if (e != cudaSuccess) return e;
    }
    if (n <= 0) return cudaSuccess;
    if (n > INT32_MAX || temp_bytes < scan_temp_bytes(n)) return cudaErrorInvalidValue;
    const cudaError_t e = cub::DeviceScan::InclusiveSum(temp, temp_bytes, in, out + 1, static_cast<int>(n), stream);
    return e != cudaSuccess ? e : cudaGetLastError();
}

struct Scratch::Entry {
    std::mutex mu;
    char* p = nullptr;
    size_t cap = 0;
};

Scratch::Scratch(cudaStream_t s, size_t bytes) {
    static std::mutex g_mu;
    static std::unordered_map<cudaStream_t, Entry*> g_entries;
    {
        std::lock_guard<std::mutex> lock(g_mu);
        Entry*& e = g_entries[s];
        if (!e) e = new Entry();  // kept for the process (streams are pooled)
        e_ = e;
    }
    e_->mu.lock();
    if (e_->cap < bytes) {
        // the old buffer's last users are ahead on s: a stream-ordered free
        if (e_->p) cudaFreeAsync(e_->p, s);
        e_->p = nullptr;
        e_->cap = 0;
        const size_t cap = bytes + bytes / 4;
        err_ = cudaMallocAsync(reinterpret_cast<void**>(&e_->p), cap, s);
        if (err_ == cudaSuccess) e_->cap = cap;
        else e_->p = nullptr;
    }
    base_ = e_->p;
    cap_ = e_->cap;
}

Scratch::~Scratch() { e_->mu.unlock(); }

void GridStorage::release() {
    pool_free(start, stream);
    pool_free(index, stream);
    pool_free(slot_pos, stream);
    pool_free(slot_nrm, stream);
    pool_free(near, stream);
    pool_free(block_info, stream);
    pool_free(block_pts, stream);
    pool_free(nrm_orig, stream);
    pool_free(block_f32, stream);
    pool_free(pos_orig, stream);
    pool_free(pos4_orig, stream);
    pool_free(nrm32_orig, stream);
    pos4_orig = nullptr;
    nrm32_orig = nullptr;
    pool_free(fine_info, stream);
    pool_free(fine_pts, stream);
    fine_info = nullptr;
    fine_pts = nullptr;
    start = index = nullptr;
    slot_pos = slot_nrm = nullptr;
    near = nullptr;
    block_info = nullptr;
    block_pts = nullptr;
    nrm_orig = nullptr;
    block_f32 = nullptr;
    pos_orig = nullptr;
}

#define LK_TRY(x)                                \
    do {                                         \
        cudaError_t e_ = (x);                    \
        if (e_ != cudaSuccess) return e_;        \
    } while (0)

cudaError_t build_grid(GridStorage& g, int kind, const double* d_pos, const double* d_nrm, int64_t n, double cell,
                       double d_max, cudaStream_t stream, bool with_blocks) {
    g.stream = stream;
    if (n <= 0 || n > INT32_MAX) return cudaErrorInvalidValue;
    GridView v{};
    v.kind = kind;
    v.cell = cell;
    if (kind == 0) {
        // proj/src/registration.cpp:82-97
        double* d_box = nullptr;
        LK_TRY(cudaMallocAsync(&d_box, 6 * sizeof(double), stream));
        k_bbox<<<1, 1024, 0, stream>>>(d_pos, n, d_box);
        double* box = static_cast<double*>(host_scratch(6 * sizeof(double)));
        if (!box) return cudaErrorMemoryAllocation;
        LK_TRY(cudaMemcpyAsync(box, d_box, 6 * sizeof(double), cudaMemcpyDeviceToHost, stream));
        LK_TRY(cudaStreamSynchronize(stream));
        cudaFreeAsync(d_box, stream);
        double origin[3];
        int dims[3];
        for (int a = 0; a < 3; ++a) {
            origin[a] = box[a] - cell;
            double extent = (box[3 + a] - origin[a]) + cell;
            dims[a] = static_cast<int>(std::floor(extent / cell)) + 2;
        }
        v.ox = origin[0];
        v.oy = origin[1];
        v.oz = origin[2];
        v.nx = dims[0];
        v.ny = dims[1];
        v.nz = dims[2];
        v.offx = v.offy = v.offz = 0;
        v.radius = 1;
    } else {
        // proj/src/grid.cpp:38-47 with center 0; dense over the occupied box + r
        int* d_b = nullptr;
        LK_TRY(cudaMallocAsync(&d_b, 6 * sizeof(int), stream));
        int init[6] = {INT32_MAX, INT32_MAX, INT32_MAX, INT32_MIN, INT32_MIN, INT32_MIN};
        LK_TRY(cudaMemcpyAsync(d_b, init, sizeof(init), cudaMemcpyHostToDevice, stream));
        k_cell_bounds<<<std::min<unsigned>(blocks_for(n, 256), 592), 256, 0, stream>>>(d_pos, n, cell, d_b);
        int* b = static_cast<int*>(host_scratch(6 * sizeof(int)));
        if (!b) return cudaErrorMemoryAllocation;
        LK_TRY(cudaMemcpyAsync(b, d_b, 6 * sizeof(int), cudaMemcpyDeviceToHost, stream));
        LK_TRY(cudaStreamSynchronize(stream));
        cudaFreeAsync(d_b, stream);
        int r = static_cast<int>(std::ceil(d_max / cell));
        v.ox = v.oy = v.oz = 0.0;
        v.radius = r;
        v.offx = b[0] - r;
        v.offy = b[1] - r;
        v.offz = b[2] - r;
        v.nx = b[3] - b[0] + 1 + 2 * r;
        v.ny = b[4] - b[1] + 1 + 2 * r;
        v.nz = b[5] - b[2] + 1 + 2 * r;
    }
    int64_t ncells = static_cast<int64_t>(v.nx) * v.ny * v.nz;
    if (ncells <= 0 || ncells > (int64_t)1 << 30) return cudaErrorInvalidValue;
    g.ncells = ncells;
    g.npoints = n;
    LK_TRY(pool_alloc(&g.start, (ncells + 1) * sizeof(int32_t), stream));
    LK_TRY(pool_alloc(&g.index, n * sizeof(int32_t), stream));
    LK_TRY(pool_alloc(&g.slot_pos, 3 * n * sizeof(double), stream));
    LK_TRY(pool_alloc(&g.slot_nrm, 3 * n * sizeof(double), stream));
    LK_TRY(pool_alloc(&g.near, ncells, stream));
    LK_TRY(pool_alloc(&g.nrm_orig, 3 * n * sizeof(double), stream));
    int32_t *d_cell_of = nullptr, *d_counts = nullptr;
    LK_TRY(cudaMallocAsync(&d_cell_of, n * sizeof(int32_t), stream));
    LK_TRY(cudaMallocAsync(&d_counts, ncells * sizeof(int32_t), stream));
    LK_TRY(cudaMemsetAsync(d_counts, 0, ncells * sizeof(int32_t), stream));
    LK_TRY(cudaMemsetAsync(g.near, 0, ncells, stream));
    k_cell_of<<<blocks_for(n, 256), 256, 0, stream>>>(d_pos, n, v, d_cell_of, d_counts);
    LK_TRY(exclusive_scan(d_counts, ncells, g.start, stream));
    LK_TRY(cudaMemsetAsync(d_counts, 0, ncells * sizeof(int32_t), stream));
    k_scatter<<<blocks_for(n, 256), 256, 0, stream>>>(d_cell_of, n, g.start, d_counts, g.index);
    k_sort_cells<<<blocks_for(ncells * 32, 256), 256, 0, stream>>>(g.start, ncells, g.index);
    k_gather_slots<<<blocks_for(n, 256), 256, 0, stream>>>(g.index, n, d_pos, d_nrm, g.slot_pos, g.slot_nrm);
    k_copy_normals<<<blocks_for(3 * n, 256), 256, 0, stream>>>(d_nrm, n, g.nrm_orig);
    if (kind == 0 || v.radius <= 2) {
        k_dilate<<<blocks_for(n, 128), 128, 0, stream>>>(d_cell_of, n, v, g.near);
    } else {
        LK_TRY(cudaMemsetAsync(g.near, 1, ncells, stream));  // wide blocks: no occupancy shortcut
    }
    // 3x3x3 block lists for radius-1 grids (27 entries per point at most)
    if (with_blocks && v.radius == 1 && 27 * n < INT32_MAX) {
        k_block_count<<<blocks_for(ncells, 256), 256, 0, stream>>>(g.start, ncells, v, d_counts);
        int32_t* d_off = nullptr;
        LK_TRY(cudaMallocAsync(&d_off, (ncells + 1) * sizeof(int32_t), stream));
        LK_TRY(exclusive_scan(d_counts, ncells, d_off, stream));
        int32_t* h_total = static_cast<int32_t*>(host_scratch(sizeof(int32_t)));
        if (!h_total) return cudaErrorMemoryAllocation;
        LK_TRY(cudaMemcpyAsync(h_total, d_off + ncells, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
        LK_TRY(cudaStreamSynchronize(stream));
        const int32_t total = *h_total;
        g.nblock = total;
        LK_TRY(pool_alloc(&g.block_info, ncells * sizeof(int2), stream));
        LK_TRY(pool_alloc(&g.block_pts, (total > 0 ? total : 1) * sizeof(double4), stream));
        LK_TRY(pool_alloc(&g.block_f32, (total > 0 ? total : 1) * sizeof(float4), stream));
        LK_TRY(pool_alloc(&g.pos_orig, 3 * n * sizeof(double), stream));
        LK_TRY(cudaMemcpyAsync(g.pos_orig, d_pos, 3 * n * sizeof(double), cudaMemcpyDeviceToDevice, stream));
        k_block_fill<<<blocks_for(ncells, 256), 256, 0, stream>>>(g.start, g.index, g.slot_pos, d_off, ncells, v,
                                                                  g.block_info, g.block_pts, g.block_f32);
        cudaFreeAsync(d_off, stream);
        // fine lists: half-size cells, points within d_max of each fine box
        v.fcell = cell / 2.0;
        v.fnx = 2 * v.nx;
        v.fny = 2 * v.ny;
        v.fnz = 2 * v.nz;
        v.fine_dmax = kind == 0 ? cell : d_max;
        const int64_t nfc = static_cast<int64_t>(v.fnx) * v.fny * v.fnz;
        if (nfc < (int64_t)1 << 30 && 8 * g.nblock < (int64_t)1 << 28) {
            const double r2 = v.fine_dmax * v.fine_dmax * (1.0 + 1e-9) + 1e-12;
            GridView bv = v;
            bv.block_info = g.block_info;
            bv.block_pts = g.block_pts;
            g.nfine = nfc;
            g.nfine_entries = 8 * g.nblock;
            LK_TRY(pool_alloc(&g.fine_info, nfc * sizeof(int2), stream));
            LK_TRY(pool_alloc(&g.fine_pts, (g.nfine_entries > 0 ? g.nfine_entries : 1) * sizeof(float4), stream));
            LK_TRY(cudaMemsetAsync(g.fine_info, 0, nfc * sizeof(int2), stream));
            const unsigned fb = static_cast<unsigned>((ncells + kFineWarps - 1) / kFineWarps);
            k_fine_build<<<fb, 32 * kFineWarps, 0, stream>>>(bv, ncells, r2, g.fine_info, g.fine_pts);
        }
    }
    LK_TRY(cudaGetLastError());
    cudaFreeAsync(d_cell_of, stream);
    cudaFreeAsync(d_counts, stream);
    v.start = g.start;
    v.index = g.index;
    v.slot_pos = g.slot_pos;
    v.slot_nrm = g.slot_nrm;
    v.near = g.near;
    v.block_info = g.block_info;
    v.block_pts = g.block_pts;
    v.nrm_orig = g.nrm_orig;
    v.block_f32 = g.block_f32;
    v.pos_orig = g.pos_orig;
    v.fine_info = g.fine_info;
    v.fine_pts = g.fine_pts;
    if (g.pos_orig && g.nrm_orig && n > 0) {
        LK_TRY(pool_alloc(&g.pos4_orig, n * sizeof(double4), stream));
        LK_TRY(pool_alloc(&g.nrm32_orig, n * sizeof(float4), stream));
        LK_TRY(make_records(g.pos_orig, g.nrm_orig, n, g.pos4_orig, g.nrm32_orig, stream));
    }
    v.pos4_orig = g.pos4_orig;
    v.nrm32_orig = g.nrm32_orig;
    v.n_points = g.npoints;
    v.n_cells = g.ncells;
    v.n_fine = g.nfine;
    v.n_fine_entries = g.fine_pts ? g.nfine_entries : 0;
    g.view = v;
    return cudaStreamSynchronize(stream);
}

__global__ void k_records(const double* __restrict__ pos, const double* __restrict__ nrm, int64_t n,
                          double4* __restrict__ pos4, float4* __restrict__ nrm32) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    if (pos4) pos4[i] = make_double4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], 0.0);
    if (nrm32)
        nrm32[i] = make_float4(static_cast<float>(nrm[3 * i]), static_cast<float>(nrm[3 * i + 1]),
                               static_cast<float>(nrm[3 * i + 2]), 0.0f);
}

cudaError_t make_records(const double* d_pos, const double* d_nrm, int64_t n, double4* d_pos4, float4* d_nrm32,
                         cudaStream_t stream) {
    if (n > 0) k_records<<<blocks_for(n, 256), 256, 0, stream>>>(d_pos, d_nrm, n, d_pos4, d_nrm32);
    return cudaGetLastError();
}

cudaError_t make_source32(const double* d_pos, int64_t n, float4* d_out, cudaStream_t stream) {
    if (n > 0) k_to_float4<<<blocks_for(n, 256), 256, 0, stream>>>(d_pos, n, d_out);
    return cudaGetLastError();
}

// Guard bands of the FP32 fast path:
// cell coordinates q = R' p + t' carry an absolute error below
// 8 * 2^-24 * (3 |p|max / cell + |t'| + n) cells; the bands below are an
// order of magnitude wider than that bound over the magnitudes admitted here.
void configure_fast_path(ScoreParams& sp, const GridView& g, double max_abs_source) {
    sp.fast = 0;
    if (!g.block_f32 || g.radius != 1) return;
    const double nmax = std::max(g.nx, std::max(g.ny, g.nz));
    const double pmax = max_abs_source / g.cell;
    if (nmax > 4096.0 || pmax > 4096.0) return;
    const double thr = (sp.d_max / g.cell) * (sp.d_max / g.cell);
    if (thr > 1.0) return;  // block radius 1 covers d_max only up to one cell
    sp.thr_cells = static_cast<float>(thr);
    sp.eps_cells = 2e-3f;
    sp.band_cells = 8e-3f;
    sp.pmax_cells = static_cast<float>(pmax);
    sp.nmax_cells = static_cast<float>(nmax);
    sp.fast = 1;
}

}  // namespace lkk
