// lk_verify.cu -- batched loop verification (north-star item 5, config E).
//
// For a batch of loop pairs (cloud_i = the earlier fragment Q with pose T_i,
// cloud_j = the later fragment P with pose T_j, measurement T mapping P into
// Q's frame) one pass computes, per pair:
//   * edge_info(Q, P, T_i, T_j, eps)         proj/src/line_process.cpp:11-33
//   * the overlap hit count of propose_loops  proj/src/fragments.cpp:61-109
//     (posed later points within r of the posed earlier cloud)
//   * evaluate_hypothesis(T, P, Q, SearchGrid(Q, cell), d_max, angle)
//                                             proj/src/registration.cpp:53-78
// and, for the pose graph's all-pairs loop search, propose_loops' overlap hit
// counts of every (later i, earlier j >= i + 2) fragment pair (propose_loops).
// Every nearest-neighbour question goes to a ring grid (lk_ring.cuh) that
// answers with the reference SearchGrid's window semantics; all 3K grids are
// built in one batched pass. The per-pair sums are the reference's own
// sequential sums in point order (one lane per accumulator), so the
// information matrix, the fitness and every count are bit-exact.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "lk_device_math.cuh"
#include "lk_kernels.cuh"
#include "lk_ring.cuh"

namespace lkk {

using namespace lkd;

namespace {

inline unsigned nblocks(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

__device__ __forceinline__ int pair_of(const int64_t* __restrict__ off, int K, int64_t i) {
    int lo = 0, hi = K;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(off + mid) <= i) lo = mid;
        else hi = mid;
    }
    return lo;
}

// out[i] = T_k p_i for the cloud k that holds point i (RigidTransform::operator*)
__global__ void k_pose_batched(const double* __restrict__ in, int64_t n, const int64_t* __restrict__ off, int K,
                               const double* __restrict__ T12, double* __restrict__ out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int k = pair_of(off, K, i);
    const double* T = T12 + 12 * k;
    const V3 y = xform(T, T + 9, ld3(in, i));
    out[3 * i] = y.x;
    out[3 * i + 1] = y.y;
    out[3 * i + 2] = y.z;
}

// edge_info queries: q in Q_k under T_i[k] against the grid over T_j[k] P_k
__global__ void k_verify_edge(const double* __restrict__ q, int64_t nq, const int64_t* __restrict__ offq, int K,
                              const double* __restrict__ Ti12, const RingGrid* __restrict__ grids, double eps2,
                              uint8_t* __restrict__ hit) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= nq) return;
    const int k = pair_of(offq, K, i);
    const double* T = Ti12 + 12 * k;
    const V3 y = xform(T, T + 9, ld3(q, i));
    hit[i] = ring_nn(grids[k], y, eps2) >= 0 ? 1 : 0;
}

// source-side queries: p in P_k posed by T_j[k] against the grid over
// T_i[k] Q_k (overlap), and T[k] p against the grid over Q_k with the normal
// gate (evaluate_hypothesis); addend = distance^2 with distance = sqrt(d2)
__global__ void k_verify_src(const double* __restrict__ p, const double* __restrict__ pn, int64_t np,
                             const int64_t* __restrict__ offp, int K, const double* __restrict__ qn,
                             const int64_t* __restrict__ offq, const double* __restrict__ Tj12,
                             const double* __restrict__ T12, const RingGrid* __restrict__ grids_o,
                             const RingGrid* __restrict__ grids_h, double r2, double d2_max, double cos_max,
                             uint8_t* __restrict__ overlap_hit, uint8_t* __restrict__ inlier,
                             double* __restrict__ addend) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= np) return;
    const int k = pair_of(offp, K, i);
    const V3 x = ld3(p, i);
    const double* Tj = Tj12 + 12 * k;
    overlap_hit[i] = ring_nn(grids_o[k], xform(Tj, Tj + 9, x), r2) >= 0 ? 1 : 0;
    const double* T = T12 + 12 * k;
    const V3 y = xform(T, T + 9, x);
    const RingGrid& gh = grids_h[k];
    const int32_t j = ring_nn(gh, y, d2_max);
    uint8_t ok = 0;
    double add = 0.0;
    if (j >= 0) {
        const V3 ns = ld3(pn, i);
        const V3 nt = ld3(qn, offq[k] + j);
        if (!is_zero(ns) && !is_zero(nt) && !(dot(rot(T, ns), nt) < cos_max)) {
            const double dist = sqrt(sqnorm(sub(ld4(gh.pos4, j), y)));
            add = dist * dist;
            ok = 1;
        }
    }
    inlier[i] = ok;
    addend[i] = add;
}

// One CTA of kSumThreads per pair. The points are staged kSumThreads at a
// time (coalesced): every hit computes its nine contributions -- the a^T a
// entries (0,0) (0,1) (0,2) (1,1) (1,2) (2,2) with a = -[q]x, then q.x, q.y,
// q.z -- into shared memory at its rank among the chunk's hits, and lane j < 9
// of warp 0 adds column j over them in point order: the reference's
// sequential sums (line_process.cpp:24-28). The same for the
// evaluate_hypothesis sq_sum over the source points (lane 9 of warp 1).
// Counts are popcounts of the hit ballots.
// out per pair: 10 doubles (9 edge sums, sq_sum) then 3 int64 at [10..12].
constexpr int kSumThreads = 256;
constexpr int kSumWarps = kSumThreads / 32;

__global__ void __launch_bounds__(kSumThreads) k_verify_sums(const double* __restrict__ q,
                                                             const int64_t* __restrict__ offq,
                                                             const uint8_t* __restrict__ edge_hit,
                                                             const int64_t* __restrict__ offp,
                                                             const uint8_t* __restrict__ overlap_hit,
                                                             const uint8_t* __restrict__ inlier,
                                                             const double* __restrict__ addend,
                                                             double* __restrict__ out) {
    // the chunk's hits compacted in point order (ballot prefix), so the
    // sequential sums read consecutive shared-memory words, loads ahead of
    // the dependent adds; lanes 0-8 of warp 0 run the nine edge sums, lane 9
    // of warp 1 the sq_sum, each over the staged chunk
    __shared__ double s_c[9][kSumThreads + 1];
    __shared__ double s_a[kSumThreads + 1];
    __shared__ int s_wq[kSumWarps + 1], s_wp[kSumWarps + 1];
    __shared__ unsigned long long s_cnt[3];
    const int k = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0ull;
    double acc = 0.0, sq = 0.0;
    unsigned long long n_edge = 0, n_over = 0, n_inl = 0;
    const int64_t q0 = offq[k], q1 = offq[k + 1], p0 = offp[k], p1 = offp[k + 1];
    const int64_t nq_c = (q1 - q0 + kSumThreads - 1) / kSumThreads, np_c = (p1 - p0 + kSumThreads - 1) / kSumThreads;
    const int64_t chunks = nq_c > np_c ? nq_c : np_c;
    const unsigned below = (1u << lane) - 1u;
    for (int64_t c = 0; c < chunks; ++c) {
        // edge_info chunk c of Q and evaluate_hypothesis chunk c of P, side by side
        const int64_t i = q0 + c * kSumThreads + threadIdx.x;
        const bool hit = i < q1 && edge_hit[i];
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        const int64_t ip = p0 + c * kSumThreads + threadIdx.x;
        const bool in = ip < p1;
        const unsigned mo = __ballot_sync(0xffffffffu, in && overlap_hit[ip]);
        const bool inl = in && inlier[ip];
        const unsigned mi = __ballot_sync(0xffffffffu, inl);
        if (lane == 0) {
            s_wq[warp + 1] = __popc(m);
            s_wp[warp + 1] = __popc(mi);
            n_edge += __popc(m);
            n_over += __popc(mo);
            n_inl += __popc(mi);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            s_wq[0] = 0;
            s_wp[0] = 0;
            for (int w = 0; w < kSumWarps; ++w) {
                s_wq[w + 1] += s_wq[w];
                s_wp[w + 1] += s_wp[w];
            }
        }
        __syncthreads();
        if (hit) {
            const int t = s_wq[warp] + __popc(m & below);
            const V3 v = ld3(q, i);
            const double a[3][3] = {{-0.0, v.z, -v.y}, {-v.z, -0.0, v.x}, {v.y, -v.x, -0.0}};
            s_c[0][t] = (a[0][0] * a[0][0] + a[1][0] * a[1][0]) + a[2][0] * a[2][0];
            s_c[1][t] = (a[0][0] * a[0][1] + a[1][0] * a[1][1]) + a[2][0] * a[2][1];
            s_c[2][t] = (a[0][0] * a[0][2] + a[1][0] * a[1][2]) + a[2][0] * a[2][2];
            s_c[3][t] = (a[0][1] * a[0][1] + a[1][1] * a[1][1]) + a[2][1] * a[2][1];
            s_c[4][t] = (a[0][1] * a[0][2] + a[1][1] * a[1][2]) + a[2][1] * a[2][2];
            s_c[5][t] = (a[0][2] * a[0][2] + a[1][2] * a[1][2]) + a[2][2] * a[2][2];
            s_c[6][t] = v.x;
            s_c[7][t] = v.y;
            s_c[8][t] = v.z;
        }
        if (inl) s_a[s_wp[warp] + __popc(mi & below)] = addend[ip];
        __syncthreads();
        if (warp == 0 && lane < 9) {
            const double* col = s_c[lane];
            const int cnt = s_wq[kSumWarps];
            int e = 0;
            for (; e + 4 <= cnt; e += 4) {
                const double x0 = col[e], x1 = col[e + 1], x2 = col[e + 2], x3 = col[e + 3];
                acc += x0;
                acc += x1;
                acc += x2;
                acc += x3;
            }
            for (; e < cnt; ++e) acc += col[e];
        }
        if (warp == 1 && lane == 9) {
            const int cnt = s_wp[kSumWarps];
            int e = 0;
            for (; e + 4 <= cnt; e += 4) {
                const double x0 = s_a[e], x1 = s_a[e + 1], x2 = s_a[e + 2], x3 = s_a[e + 3];
                sq += x0;
                sq += x1;
                sq += x2;
                sq += x3;
            }
            for (; e < cnt; ++e) sq += s_a[e];
        }
        __syncthreads();
    }
    if (lane == 0) {
        atomicAdd(&s_cnt[0], n_edge);
        atomicAdd(&s_cnt[1], n_over);
        atomicAdd(&s_cnt[2], n_inl);
    }
    __syncthreads();
    double* o = out + 16 * k;
    if (warp == 0 && lane < 9) o[lane] = acc;
    if (warp == 1 && lane == 9) o[9] = sq;
    if (threadIdx.x == 0) {
        long long* c = reinterpret_cast<long long*>(o);
        c[10] = static_cast<long long>(s_cnt[0]);
        c[11] = static_cast<long long>(s_cnt[1]);
        c[12] = static_cast<long long>(s_cnt[2]);
    }
}

// Zero-copy gather of many pinned host arrays into device slots: item k
// copies count[k] doubles from src[k] (a device-mapped pinned host pointer)
// to dst[k]; blockIdx.y picks the item, blockIdx.x strides inside it.
struct GatherItem {
    const double* src;
    double* dst;
    int64_t count;
};

__global__ void k_gather_host(const GatherItem* __restrict__ items) {
    const GatherItem it = items[blockIdx.y];
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < it.count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        it.dst[i] = it.src[i];
}

// LK_ZERO_COPY=0: always use one cudaMemcpyAsync per array
bool zero_copy_enabled() {
    static int cached = -1;
    if (cached < 0) {
        const char* e = std::getenv("LK_ZERO_COPY");
        cached = (e && e[0] == '0') ? 0 : 1;
    }
    return cached == 1;
}

// Device-mapped address of a page-locked host pointer, or null (pageable).
const double* mapped(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return a.type == cudaMemoryTypeHost ? static_cast<const double*>(a.devicePointer) : nullptr;
}

// propose_loops overlap (proj/src/fragments.cpp:86-100): pair k = (later i,
// earlier j); query q of pair k is point q - qoff[k] of posed fragment i,
// hit iff the reference SearchGrid over posed fragment j (cell = r) finds a
// point within r (nn_within existence). Warp-aggregated integer counts.
__global__ void k_propose_hits(const double* __restrict__ posed, const int64_t* __restrict__ foff,
                               const int32_t* __restrict__ pair_ij, const int64_t* __restrict__ qoff, int K,
                               const RingGrid* __restrict__ grids, double r2, unsigned long long* __restrict__ hits) {
    const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const bool live = q < qoff[K];
    int k = 0;
    bool hit = false;
    if (live) {
        k = pair_of(qoff, K, q);
        const int fi = pair_ij[2 * k], fj = pair_ij[2 * k + 1];
        const V3 y = ld3(posed, foff[fi] + (q - qoff[k]));
        hit = ring_nn(grids[fj], y, r2) >= 0;
    }
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (!m) return;
    // lanes of one pair (the common case) add once
    const int lane = threadIdx.x & 31;
    const unsigned same = __match_any_sync(0xffffffffu, live ? k : -1);
    const unsigned mine = m & same;
    if (hit && lane == __ffs(mine) - 1) atomicAdd(hits + k, static_cast<unsigned long long>(__popc(mine)));
}

}  // namespace

cudaError_t verify_batch(const VerifyInput& in, VerifyOutput* out, cudaStream_t stream) {
    // LK_TRACE: host timestamps of the phases (diagnostic)
    static const bool trace = std::getenv("LK_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!trace) return;
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        std::fprintf(stderr, "[lk verify] %-22s %8.3f ms\n", what, ms);
    };
    const int K = in.n_pairs;
    const int64_t nq = in.offq[K], np = in.offp[K];
    cudaError_t e = cudaSuccess;
    double *d_qpos = nullptr, *d_qn = nullptr, *d_ppos = nullptr, *d_pn = nullptr, *d_T = nullptr,
           *d_grid_pts = nullptr, *d_addend = nullptr, *d_out = nullptr;
    int64_t *d_offq = nullptr, *d_offp = nullptr;
    uint8_t* d_flags = nullptr;
    RingBatch rb;
    auto cleanup = [&] {
        rb.release();
        for (void* p : {(void*)d_qpos, (void*)d_qn, (void*)d_ppos, (void*)d_pn, (void*)d_T, (void*)d_grid_pts,
                        (void*)d_addend, (void*)d_out, (void*)d_offq, (void*)d_offp, (void*)d_flags})
            pool_free(p, stream);
    };
#define VF_TRY(x)               \
    do {                        \
        e = (x);                \
        if (e != cudaSuccess) { \
            cleanup();          \
            return e;           \
        }                       \
    } while (0)
    VF_TRY(pool_alloc(&d_qpos, 3 * nq * sizeof(double), stream));
    VF_TRY(pool_alloc(&d_ppos, 3 * np * sizeof(double), stream));
    VF_TRY(pool_alloc(&d_offq, (K + 1) * sizeof(int64_t), stream));
    VF_TRY(pool_alloc(&d_offp, (K + 1) * sizeof(int64_t), stream));
    VF_TRY(pool_alloc(&d_T, 3 * 12 * K * sizeof(double), stream));
    // each cloud straight from the caller's buffer into its slot (pinned
    // buffers go at full PCIe rate; no host-side packing)
    std::vector<void*> dsts, srcs;
    std::vector<size_t> sizes;
    auto add_copies = [&](double* dst, const double* const* src, const int64_t* off) {
        for (int k = 0; k < K; ++k) {
            dsts.push_back(dst + 3 * off[k]);
            srcs.push_back(const_cast<double*>(src[k]));
            sizes.push_back(3 * (off[k + 1] - off[k]) * sizeof(double));
        }
    };
    add_copies(d_qpos, in.qpos, in.offq);
    add_copies(d_ppos, in.ppos, in.offp);
    VF_TRY(cudaMemcpyAsync(d_offq, in.offq, (K + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, stream));
    VF_TRY(cudaMemcpyAsync(d_offp, in.offp, (K + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, stream));
    const double* d_Ti = d_T;
    const double* d_Tj = d_T + 12 * K;
    const double* d_Tr = d_T + 24 * K;
    VF_TRY(cudaMemcpyAsync(d_T, in.Ti, 12 * K * sizeof(double), cudaMemcpyHostToDevice, stream));
    VF_TRY(cudaMemcpyAsync(d_T + 12 * K, in.Tj, 12 * K * sizeof(double), cudaMemcpyHostToDevice, stream));
    if (in.full) {
        VF_TRY(pool_alloc(&d_qn, 3 * nq * sizeof(double), stream));
        VF_TRY(pool_alloc(&d_pn, 3 * np * sizeof(double), stream));
        add_copies(d_qn, in.qnrm, in.offq);
        add_copies(d_pn, in.pnrm, in.offp);
        VF_TRY(cudaMemcpyAsync(d_T + 24 * K, in.T, 12 * K * sizeof(double), cudaMemcpyHostToDevice, stream));
    }
    mark("allocs");
    // page-locked callers' clouds are read straight over PCIe by one gather
    // kernel (one launch instead of 4K copies); otherwise one copy per array
    std::vector<GatherItem> items;
    if (zero_copy_enabled()) {
        items.reserve(dsts.size());
        for (size_t c = 0; c < dsts.size(); ++c) {
            const double* m = sizes[c] > 0 ? mapped(srcs[c]) : nullptr;
            if (sizes[c] > 0 && !m) {
                items.clear();
                break;
            }
            if (sizes[c] > 0)
                items.push_back(GatherItem{m, static_cast<double*>(dsts[c]),
                                           static_cast<int64_t>(sizes[c] / sizeof(double))});
        }
    }
    if (!items.empty() && items.size() <= 65535) {
        GatherItem* d_items = nullptr;
        const size_t bytes = items.size() * sizeof(GatherItem);
        void* h_items = host_scratch(bytes);
        if (!h_items) VF_TRY(cudaErrorMemoryAllocation);
        std::memcpy(h_items, items.data(), bytes);
        VF_TRY(cudaMallocAsync(&d_items, bytes, stream));
        VF_TRY(cudaMemcpyAsync(d_items, h_items, bytes, cudaMemcpyHostToDevice, stream));
        k_gather_host<<<dim3(8, static_cast<unsigned>(items.size())), 256, 0, stream>>>(d_items);
        VF_TRY(cudaGetLastError());
        cudaFreeAsync(d_items, stream);
    } else {
        for (size_t c = 0; c < dsts.size(); ++c)
            VF_TRY(cudaMemcpyAsync(dsts[c], srcs[c], sizes[c], cudaMemcpyHostToDevice, stream));
    }
    mark("copies enqueued");
    // grid clouds: [T_j P_k]_k for edge_info, then (full) [T_i Q_k]_k, [Q_k]_k
    const int G = in.full ? 3 * K : K;
    const int64_t ng = np + (in.full ? 2 * nq : 0);
    VF_TRY(pool_alloc(&d_grid_pts, 3 * ng * sizeof(double), stream));
    k_pose_batched<<<nblocks(np, 256), 256, 0, stream>>>(d_ppos, np, d_offp, K, d_Tj, d_grid_pts);
    std::vector<int64_t> goff(static_cast<size_t>(G) + 1, 0);
    std::vector<double> gd(static_cast<size_t>(G)), gc(static_cast<size_t>(G));
    for (int k = 0; k < K; ++k) {
        goff[k + 1] = in.offp[k + 1];
        gd[k] = in.epsilon;
        gc[k] = in.epsilon;  // build_grid(posed_j, epsilon): cell = epsilon
    }
    if (in.full) {
        k_pose_batched<<<nblocks(nq, 256), 256, 0, stream>>>(d_qpos, nq, d_offq, K, d_Ti, d_grid_pts + 3 * np);
        VF_TRY(cudaMemcpyAsync(d_grid_pts + 3 * (np + nq), d_qpos, 3 * nq * sizeof(double), cudaMemcpyDeviceToDevice,
                               stream));
        for (int k = 0; k < K; ++k) {
            goff[K + k + 1] = np + in.offq[k + 1];
            gd[K + k] = in.overlap_radius;
            gc[K + k] = in.overlap_radius;  // build_grid(posed[j], overlap_radius)
            goff[2 * K + k + 1] = np + nq + in.offq[k + 1];
            gd[2 * K + k] = in.d_max;
            gc[2 * K + k] = in.grid_cell;
        }
    }
    VF_TRY(build_ring_grids(rb, d_grid_pts, goff.data(), G, gd.data(), gc.data(), stream));
    mark("ring grids");
    VF_TRY(pool_alloc(&d_flags, (nq + 2 * np + 3) * sizeof(uint8_t), stream));
    uint8_t* edge_hit = d_flags;
    uint8_t* overlap_hit = d_flags + nq;
    uint8_t* inl = d_flags + nq + np;
    VF_TRY(pool_alloc(&d_addend, (np > 0 ? np : 1) * sizeof(double), stream));
    VF_TRY(pool_alloc(&d_out, 16 * K * sizeof(double), stream));
    VF_TRY(cudaMemsetAsync(d_flags, 0, nq + 2 * np + 3, stream));
    k_verify_edge<<<nblocks(nq, 128), 128, 0, stream>>>(d_qpos, nq, d_offq, K, d_Ti, rb.d_views,
                                                        in.epsilon * in.epsilon, edge_hit);
    if (in.full)
        k_verify_src<<<nblocks(np, 128), 128, 0, stream>>>(
            d_ppos, d_pn, np, d_offp, K, d_qn, d_offq, d_Tj, d_Tr, rb.d_views + K, rb.d_views + 2 * K,
            in.overlap_radius * in.overlap_radius, in.d_max * in.d_max, in.cos_max, overlap_hit, inl, d_addend);
    k_verify_sums<<<K, kSumThreads, 0, stream>>>(d_qpos, d_offq, edge_hit, d_offp, overlap_hit, inl, d_addend, d_out);
    std::vector<double> h(16 * static_cast<size_t>(K));
    VF_TRY(cudaMemcpyAsync(h.data(), d_out, h.size() * sizeof(double), cudaMemcpyDeviceToHost, stream));
    mark("kernels enqueued");
    VF_TRY(cudaStreamSynchronize(stream));
    mark("done");
#undef VF_TRY
    cleanup();
    for (int k = 0; k < K; ++k) {
        const double* o = h.data() + 16 * k;
        const long long* c = reinterpret_cast<const long long*>(o);
        VerifyOutput& r = out[k];
        // the 6x6 of line_process.cpp:24-28 from the ordered sums
        double L[6][6] = {};
        const double ata[3][3] = {{o[0], o[1], o[2]}, {o[1], o[3], o[4]}, {o[2], o[4], o[5]}};
        const double px = o[6], py = o[7], pz = o[8];
        // TR += a^T, BL += a with a = -[p]x: +0.0 on the diagonals (sums of -0.0 from +0.0)
        const double A[3][3] = {{0.0, pz, -py}, {-pz, 0.0, px}, {py, -px, 0.0}};
        const double n_pairs = static_cast<double>(c[10]);
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                L[a][b] = ata[a][b];
                L[a][3 + b] = A[b][a];
                L[3 + a][b] = A[a][b];
                L[3 + a][3 + b] = a == b ? n_pairs : 0.0;
            }
        for (int a = 0; a < 6; ++a)
            for (int b = 0; b < 6; ++b) r.info[6 * a + b] = c[10] > 0 ? L[a][b] : 0.0;
        r.pair_count = c[10];
        r.overlap_hits = c[11];
        r.inliers = c[12];
        r.sq_sum = o[9];
    }
    return cudaSuccess;
}

// proj/src/fragments.cpp:61-109 on the device: pose every fragment
// (RigidTransform::operator*), one ring grid per posed fragment with the
// reference's build_grid(posed[f], overlap_radius) window, the hit counts of
// every (i, j) pair in one launch. The caller filters and sorts.
cudaError_t propose_loops(const double* h_xyz, const int64_t* h_foff, int32_t n, const double* h_T12,
                          const int32_t* h_pairs, int32_t K, double radius, int64_t* h_hits, cudaStream_t stream) {
    const int64_t np = h_foff[n];
    cudaError_t e = cudaSuccess;
    double *d_xyz = nullptr, *d_posed = nullptr, *d_T = nullptr;
    int64_t *d_foff = nullptr, *d_qoff = nullptr;
    int32_t* d_pairs = nullptr;
    unsigned long long* d_hits = nullptr;
    RingBatch rb;
    auto cleanup = [&] {
        rb.release();
        for (void* p : {(void*)d_xyz, (void*)d_posed, (void*)d_T, (void*)d_foff, (void*)d_qoff, (void*)d_pairs,
                        (void*)d_hits})
            pool_free(p, stream);
    };
#define PL_TRY(x)               \
    do {                        \
        e = (x);                \
        if (e != cudaSuccess) { \
            cleanup();          \
            return e;           \
        }                       \
    } while (0)
    std::vector<int64_t> qoff(static_cast<size_t>(K) + 1, 0);
    for (int k = 0; k < K; ++k) {
        const int i = h_pairs[2 * k];
        qoff[k + 1] = qoff[k] + (h_foff[i + 1] - h_foff[i]);
    }
    PL_TRY(pool_alloc(&d_xyz, 3 * np * sizeof(double), stream));
    PL_TRY(pool_alloc(&d_posed, 3 * np * sizeof(double), stream));
    PL_TRY(pool_alloc(&d_T, 12 * static_cast<int64_t>(n) * sizeof(double), stream));
    PL_TRY(pool_alloc(&d_foff, (n + 1) * sizeof(int64_t), stream));
    PL_TRY(pool_alloc(&d_qoff, (K + 1) * sizeof(int64_t), stream));
    PL_TRY(pool_alloc(&d_pairs, 2 * static_cast<int64_t>(K > 0 ? K : 1) * sizeof(int32_t), stream));
    PL_TRY(pool_alloc(&d_hits, (K > 0 ? K : 1) * sizeof(unsigned long long), stream));
    PL_TRY(cudaMemcpyAsync(d_xyz, h_xyz, 3 * np * sizeof(double), cudaMemcpyHostToDevice, stream));
    PL_TRY(cudaMemcpyAsync(d_T, h_T12, 12 * static_cast<int64_t>(n) * sizeof(double), cudaMemcpyHostToDevice, stream));
    PL_TRY(cudaMemcpyAsync(d_foff, h_foff, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, stream));
    PL_TRY(cudaMemcpyAsync(d_qoff, qoff.data(), (K + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, stream));
    if (K > 0) PL_TRY(cudaMemcpyAsync(d_pairs, h_pairs, 2 * K * sizeof(int32_t), cudaMemcpyHostToDevice, stream));
    PL_TRY(cudaMemsetAsync(d_hits, 0, (K > 0 ? K : 1) * sizeof(unsigned long long), stream));
    k_pose_batched<<<nblocks(np, 256), 256, 0, stream>>>(d_xyz, np, d_foff, n, d_T, d_posed);
    std::vector<double> gd(static_cast<size_t>(n), radius), gc(static_cast<size_t>(n), radius);
    PL_TRY(build_ring_grids(rb, d_posed, h_foff, n, gd.data(), gc.data(), stream));
    if (qoff[K] > 0)
        k_propose_hits<<<nblocks(qoff[K], 128), 128, 0, stream>>>(d_posed, d_foff, d_pairs, d_qoff, K, rb.d_views,
                                                                 radius * radius, d_hits);
    PL_TRY(cudaGetLastError());
    std::vector<unsigned long long> h(static_cast<size_t>(K > 0 ? K : 1));
    PL_TRY(cudaMemcpyAsync(h.data(), d_hits, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream));
    PL_TRY(cudaStreamSynchronize(stream));
#undef PL_TRY
    cleanup();
    for (int k = 0; k < K; ++k) h_hits[k] = static_cast<int64_t>(h[k]);
    return cudaSuccess;
}

}  // namespace lkk
