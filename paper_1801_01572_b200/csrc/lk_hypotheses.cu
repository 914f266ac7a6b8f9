// lk_hypotheses.cu -- the registration hot path on sm_100a (K2-K5, K7).
//
//   k_hyp_sample  RngStream(seed, i) -> 4 distinct sources -> cache -> prerejected
//                 (proj/src/registration.cpp:21-51, 288-298); survivors compacted
//                 with warp-aggregated atomics (Algorithm 1 "stream compact").
//   k_kabsch      FP64 Kabsch + restated Jacobi SVD per survivor
//                 (proj/src/geometry.cpp:62-91); degenerate ones counted.
//   k_score       warp per candidate, 32 consecutive source points per step:
//                 transform, exact NN within d_max over the cell block, normal
//                 gate, inliers, sequential FP64 sum of d2 in point order, exact
//                 miss-budget exit (proj/src/registration.cpp:155-219). The last
//                 CTA to finish reduces the per-CTA bests under the strict total
//                 order (registration.cpp:272-276) and writes the rank record.
//
// Parity: the miss-budget exit is order-free (misses only grow), so exiting
// on the chunk where misses first exceed the budget disqualifies exactly the
// reference's set; the sum is accumulated lane by lane in point order so the
// fitness of every fully scored candidate is bit-identical to the reference's.
#include <cstdint>

#include "lk_device_math.cuh"
#include "lk_kernels.cuh"

namespace lkk {

using namespace lkd;

namespace {

constexpr unsigned kFull = 0xffffffffu;

// Device image of lk_reg_record (include/loopkit_b200.h), 192 bytes.
struct RecordDev {
    int64_t valid;
    int64_t inliers;
    double fitness;
    int64_t index;
    double R[9];
    double t[3];
    int64_t sampled, prerejected, degenerate, evaluated, qualified;
    int64_t w_ref;
    int64_t evals_executed;
    int64_t reserved;
};
static_assert(sizeof(RecordDev) == 192, "record layout");

__device__ __forceinline__ unsigned long long warp_atomic_add(unsigned long long* p, bool pred) {
    unsigned mask = __ballot_sync(kFull, pred);
    int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    int leader = __ffs(mask) - 1;
    if (mask && lane == leader) base = atomicAdd(p, static_cast<unsigned long long>(__popc(mask)));
    base = __shfl_sync(kFull, base, leader < 0 ? 0 : leader);
    return base + __popc(mask & ((1u << lane) - 1u));
}

__global__ void __launch_bounds__(256) k_hyp_sample(int64_t begin, int64_t count, uint64_t seed_mix, uint32_t ns,
                                                    uint32_t thresh, const int32_t* __restrict__ cache,
                                                    const double* __restrict__ spos,
                                                    const double* __restrict__ tpos, double tau,
                                                    int64_t* __restrict__ surv_index, int32_t* __restrict__ surv_ids,
                                                    Counters* __restrict__ ctr) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    // uniform trip count per warp so the warp-wide ballots stay convergent
    const int64_t rounds = (count + stride - 1) / stride;
    for (int64_t r = 0; r < rounds; ++r) {
        int64_t j = r * stride + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
        bool live = j < count;
        bool survive = false;
        int s[4] = {0, 0, 0, 0}, d[4] = {0, 0, 0, 0};
        if (live) {
            Rng rng(seed_mix, static_cast<uint64_t>(begin + j));
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                while (true) {
                    int idx = static_cast<int>(rng.next_bounded(ns, thresh));
                    bool dup = false;
#pragma unroll
                    for (int m = 0; m < 4; ++m) dup = dup || (m < k && s[m] == idx);
                    if (!dup) {
                        s[k] = idx;
                        break;
                    }
                }
                d[k] = __ldg(cache + s[k]);
            }
            V3 sp[4], dp[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                sp[k] = ld3(spos, s[k]);
                dp[k] = ld3(tpos, d[k]);
            }
            survive = !prerejected(sp, dp, tau);
        }
        unsigned long long slot = warp_atomic_add(&ctr->n_survivors, survive);
        unsigned rej = __ballot_sync(kFull, live && !survive);
        if ((threadIdx.x & 31) == 0 && rej) atomicAdd(&ctr->prerejected, static_cast<unsigned long long>(__popc(rej)));
        if (survive) {
            surv_index[slot] = begin + j;
            int4* ids = reinterpret_cast<int4*>(surv_ids + 8 * slot);
            ids[0] = make_int4(s[0], s[1], s[2], s[3]);
            ids[1] = make_int4(d[0], d[1], d[2], d[3]);
        }
    }
}

__global__ void __launch_bounds__(128) k_kabsch(const double* __restrict__ spos, const double* __restrict__ tpos,
                                                const int64_t* __restrict__ surv_index,
                                                const int32_t* __restrict__ surv_ids, int64_t* __restrict__ cand_index,
                                                double* __restrict__ cand_rt, Counters* __restrict__ ctr) {
    const int64_t n = static_cast<int64_t>(ctr->n_survivors);
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t rounds = (n + stride - 1) / stride;
    for (int64_t r = 0; r < rounds; ++r) {
        int64_t j = r * stride + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
        bool live = j < n;
        bool ok = false;
        double R[9], t[3];
        if (live) {
            const int4* ids = reinterpret_cast<const int4*>(surv_ids + 8 * j);
            int4 a = ids[0], b = ids[1];
            V3 sp[4] = {ld3(spos, a.x), ld3(spos, a.y), ld3(spos, a.z), ld3(spos, a.w)};
            V3 dp[4] = {ld3(tpos, b.x), ld3(tpos, b.y), ld3(tpos, b.z), ld3(tpos, b.w)};
            ok = kabsch4(sp, dp, R, t);
        }
        unsigned long long slot = warp_atomic_add(&ctr->n_candidates, ok);
        unsigned deg = __ballot_sync(kFull, live && !ok);
        if ((threadIdx.x & 31) == 0 && deg) atomicAdd(&ctr->degenerate, static_cast<unsigned long long>(__popc(deg)));
        if (ok) {
            cand_index[slot] = surv_index[j];
            double* o = cand_rt + 12 * slot;
#pragma unroll
            for (int k = 0; k < 9; ++k) o[k] = R[k];
#pragma unroll
            for (int k = 0; k < 3; ++k) o[9 + k] = t[k];
        }
    }
}

// Exact NN within d_max over the cell block of y, then the normal gate.
// Returns true for an inlier; `addend` is what the reference adds to sq_sum.
__device__ __forceinline__ bool eval_point(const GridView& g, const double* R, const double* t, V3 p, V3 ns,
                                           const ScoreParams& sp, double& addend) {
    V3 y = xform(R, t, p);
    double fx = floor((y.x - g.ox) / g.cell) - static_cast<double>(g.offx);
    double fy = floor((y.y - g.oy) / g.cell) - static_cast<double>(g.offy);
    double fz = floor((y.z - g.oz) / g.cell) - static_cast<double>(g.offz);
    if (!(fx >= 0.0 && fy >= 0.0 && fz >= 0.0 && fx < g.nx && fy < g.ny && fz < g.nz)) return false;
    const int ix = static_cast<int>(fx), iy = static_cast<int>(fy), iz = static_cast<int>(fz);
    if (!__ldg(g.near + (static_cast<int64_t>(ix) * g.ny + iy) * g.nz + iz)) return false;
    const int r = g.radius;
    const int x0 = max(ix - r, 0), x1 = min(ix + r, g.nx - 1);
    const int y0 = max(iy - r, 0), y1 = min(iy + r, g.ny - 1);
    const int z0 = max(iz - r, 0), z1 = min(iz + r, g.nz - 1);
    double best_d2 = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    int32_t best_slot = -1;
    int32_t best_orig = INT32_MAX;
    for (int x = x0; x <= x1; ++x) {
        for (int yy = y0; yy <= y1; ++yy) {
            const int64_t row = (static_cast<int64_t>(x) * g.ny + yy) * g.nz;
            const int32_t s0 = __ldg(g.start + row + z0);
            const int32_t s1 = __ldg(g.start + row + z1 + 1);
            for (int32_t s = s0; s < s1; ++s) {
                V3 q = ld3(g.slot_pos, s);
                double d2 = sqnorm(sub(q, y));
                if (d2 > sp.d2_max) continue;
                int32_t orig = __ldg(g.index + s);
                if (d2 < best_d2 || (d2 == best_d2 && orig < best_orig)) {
                    best_d2 = d2;
                    best_slot = s;
                    best_orig = orig;
                }
            }
        }
    }
    if (best_slot < 0) return false;
    V3 nt = ld3(g.slot_nrm, best_slot);
    if (is_zero(ns) || is_zero(nt)) return false;
    if (!(dot(rot(R, ns), nt) >= sp.cos_max)) return false;
    if (sp.fitness_from_distance) {
        double dist = sqrt(best_d2);
        addend = dist * dist;
    } else {
        addend = best_d2;
    }
    return true;
}

// strict total order of run_hypotheses (ratio = inliers / Ns is monotone in inliers)
__device__ __forceinline__ bool better(int64_t ia, double fa, int64_t xa, int64_t ib, double fb, int64_t xb) {
    if (ia != ib) return ia > ib;
    if (fa != fb) return fa < fb;
    return xa < xb;
}

constexpr int kScoreThreads = 256;
constexpr int kScoreWarps = kScoreThreads / 32;

__global__ void __launch_bounds__(kScoreThreads) k_score(SourceView src, GridView g, ScoreParams sp,
                                                         const double* __restrict__ cand_rt,
                                                         const int64_t* __restrict__ cand_index, int64_t n_fixed,
                                                         int64_t sampled, int64_t* __restrict__ out_inliers,
                                                         double* __restrict__ out_sum, Counters* __restrict__ ctr,
                                                         BestRec* __restrict__ block_best, RecordDev* __restrict__ rec) {
    __shared__ BestRec s_best[kScoreWarps];
    __shared__ unsigned long long s_ticket;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n_cand = n_fixed >= 0 ? n_fixed : static_cast<int64_t>(ctr->n_candidates);
    const int64_t ns = src.n;
    const double inv_n = static_cast<double>(ns);

    BestRec best{0, 0, 0.0, INT64_MAX, -1};
    unsigned long long qualified = 0, w_ref = 0, executed = 0;

    for (;;) {
        unsigned long long k = 0;
        if (lane == 0) k = atomicAdd(&ctr->work_next, 1ull);
        k = __shfl_sync(kFull, k, 0);
        if (static_cast<int64_t>(k) >= n_cand) break;
        double R[9], t[3];
        const double* crt = cand_rt + 12 * k;
#pragma unroll
        for (int q = 0; q < 9; ++q) R[q] = __ldg(crt + q);
#pragma unroll
        for (int q = 0; q < 3; ++q) t[q] = __ldg(crt + 9 + q);

        int64_t inliers = 0, misses = 0, visited = ns, done = ns;
        double sum = 0.0;
        bool exited = false;
        for (int64_t base = 0; base < ns; base += 32) {
            const int64_t i = base + lane;
            const bool valid = i < ns;
            bool inl = false;
            double addend = 0.0;
            if (valid) inl = eval_point(g, R, t, ld3(src.pos, i), ld3(src.nrm, i), sp, addend);
            const unsigned inl_mask = __ballot_sync(kFull, inl);
            const unsigned miss_mask = __ballot_sync(kFull, valid && !inl);
            // sq_sum += best_d2 in point order (registration.cpp:206)
            unsigned m = inl_mask;
            while (m) {
                const int L = __ffs(m) - 1;
                m &= m - 1;
                sum += __shfl_sync(kFull, addend, L);
            }
            inliers += __popc(inl_mask);
            const int nm = __popc(miss_mask);
            if (misses + nm > sp.miss_budget) {
                // the reference returns at its (budget + 1)-th miss
                int need = static_cast<int>(sp.miss_budget - misses);  // misses to skip in this chunk
                unsigned mm = miss_mask;
                for (int q = 0; q < need; ++q) mm &= mm - 1;
                visited = base + (__ffs(mm) - 1) + 1;
                done = min(base + 32, ns);
                exited = true;
                break;
            }
            misses += nm;
        }
        w_ref += static_cast<unsigned long long>(visited);
        executed += static_cast<unsigned long long>(done);
        const int64_t hyp = cand_index ? __ldg(cand_index + k) : static_cast<int64_t>(k);
        if (out_inliers && lane == 0) {
            out_inliers[k] = exited ? -1 : inliers;
            out_sum[k] = exited ? 0.0 : sum;
        }
        if (!exited) {
            const double ratio = static_cast<double>(inliers) / inv_n;
            const double fitness = inliers > 0 ? sum / static_cast<double>(inliers) : 0.0;
            if (!(ratio < sp.min_ratio || fitness > sp.max_fitness)) {
                qualified += 1;
                if (!best.valid || better(inliers, fitness, hyp, best.inliers, best.fitness, best.index))
                    best = BestRec{1, inliers, fitness, hyp, static_cast<int64_t>(k)};
            }
        }
    }
    if (lane == 0) {
        if (qualified) atomicAdd(&ctr->qualified, qualified);
        if (w_ref) atomicAdd(&ctr->w_ref, w_ref);
        if (executed) atomicAdd(&ctr->evals_executed, executed);
        s_best[warp] = best;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        BestRec b = s_best[0];
        for (int w = 1; w < kScoreWarps; ++w) {
            const BestRec& c = s_best[w];
            if (c.valid && (!b.valid || better(c.inliers, c.fitness, c.index, b.inliers, b.fitness, b.index))) b = c;
        }
        block_best[blockIdx.x] = b;
        __threadfence();
        s_ticket = atomicAdd(&ctr->blocks_done, 1ull);
    }
    __syncthreads();
    if (s_ticket != gridDim.x - 1) return;
    // last CTA: reduce all per-CTA bests and write the record
    __threadfence();
    if (threadIdx.x == 0) {
        BestRec b{0, 0, 0.0, INT64_MAX, -1};
        for (unsigned w = 0; w < gridDim.x; ++w) {
            BestRec c;
            c.valid = __ldcg(&block_best[w].valid);
            c.inliers = __ldcg(&block_best[w].inliers);
            c.fitness = __ldcg(&block_best[w].fitness);
            c.index = __ldcg(&block_best[w].index);
            c.slot = __ldcg(&block_best[w].slot);
            if (c.valid && (!b.valid || better(c.inliers, c.fitness, c.index, b.inliers, b.fitness, b.index))) b = c;
        }
        RecordDev r{};
        r.valid = b.valid;
        r.inliers = b.valid ? b.inliers : 0;
        r.fitness = b.valid ? b.fitness : 0.0;
        r.index = b.valid ? b.index : -1;
        for (int q = 0; q < 9; ++q) r.R[q] = b.valid ? cand_rt[12 * b.slot + q] : 0.0;
        for (int q = 0; q < 3; ++q) r.t[q] = b.valid ? cand_rt[12 * b.slot + 9 + q] : 0.0;
        r.sampled = sampled;
        r.prerejected = static_cast<int64_t>(__ldcg(&ctr->prerejected));
        r.degenerate = static_cast<int64_t>(__ldcg(&ctr->degenerate));
        r.evaluated = n_cand;
        r.qualified = static_cast<int64_t>(__ldcg(&ctr->qualified));
        r.w_ref = static_cast<int64_t>(__ldcg(&ctr->w_ref));
        r.evals_executed = static_cast<int64_t>(__ldcg(&ctr->evals_executed));
        r.reserved = 0;
        *rec = r;
    }
}

int score_blocks_per_sm() {
    static int cached = 0;
    if (!cached) {
        int b = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_score, kScoreThreads, 0) != cudaSuccess || b < 1) b = 1;
        cached = b;
    }
    return cached;
}

}  // namespace

void RunBuffers::release() {
    cudaFree(surv_index);
    cudaFree(surv_ids);
    cudaFree(cand_index);
    cudaFree(cand_rt);
    cudaFree(counters);
    cudaFree(block_best);
    surv_index = nullptr;
    surv_ids = nullptr;
    cand_index = nullptr;
    cand_rt = nullptr;
    counters = nullptr;
    block_best = nullptr;
    capacity = 0;
    n_blocks = 0;
}

cudaError_t RunBuffers::ensure(int64_t cap, int32_t score_blocks) {
    cudaError_t e = cudaSuccess;
    if (!counters && (e = cudaMalloc(&counters, sizeof(Counters))) != cudaSuccess) return e;
    if (score_blocks > n_blocks) {
        cudaFree(block_best);
        if ((e = cudaMalloc(&block_best, score_blocks * sizeof(BestRec))) != cudaSuccess) return e;
        n_blocks = score_blocks;
    }
    if (cap > capacity) {
        cudaFree(surv_index);
        cudaFree(surv_ids);
        cudaFree(cand_index);
        cudaFree(cand_rt);
        surv_index = nullptr;
        surv_ids = nullptr;
        cand_index = nullptr;
        cand_rt = nullptr;
        capacity = 0;
        if ((e = cudaMalloc(&surv_index, cap * sizeof(int64_t))) != cudaSuccess) return e;
        if ((e = cudaMalloc(&surv_ids, cap * 8 * sizeof(int32_t))) != cudaSuccess) return e;
        if ((e = cudaMalloc(&cand_index, cap * sizeof(int64_t))) != cudaSuccess) return e;
        if ((e = cudaMalloc(&cand_rt, cap * 12 * sizeof(double))) != cudaSuccess) return e;
        capacity = cap;
    }
    return cudaSuccess;
}

cudaError_t run_hypotheses_range(const SourceView& src, const double* d_tgt_pos, const int32_t* d_cache,
                                 const GridView& grid, const ScoreParams& sp, uint64_t seed, double tau, int64_t begin,
                                 int64_t end, RunBuffers& rb, void* d_record, cudaStream_t stream, int sm_count,
                                 cudaEvent_t* events) {
    const int64_t count = end - begin;
    const int blocks = sm_count * score_blocks_per_sm();
    cudaError_t e = rb.ensure(count > 0 ? count : 1, blocks);
    if (e != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(rb.counters, 0, sizeof(Counters), stream)) != cudaSuccess) return e;
    const uint32_t ns = static_cast<uint32_t>(src.n);
    const uint32_t thresh = static_cast<uint32_t>(0x100000000ull % ns);
    if (events) cudaEventRecord(events[0], stream);
    if (count > 0) {
        int64_t want = (count + 255) / 256;
        unsigned gs = static_cast<unsigned>(want < sm_count * 16 ? want : sm_count * 16);
        k_hyp_sample<<<gs, 256, 0, stream>>>(begin, count, splitmix64(seed), ns, thresh, d_cache, src.pos, d_tgt_pos,
                                             tau, rb.surv_index, rb.surv_ids, rb.counters);
    }
    if (events) cudaEventRecord(events[1], stream);
    if (count > 0) {
        k_kabsch<<<sm_count * 8, 128, 0, stream>>>(src.pos, d_tgt_pos, rb.surv_index, rb.surv_ids, rb.cand_index,
                                                   rb.cand_rt, rb.counters);
    }
    if (events) cudaEventRecord(events[2], stream);
    k_score<<<blocks, kScoreThreads, 0, stream>>>(src, grid, sp, rb.cand_rt, rb.cand_index, -1, count, nullptr,
                                                  nullptr, rb.counters, rb.block_best,
                                                  static_cast<RecordDev*>(d_record));
    if (events) cudaEventRecord(events[3], stream);
    return cudaGetLastError();
}

cudaError_t score_candidates(const SourceView& src, const GridView& grid, const ScoreParams& sp, const double* d_rt,
                             int64_t C, RunBuffers& rb, int64_t* d_out_inliers, double* d_out_sum, void* d_record,
                             cudaStream_t stream, int sm_count) {
    const int blocks = sm_count * score_blocks_per_sm();
    cudaError_t e = rb.ensure(1, blocks);
    if (e != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(rb.counters, 0, sizeof(Counters), stream)) != cudaSuccess) return e;
    k_score<<<blocks, kScoreThreads, 0, stream>>>(src, grid, sp, d_rt, nullptr, C, C, d_out_inliers, d_out_sum,
                                                  rb.counters, rb.block_best, static_cast<RecordDev*>(d_record));
    return cudaGetLastError();
}

}  // namespace lkk
