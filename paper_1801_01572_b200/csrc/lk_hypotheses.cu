// lk_hypotheses.cu -- the registration hot path on sm_100a (K2-K5, K7).
//
//   k_hyp_sample    RngStream(seed, i) -> 4 distinct sources -> cache -> prerejected
//                   (proj/src/registration.cpp:21-51, 288-298); survivors compacted
//                   with warp-aggregated atomics (Algorithm 1 "stream compact").
//   k_kabsch        FP64 Kabsch + restated Jacobi SVD per survivor
//                   (proj/src/geometry.cpp:62-91); degenerate ones counted.
//   k_score_cta     persistent CTA per candidate (the default scorer): rounds of
//                   2,048 source points -- FP32 fine-cell lookups settle the
//                   certain misses, a shared-memory queue sends the rest to the
//                   exact FP64 resolution (guard bands), ballots and
//                   the reference's miss budget in point order; order-bounded
//                   sums with the sequential chain on demand; the last CTA
//                   writes the rank record (registration.cpp:155-219, 253-332).
//   k_score_units   the same work split into (candidate, round) units when a
//                   rank has fewer candidates than CTAs (strong scaling).
//   k_score_list / k_score_list_ring / k_score
//                   explicit candidate lists (EvalGrid with fine lists, dense
//                   targets through the ring grid, SearchGrid semantics).
//
// Parity: disqualification by the miss budget depends only on the total miss
// count (misses only grow), so evaluating every point and deciding afterwards
// disqualifies exactly the reference's set; the reference's visit count is
// recovered from the ordered miss ballots. Sums are added lane by lane in
// point order, so every fitness is bit-identical to the reference's.
#include <cstdint>
#include <cstdlib>

#include "lk_device_math.cuh"
#include "lk_kernels.cuh"
#include "lk_score_common.cuh"
#include "lk_ring.cuh"

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

// Byte ranges the scoring phase gathers from (grid lists, target and source
// arrays). k_hyp_sample pulls them into L2 with bulk prefetches as it starts,
// so the scoring kernel's dependent gathers hit L2 instead of DRAM.
struct PrefetchList {
    static constexpr int kMax = 8;
    const char* ptr[kMax];
    unsigned long long bytes[kMax];
    int n;
};
constexpr unsigned kPrefetchChunk = 64 << 10;

__device__ __forceinline__ void l2_prefetch_bulk(const void* p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__global__ void __launch_bounds__(256) k_hyp_sample(int64_t begin, int64_t count, uint64_t seed_mix, uint32_t ns,
                                                    uint32_t thresh, const int32_t* __restrict__ cache,
                                                    const double* __restrict__ spos,
                                                    const double* __restrict__ tpos, double tau,
                                                    int64_t* __restrict__ surv_index, int32_t* __restrict__ surv_ids,
                                                    Counters* __restrict__ ctr, const __grid_constant__ PrefetchList pf) {
    if (blockIdx.x < pf.n) {
        // range blockIdx.x, 64 KB per thread-step (16-byte granules)
        const char* p = pf.ptr[blockIdx.x];
        const unsigned long long nb = pf.bytes[blockIdx.x] & ~15ull;
        for (unsigned long long o = static_cast<unsigned long long>(threadIdx.x) * kPrefetchChunk; o < nb;
             o += static_cast<unsigned long long>(blockDim.x) * kPrefetchChunk) {
            const unsigned long long left = nb - o;
            l2_prefetch_bulk(p + o, static_cast<unsigned>(left < kPrefetchChunk ? left : kPrefetchChunk));
        }
    }
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
            }
            // prerejected (registration.cpp:42-51) edge by edge, loading the
            // corners as the edges need them: most quadruples fail on the
            // first edge, so most skip half of the gathers
            V3 sp[4], dp[4];
            auto corner = [&](int k) {
                d[k] = __ldg(cache + s[k]);
                sp[k] = ld3(spos, s[k]);
                dp[k] = ld3(tpos, d[k]);
            };
            auto edge_fails = [&](int a, int b) {
                const double es = sqrt(sqnorm(sub(sp[a], sp[b])));
                const double ed = sqrt(sqnorm(sub(dp[a], dp[b])));
                return es < tau * ed || ed < tau * es;
            };
            corner(0);
            corner(1);
            bool rej = edge_fails(0, 1);
            if (!rej) {
                corner(2);
                rej = edge_fails(1, 2);
                if (!rej) {
                    corner(3);
                    rej = edge_fails(2, 3) || edge_fails(3, 0);
                }
            }
            survive = !rej;
        }
        // prerejected = sampled - survivors (every live hypothesis is one or
        // the other), so only the survivors touch a counter
        unsigned long long slot = warp_atomic_add(&ctr->n_survivors, survive);
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
                                                double* __restrict__ cand_rt, Counters* __restrict__ ctr,
                                                double* __restrict__ u_sum = nullptr,
                                                unsigned* __restrict__ u_done = nullptr, int64_t u_cap = 0) {
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
            if (static_cast<int64_t>(slot) < u_cap) {  // the unit scorer's per-candidate sum and unit count
                u_sum[slot] = 0.0;
                u_done[slot] = 0u;
            }
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
    const int64_t c = (static_cast<int64_t>(ix) * g.ny + iy) * g.nz + iz;
    double best_d2 = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    int32_t best_orig = INT32_MAX;
    if (g.block_info) {
        const int2 bi = __ldg(g.block_info + c);
        if (bi.y == 0) return false;  // not near-occupied
        for (int32_t e = bi.x; e < bi.x + bi.y; ++e) {
            const double2* bp = reinterpret_cast<const double2*>(g.block_pts + e);
            const double2 qa = __ldg(bp), qb = __ldg(bp + 1);
            const double dx = qa.x - y.x, dy = qa.y - y.y, dz = qb.x - y.z;
            const double d2 = (dx * dx + dy * dy) + dz * dz;
            if (d2 > sp.d2_max) continue;
            const int32_t orig = static_cast<int32_t>(qb.y);
            if (d2 < best_d2 || (d2 == best_d2 && orig < best_orig)) {
                best_d2 = d2;
                best_orig = orig;
            }
        }
    } else {
        if (!__ldg(g.near + c)) return false;
        const int r = g.radius;
        const int x0 = max(ix - r, 0), x1 = min(ix + r, g.nx - 1);
        const int y0 = max(iy - r, 0), y1 = min(iy + r, g.ny - 1);
        const int z0 = max(iz - r, 0), z1 = min(iz + r, g.nz - 1);
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
                        best_orig = orig;
                    }
                }
            }
        }
    }
    if (best_orig == INT32_MAX) return false;
    V3 nt = ld3(g.nrm_orig, best_orig);
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

// ---- FP32 guard-band fast path ----------
// Cell coordinates q = R' p + t' (R' = R / cell, t' = (t - o) / cell - off) and
// the block scan run in FP32; every decision that the FP32 values cannot
// certify -- a coordinate within eps of a cell face, an entry within the band
// of d_max, two entries within twice the band of each other -- and every
// quantity that feeds the result (the winning d2, the normal gate) is
// evaluated in FP64 exactly as the reference does.
// Per-candidate FP32 image of (R, t) in grid cell units and its guard bands.
// Error bound of q = R' p + t' evaluated by the fmaf chain below (rows of R
// have unit norm): |dq| <= 2^-24 (5 |p|max + 4 |t'|) cells; entries carry
// <= 2^-24 n. With delta = both, d2 within one cell is off by at most
// 2 sqrt3 delta + 3 delta^2 (+ FP32 rounding of d2 itself); bands are 4x that.
__device__ __forceinline__ FastRT make_fast(const double* R, const double* t, const GridView& g,
                                            const ScoreParams& sp) {
    FastRT f;
#pragma unroll
    for (int k = 0; k < 9; ++k) f.r[k] = static_cast<float>(R[k] / g.cell);
    f.t[0] = static_cast<float>((t[0] - g.ox) / g.cell - g.offx);
    f.t[1] = static_cast<float>((t[1] - g.oy) / g.cell - g.offy);
    f.t[2] = static_cast<float>((t[2] - g.oz) / g.cell - g.offz);
    const float u = 5.9604645e-8f;  // 2^-24
    const float tn = sqrtf(f.t[0] * f.t[0] + f.t[1] * f.t[1] + f.t[2] * f.t[2]);
    const float dq = u * (5.0f * sp.pmax_cells + 4.0f * tn + 4.0f);
    const float de = u * (sp.nmax_cells + 2.0f);
    const float delta = dq + de;
    f.eps = 4.0f * dq + 1e-6f;
    f.band = 4.0f * (3.5f * delta + 3.0f * delta * delta + 8.0f * u) + 1e-7f;
    f.ok = (sp.fast && f.eps < 0.02f && f.band < 0.02f) ? 1.0f : 0.0f;
    f.pad = 0.0f;
    return f;
}

__device__ __forceinline__ FastRT load_fast(const FastRT* __restrict__ p) {
    const float4* q = reinterpret_cast<const float4*>(p);
    const float4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2), d = __ldg(q + 3);
    FastRT f;
    f.r[0] = a.x; f.r[1] = a.y; f.r[2] = a.z; f.r[3] = a.w;
    f.r[4] = b.x; f.r[5] = b.y; f.r[6] = b.z; f.r[7] = b.w;
    f.r[8] = c.x; f.t[0] = c.y; f.t[1] = c.z; f.t[2] = c.w;
    f.eps = d.x; f.band = d.y; f.ok = d.z; f.pad = d.w;
    return f;
}

// FastRT of every candidate (n_fixed >= 0, or the device candidate count).
__global__ void k_prep_fast(const double* __restrict__ cand_rt, int64_t n_fixed, const Counters* __restrict__ ctr,
                            GridView g, ScoreParams sp, FastRT* __restrict__ out) {
    const int64_t n = n_fixed >= 0 ? n_fixed : static_cast<int64_t>(ctr->n_candidates);
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double R[9], t[3];
#pragma unroll
        for (int q = 0; q < 9; ++q) R[q] = cand_rt[12 * k + q];
#pragma unroll
        for (int q = 0; q < 3; ++q) t[q] = cand_rt[12 * k + 9 + q];
        out[k] = make_fast(R, t, g, sp);
    }
}

__device__ __forceinline__ bool eval_point_fast(const GridView& g, const double* R, const double* t,
                                                const FastRT& F, const SourceView& src, int64_t i,
                                                const ScoreParams& sp, double& addend) {
    if (F.ok == 0.0f) return eval_point(g, R, t, ld3(src.pos, i), ld3(src.nrm, i), sp, addend);
    const float4 P = __ldg(src.pos32 + i);
    const float qx = fmaf(F.r[0], P.x, fmaf(F.r[1], P.y, fmaf(F.r[2], P.z, F.t[0])));
    const float qy = fmaf(F.r[3], P.x, fmaf(F.r[4], P.y, fmaf(F.r[5], P.z, F.t[1])));
    const float qz = fmaf(F.r[6], P.x, fmaf(F.r[7], P.y, fmaf(F.r[8], P.z, F.t[2])));
    const float eps = F.eps;
    // certainly outside the grid
    if (qx < -eps || qy < -eps || qz < -eps || qx >= g.nx + eps || qy >= g.ny + eps || qz >= g.nz + eps)
        return false;
    const float fx = floorf(qx), fy = floorf(qy), fz = floorf(qz);
    const float rx = qx - fx, ry = qy - fy, rz = qz - fz;
    if (rx < eps || rx > 1.0f - eps || ry < eps || ry > 1.0f - eps || rz < eps || rz > 1.0f - eps)
        return eval_point(g, R, t, ld3(src.pos, i), ld3(src.nrm, i), sp, addend);  // near a cell face
    const int ix = static_cast<int>(fx), iy = static_cast<int>(fy), iz = static_cast<int>(fz);
    if (ix < 0 || iy < 0 || iz < 0 || ix >= g.nx || iy >= g.ny || iz >= g.nz) return false;
    const int2 bi = __ldg(g.block_info + (static_cast<int64_t>(ix) * g.ny + iy) * g.nz + iz);
    if (bi.y == 0) return false;  // not near-occupied
    // FP32 scan keeping the three smallest d2 (entries of the two best)
    const float inf = __int_as_float(0x7f800000);
    float f1 = inf, f2 = inf, f3 = inf;
    int32_t o1 = -1, o2 = -1;
    for (int32_t e = bi.x; e < bi.x + bi.y; ++e) {
        const float4 E = __ldg(g.block_f32 + e);
        const float dx = qx - E.x, dy = qy - E.y, dz = qz - E.z;
        const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
        const int32_t o = __float_as_int(E.w);
        if (d2 < f1) {
            f3 = f2;
            f2 = f1;
            o2 = o1;
            f1 = d2;
            o1 = o;
        } else if (d2 < f2) {
            f3 = f2;
            f2 = d2;
            o2 = o;
        } else if (d2 < f3) {
            f3 = d2;
        }
    }
    const float band = F.band;
    if (f1 > sp.thr_cells + band) return false;  // every entry is certainly beyond d_max
    // exact FP64 from here on
    const V3 y = xform(R, t, ld3(src.pos, i));
    double best_d2 = __longlong_as_double(0x7ff0000000000000ll);
    int32_t best_orig = INT32_MAX;
    const float lim = f1 + 2.0f * band;
    if (f3 <= lim) {
        // three or more entries tie within the guard: resolve all of them exactly
        for (int32_t e = bi.x; e < bi.x + bi.y; ++e) {
            const float4 E = __ldg(g.block_f32 + e);
            const float dx = qx - E.x, dy = qy - E.y, dz = qz - E.z;
            if (fmaf(dx, dx, fmaf(dy, dy, dz * dz)) > lim) continue;
            const int32_t orig = __float_as_int(E.w);
            const double d2 = sqnorm(sub(ld3(g.pos_orig, orig), y));
            if (d2 > sp.d2_max) continue;
            if (d2 < best_d2 || (d2 == best_d2 && orig < best_orig)) {
                best_d2 = d2;
                best_orig = orig;
            }
        }
    } else {
        // the FP32 winner, and the runner-up if it is within the guard
        const double d2a = sqnorm(sub(ld3(g.pos_orig, o1), y));
        if (d2a <= sp.d2_max) {
            best_d2 = d2a;
            best_orig = o1;
        }
        if (f2 <= lim) {
            const double d2b = sqnorm(sub(ld3(g.pos_orig, o2), y));
            if (d2b <= sp.d2_max && (d2b < best_d2 || (d2b == best_d2 && o2 < best_orig))) {
                best_d2 = d2b;
                best_orig = o2;
            }
        }
    }
    if (best_orig == INT32_MAX) return false;
    const V3 ns = ld3(src.nrm, i);
    const V3 nt = ld3(g.nrm_orig, best_orig);
    if (is_zero(ns) || is_zero(nt)) return false;
    if (!(dot(rot(R, ns), nt) >= sp.cos_max)) return false;
    if (sp.fitness_from_distance) {
        const double dist = sqrt(best_d2);
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
__device__ __forceinline__ bool better(const BestRec& a, const BestRec& b) {
    return a.valid && (!b.valid || better(a.inliers, a.fitness, a.index, b.inliers, b.fitness, b.index));
}

constexpr int kScoreThreads = 256;
constexpr int kScoreWarps = kScoreThreads / 32;

struct WarpTally {
    BestRec best{0, 0, 0.0, INT64_MAX, -1};
    unsigned long long qualified = 0, w_ref = 0, executed = 0;

    __device__ __forceinline__ void candidate(int64_t inliers, double sum, int64_t ns, const ScoreParams& sp,
                                              int64_t hyp, int64_t slot) {
        const double ratio = static_cast<double>(inliers) / static_cast<double>(ns);
        const double fitness = inliers > 0 ? sum / static_cast<double>(inliers) : 0.0;
        if (ratio < sp.min_ratio || fitness > sp.max_fitness) return;
        qualified += 1;
        BestRec c{1, inliers, fitness, hyp, slot};
        if (better(c, best)) best = c;
    }
};

// Per-CTA: fold the warps' tallies, publish the CTA best and counters.
// Returns true in the CTA that finishes last (it then owns the final reduce).
__device__ bool publish_cta(const WarpTally& wt, Counters* ctr, BestRec* block_best, int slot, bool want_ticket) {
    __shared__ BestRec s_best[kScoreWarps];
    __shared__ unsigned long long s_tally[kScoreWarps][3];
    __shared__ unsigned long long s_ticket;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        s_tally[warp][0] = wt.qualified;
        s_tally[warp][1] = wt.w_ref;
        s_tally[warp][2] = wt.executed;
        s_best[warp] = wt.best;
    }
    __syncthreads();
    // one thread per CTA touches the global counters (same-address atomics
    // from every warp serialise in one L2 slice)
    if (threadIdx.x == 0) {
        unsigned long long q = 0, w = 0, x = 0;
        for (int k = 0; k < kScoreWarps; ++k) {
            q += s_tally[k][0];
            w += s_tally[k][1];
            x += s_tally[k][2];
        }
        if (q) atomicAdd(&ctr->qualified, q);
        if (w) atomicAdd(&ctr->w_ref, w);
        if (x) atomicAdd(&ctr->evals_executed, x);
        BestRec b = s_best[0];
        for (int k = 1; k < kScoreWarps; ++k)
            if (better(s_best[k], b)) b = s_best[k];
        block_best[slot] = b;
        __threadfence();
        s_ticket = want_ticket ? atomicAdd(&ctr->blocks_done, 1ull) : 0ull;
    }
    __syncthreads();
    return want_ticket && s_ticket == gridDim.x - 1;
}

// Final reduce over n_best per-CTA bests (strict total order) -> record.
__device__ void write_record(const BestRec* block_best, int n_best, const double* cand_rt, int64_t n_cand,
                             int64_t sampled, Counters* ctr, RecordDev* rec) {
    __threadfence();
    if (threadIdx.x != 0) return;
    BestRec b{0, 0, 0.0, INT64_MAX, -1};
    for (int w = 0; w < n_best; ++w) {
        BestRec c;
        c.valid = __ldcg(&block_best[w].valid);
        c.inliers = __ldcg(&block_best[w].inliers);
        c.fitness = __ldcg(&block_best[w].fitness);
        c.index = __ldcg(&block_best[w].index);
        c.slot = __ldcg(&block_best[w].slot);
        if (better(c, b)) b = c;
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

__device__ __forceinline__ void load_rt(const double* __restrict__ crt, double* R, double* t) {
    const double2* p = reinterpret_cast<const double2*>(crt);
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        double2 v = __ldg(p + q);
        double a = v.x, b = v.y;
        int k0 = 2 * q, k1 = 2 * q + 1;
        if (k0 < 9) R[k0] = a; else t[k0 - 9] = a;
        if (k1 < 9) R[k1] = b; else t[k1 - 9] = b;
    }
}

// Warp per candidate, points streamed in order (explicit candidate lists and
// SearchGrid targets: evaluate_hypothesis semantics).
__global__ void __launch_bounds__(kScoreThreads) k_score(SourceView src, GridView g, ScoreParams sp,
                                                         const double* __restrict__ cand_rt,
                                                         const FastRT* __restrict__ cand_fast,
                                                         const int64_t* __restrict__ cand_index, int64_t cand_begin,
                                                         int64_t n_fixed, int64_t sampled,
                                                         int64_t* __restrict__ out_inliers, double* __restrict__ out_sum,
                                                         Counters* __restrict__ ctr, BestRec* __restrict__ block_best,
                                                         int best_offset, RecordDev* __restrict__ rec) {
    const int lane = threadIdx.x & 31;
    const int64_t n_cand = n_fixed >= 0 ? n_fixed : static_cast<int64_t>(ctr->n_candidates);
    const int64_t ns = src.n;
    WarpTally wt;
    for (;;) {
        unsigned long long k = 0;
        if (lane == 0) k = cand_begin + atomicAdd(&ctr->work_next, 1ull);
        k = __shfl_sync(kFull, k, 0);
        if (static_cast<int64_t>(k) >= n_cand) break;
        double R[9], t[3];
        load_rt(cand_rt + 12 * k, R, t);
        const FastRT F = load_fast(cand_fast + k);
        int64_t inliers = 0, misses = 0, visited = ns, done = ns;
        double sum = 0.0;
        bool exited = false;
        for (int64_t base = 0; base < ns; base += 32) {
            const int64_t i = base + lane;
            const bool valid = i < ns;
            bool inl = false;
            double addend = 0.0;
            if (valid) inl = eval_point_fast(g, R, t, F, src, i, sp, addend);
            const unsigned inl_mask = __ballot_sync(kFull, inl);
            const unsigned miss_mask = __ballot_sync(kFull, valid && !inl);
            // sq_sum += best_d2 in point order (registration.cpp:206); a
            // non-inlier lane adds +0.0, which leaves the sum unchanged
            if (inl_mask) {
#pragma unroll
                for (int L = 0; L < 32; ++L) sum += __shfl_sync(kFull, addend, L);
            }
            inliers += __popc(inl_mask);
            const int nm = __popc(miss_mask);
            if (misses + nm > sp.miss_budget) {
                // the reference returns at its (budget + 1)-th miss
                int need = static_cast<int>(sp.miss_budget - misses);
                unsigned mm = miss_mask;
                for (int q = 0; q < need; ++q) mm &= mm - 1;
                visited = base + (__ffs(mm) - 1) + 1;
                done = min(base + 32, ns);
                exited = true;
                break;
            }
            misses += nm;
        }
        wt.w_ref += static_cast<unsigned long long>(visited);
        wt.executed += static_cast<unsigned long long>(done);
        const int64_t hyp = cand_index ? __ldg(cand_index + k) : static_cast<int64_t>(k);
        if (out_inliers && lane == 0) {
            out_inliers[k] = exited ? -1 : inliers;
            out_sum[k] = exited ? 0.0 : sum;
        }
        if (!exited) wt.candidate(inliers, sum, ns, sp, hyp, static_cast<int64_t>(k));
    }
    const bool last = publish_cta(wt, ctr, block_best, best_offset + blockIdx.x, rec != nullptr);
    if (last) write_record(block_best, best_offset + gridDim.x, cand_rt, n_cand, sampled, ctr, rec);
}

// Exact resolution of one query over its fine list: FP32 top-3 with the guard
// band, FP64 d2 for every entry that can be the minimum, the normal gate.
// Every entry comes from the block list of the query's EvalGrid cell (the
// certain fine cell halved: (y - o) / fcell is exactly 2 (y - o) / cell in
// FP64), i.e. from the reference's own search window (registration.cpp:167-169),
// and Voronoi pruning only drops entries another listed entry beats everywhere
// in the cell, so the minimum over the list is the reference's neighbour.
// Out of line so its registers do not count against the callers' occupancy;
// everything is reloaded from global memory (rt = the candidate's 12 doubles).
__device__ __noinline__ bool eval_point_slow(const GridView& g, const double* rt, const SourceView& src, int64_t i,
                                             const ScoreParams& sp, double* addend) {
    double R[9], t[3];
    load_rt(rt, R, t);
    return eval_point(g, R, t, ld3(src.pos, i), ld3(src.nrm, i), sp, *addend);
}

__device__ __forceinline__ bool resolve_fine(const GridView& g, const double* R, const double* t, const float* Rf,
                                             const FastRT& F, const SourceView& src, int64_t i, V3 p, float4 ns32,
                                             float qx, float qy, float qz, int32_t off, int32_t cnt,
                                             const ScoreParams& sp, double& addend) {
    const float inf = __int_as_float(0x7f800000);
    float f1 = inf, f2 = inf, f3 = inf;
    int32_t o1 = -1, o2 = -1;
    int32_t e = off;
    const int32_t end = off + cnt;
    for (; e + 3 < end; e += 4) {  // four independent loads in flight
        const float4 A = __ldg(g.fine_pts + e), B = __ldg(g.fine_pts + e + 1);
        const float4 C = __ldg(g.fine_pts + e + 2), D = __ldg(g.fine_pts + e + 3);
        float x, y, z;
        x = qx - A.x; y = qy - A.y; z = qz - A.z;
        top3(fmaf(x, x, fmaf(y, y, z * z)), __float_as_int(A.w), f1, f2, f3, o1, o2);
        x = qx - B.x; y = qy - B.y; z = qz - B.z;
        top3(fmaf(x, x, fmaf(y, y, z * z)), __float_as_int(B.w), f1, f2, f3, o1, o2);
        x = qx - C.x; y = qy - C.y; z = qz - C.z;
        top3(fmaf(x, x, fmaf(y, y, z * z)), __float_as_int(C.w), f1, f2, f3, o1, o2);
        x = qx - D.x; y = qy - D.y; z = qz - D.z;
        top3(fmaf(x, x, fmaf(y, y, z * z)), __float_as_int(D.w), f1, f2, f3, o1, o2);
    }
    for (; e < end; ++e) {
        const float4 A = __ldg(g.fine_pts + e);
        const float ax = qx - A.x, ay = qy - A.y, az = qz - A.z;
        top3(fmaf(ax, ax, fmaf(ay, ay, az * az)), __float_as_int(A.w), f1, f2, f3, o1, o2);
    }
    const float band = F.band;
    if (f1 > F.pad + band) return false;  // nothing within d_max of y
    // the FP32 winner's normal is fetched with its position: it is the
    // neighbour in all but near-tie cases, and saves a dependent round trip
    const bool pre_nt = Rf && g.nrm32_orig;
    const float4 nt1 = pre_nt ? __ldg(g.nrm32_orig + o1) : make_float4(0.f, 0.f, 0.f, 0.f);
    const V3 y = xform(R, t, p);
    double best_d2 = __longlong_as_double(0x7ff0000000000000ll);
    int32_t best_orig = INT32_MAX;
    auto consider = [&](int32_t o) {
        const V3 q = g.pos4_orig ? ld4(g.pos4_orig, o) : ld3(g.pos_orig, o);
        const double d2 = sqnorm(sub(q, y));
        if (d2 > sp.d2_max) return;
        if (d2 < best_d2 || (d2 == best_d2 && o < best_orig)) {
            best_d2 = d2;
            best_orig = o;
        }
    };
    const float lim = f1 + 2.0f * band;
    if (f3 <= lim) {
        for (int32_t k = off; k < end; ++k) {
            const float4 E = __ldg(g.fine_pts + k);
            const float dx = qx - E.x, dy = qy - E.y, dz = qz - E.z;
            if (fmaf(dx, dx, fmaf(dy, dy, dz * dz)) <= lim) consider(__float_as_int(E.w));
        }
    } else {
        consider(o1);
        if (f2 <= lim) consider(o2);
    }
    if (best_orig == INT32_MAX) return false;
    bool gate_done = false;
    if (Rf && g.nrm32_orig) {
        // FP32 normal gate; only a value within the guard of cos_max (or a zero
        // FP32 normal) is decided by the reference's FP64 expression below
        const float4 nt = best_orig == o1 ? nt1 : __ldg(g.nrm32_orig + best_orig);
        const float ns1 = fabsf(ns32.x) + fabsf(ns32.y) + fabsf(ns32.z);
        const float nt1 = fabsf(nt.x) + fabsf(nt.y) + fabsf(nt.z);
        if (ns1 > 0.0f && nt1 > 0.0f) {
            const float ax = fmaf(Rf[0], ns32.x, fmaf(Rf[1], ns32.y, Rf[2] * ns32.z));
            const float ay = fmaf(Rf[3], ns32.x, fmaf(Rf[4], ns32.y, Rf[5] * ns32.z));
            const float az = fmaf(Rf[6], ns32.x, fmaf(Rf[7], ns32.y, Rf[8] * ns32.z));
            const double d = static_cast<double>(fmaf(ax, nt.x, fmaf(ay, nt.y, az * nt.z)));
            const double guard = static_cast<double>(kGateGuard * ns1 * nt1);
            if (d < sp.cos_max - guard) return false;
            gate_done = d > sp.cos_max + guard;
        }
    }
    if (!gate_done) {
        const V3 ns = ld3(src.nrm, i);
        const V3 nt = ld3(g.nrm_orig, best_orig);
        if (is_zero(ns) || is_zero(nt)) return false;
        if (!(dot(rot(R, ns), nt) >= sp.cos_max)) return false;
    }
    if (sp.fitness_from_distance) {
        const double dist = sqrt(best_d2);
        addend = dist * dist;
    } else {
        addend = best_d2;
    }
    return true;
}

__device__ __forceinline__ double order_bound(int64_t n) { return 2.0 * static_cast<double>(n + 1) * 1.1102230246251565e-16 + 4.5e-16; }


// ---- candidate-CTA scoring ------------------------------------------------
// One CTA owns one candidate at a time (persistent grid, candidates taken from
// a ticket counter) and walks its source points in rounds of kCtaPts:
//   A. every thread transforms its points in FP32 (fine-cell units), settles
//      the certain misses and appends the rest to a shared-memory queue with
//      their fine-list (offset, count), or the exact FP64 tag;
//   B. the queue is resolved densely by all threads (resolve_fine /
//      eval_point_slow); results land as bits of the round's ballots (double
//      buffered by round parity); the inliers' d2 go to the CTA's scratch slot
//      in point order and into per-thread partial sums;
//   C. every warp applies the reference's miss budget to the round's ballots
//      (exit => the visited count from the ordered ballots, warp 0).
// At the end of a candidate the partial sums give its fitness within a
// rigorous order bound; qualification and the comparison with the CTA's best
// are decided by the bound, and only when it straddles a decision is the
// reference's own sequential sum (registration.cpp:206) run from the scratch
// slot. Each CTA's best ends with its exact sequential sum, so the strict
// total order (registration.cpp:272-276) across CTAs is exact; the last CTA
// writes the rank record. Two scratch slots per CTA (current, best) swap
// instead of copying.
constexpr int kCtaThreads = 256;
constexpr int kCtaWarps = kCtaThreads / 32;
constexpr int kCtaPer = 8;                         // points per thread per round
constexpr int kCtaPts = kCtaThreads * kCtaPer;     // points per round
// points per (candidate, unit) work item of k_score_units. Shorter units were
// measured slower (125k / 250k / 500k hypotheses per rank: 256 points 0.213 /
// 0.304 / 0.480 ms, 512: 0.189 / 0.250 / 0.371, 1024: 0.178 / 0.226 / 0.318,
// 2048: 0.182 / 0.226 / 0.299): per-unit setup and the lost early exits cost
// more than the shorter unit latency saves.
#ifndef LK_UNIT_PTS
#define LK_UNIT_PTS 2048
#endif
constexpr int kUnitPts = LK_UNIT_PTS;
static_assert(kUnitPts % kCtaThreads == 0 && kUnitPts <= kCtaPts, "unit = whole thread rows of a round");
constexpr int kCtaWords = kCtaPts / 32;            // ballot words per round (32 or 64)
static_assert(kCtaWords % 32 == 0, "ballot words come in warp-sized groups");
constexpr int kCtaSlow = 0xffff;                   // queue count tag: exact FP64 fallback
constexpr int kCtaChainChunks = kCtaPts / 32;      // chain window: the queue's 16 KB as doubles

struct CtaSmem {
    union {
        int2 q[kCtaPts];            // A/B: (local | count << 16, fine-list offset)
        double chain[kCtaPts];      // exact chains: compacted addends of 64 chunks
    };
    uint32_t inl[2][kCtaWords];
    uint32_t miss[2][kCtaWords];
    uint32_t cmask[kCtaChainChunks];
    int coff[kCtaChainChunks];
    double R[9], t[3];
    float Rf[9];
    FastRT F;
    double red[kCtaWarps];
    int scan[kCtaWarps];
    // per round parity b: queue counts of round b (list scans / exact-fallback
    // entries, the latter queued from the back of q). Round r's phase B clears
    // parity b ^ 1, so no reset ever races the next round's phase-A atomics.
    int nq[2];
    int nslow[2];
    int next;  // B: next queue entry a warp takes (dynamic, 32 at a time)
    int flag;
    int swap;
    double exact[2];
    int64_t cand;
};

// Sequential FP64 sum of one candidate's inliers' d2 in point order
// (registration.cpp:206) by a whole CTA from its ballot words `im` and
// addends `ad` (global scratch): 64 chunks at a time are compacted in point
// order into shared memory, then thread 0 runs the dependent add chain.
// Result valid in thread 0. All threads must call it.
__device__ double cta_chain(const uint32_t* im, const double* ad, int32_t n_chunks, CtaSmem& S) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned below = (1u << lane) - 1u;
    double sum = 0.0;
    for (int32_t c0 = 0; c0 < n_chunks; c0 += kCtaChainChunks) {
        const int nc = n_chunks - c0 < kCtaChainChunks ? n_chunks - c0 : kCtaChainChunks;
        const uint32_t m = threadIdx.x < nc ? __ldcg(im + c0 + threadIdx.x) : 0u;
        // block exclusive scan of the popcounts
        const int v = __popc(m);
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) S.scan[warp] = incl;
        __syncthreads();
        int base = 0, total = 0;
#pragma unroll
        for (int w = 0; w < kCtaWarps; ++w) {
            base += w < warp ? S.scan[w] : 0;
            total += S.scan[w];
        }
        if (threadIdx.x < kCtaChainChunks) {
            S.cmask[threadIdx.x] = m;
            S.coff[threadIdx.x] = base + incl - v;
        }
        __syncthreads();
#pragma unroll 4
        for (int q = warp; q < nc; q += kCtaWarps) {
            const uint32_t mq = S.cmask[q];
            if ((mq >> lane) & 1u) S.chain[S.coff[q] + __popc(mq & below)] = __ldcg(ad + static_cast<int64_t>(c0 + q) * 32 + lane);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int k = 0;
            for (; k + 4 <= total; k += 4) {
                const double x0 = S.chain[k], x1 = S.chain[k + 1], x2 = S.chain[k + 2], x3 = S.chain[k + 3];
                sum += x0;
                sum += x1;
                sum += x2;
                sum += x3;
            }
            for (; k < total; ++k) sum += S.chain[k];
        }
        __syncthreads();
    }
    return sum;
}

// The miss budget over one round's ballots (kCtaWords words, word w covering
// points base + 32 w ..): returns the round's miss count (every thread); when
// misses + count exceeds the budget, warp 0 sets `visited` to the reference's
// visit count (its (budget + 1)-th miss, registration.cpp:211-214).
__device__ __forceinline__ int round_misses(const uint32_t* __restrict__ words, int64_t base, int64_t misses,
                                            const ScoreParams& sp, int64_t& visited) {
    const int lane = threadIdx.x & 31;
    unsigned c = 0;
#pragma unroll
    for (int w = lane; w < kCtaWords; w += 32) c += __popc(words[w]);
    const int total = static_cast<int>(__reduce_add_sync(kFull, c));
    if (misses + total > sp.miss_budget && (threadIdx.x >> 5) == 0) {
        int64_t before = misses;
        for (int h = 0; h < kCtaWords / 32; ++h) {
            const uint32_t mw = words[h * 32 + lane];
            const int cnt = __popc(mw);
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(kFull, incl, o);
                if (lane >= o) incl += y;
            }
            const unsigned over = __ballot_sync(kFull, before + incl > sp.miss_budget);
            if (over) {
                const int L = __ffs(over) - 1;
                const int64_t bef = before + __shfl_sync(kFull, incl - cnt, L);
                unsigned m = __shfl_sync(kFull, mw, L);
                const int need = static_cast<int>(sp.miss_budget - bef);
                for (int q = 0; q < need; ++q) m &= m - 1;
                visited = base + static_cast<int64_t>(h * 32 + L) * 32 + (__ffs(m) - 1) + 1;
                break;
            }
            before += __shfl_sync(kFull, incl, 31);
        }
    }
    return total;
}

// Phases A and B of one round of kCtaPts points starting at `base` for the
// candidate staged in S (R, t, Rf, F): FP32 location, the shared-memory queue
// and its dense FP64-exact resolution. Leaves the round's ballots in S.inl[b] /
// S.miss[b], the inliers' d2 in add[i] and their (any-order) sum in `part`;
// clears the other parity's ballots; ends with a block barrier.
__device__ __forceinline__ void score_round_ab(CtaSmem& S, const SourceView& src, const GridView& g,
                                               const ScoreParams& sp, const double* cand_rt_c, int64_t base, int b,
                                               int64_t ns, double* __restrict__ add, double& part) {
    const int lane = threadIdx.x & 31;
    const FastRT& F = S.F;
    if (threadIdx.x == 0) S.next = 0;
    // A. FP32 location of the round's points
#pragma unroll
    for (int u = 0; u < kCtaPer; ++u) {
        const int local = u * kCtaThreads + threadIdx.x;
        const int64_t i = base + local;
        int state = 0;  // 0 certain miss, 1 exact fallback, 2 fine-list scan
        int2 bi = make_int2(0, 0);
        if (i < ns) {
            if (F.ok == 0.0f) {
                state = 1;
            } else {
                const float4 P = __ldg(src.pos32 + i);
                const float qx = fmaf(F.r[0], P.x, fmaf(F.r[1], P.y, fmaf(F.r[2], P.z, F.t[0])));
                const float qy = fmaf(F.r[3], P.x, fmaf(F.r[4], P.y, fmaf(F.r[5], P.z, F.t[1])));
                const float qz = fmaf(F.r[6], P.x, fmaf(F.r[7], P.y, fmaf(F.r[8], P.z, F.t[2])));
                const float eps = F.eps;
                if (!(qx < -eps || qy < -eps || qz < -eps || qx >= g.fnx + eps || qy >= g.fny + eps ||
                      qz >= g.fnz + eps)) {
                    const float fx = floorf(qx), fy = floorf(qy), fz = floorf(qz);
                    const float rx = qx - fx, ry = qy - fy, rz = qz - fz;
                    if (rx < eps || rx > 1.0f - eps || ry < eps || ry > 1.0f - eps || rz < eps ||
                        rz > 1.0f - eps) {
                        state = 1;
                    } else {
                        const int ix = static_cast<int>(fx), iy = static_cast<int>(fy),
                                  iz = static_cast<int>(fz);
                        if (ix >= 0 && iy >= 0 && iz >= 0 && ix < g.fnx && iy < g.fny && iz < g.fnz) {
                            bi = __ldg(g.fine_info + (static_cast<int64_t>(ix) * g.fny + iy) * g.fnz + iz);
                            if (bi.y > 0) state = bi.y < kCtaSlow ? 2 : 1;
                        }
                    }
                }
            }
        }
        const unsigned mm = __ballot_sync(kFull, i < ns && state == 0);
        if (lane == 0) S.miss[b][local >> 5] = mm;
        // list scans from the front of q, exact fallbacks from the back; B
        // hands out the (rare, slow) fallbacks first and together, so they
        // share warp chunks with each other and do not end up in the tail
        const unsigned mf = __ballot_sync(kFull, state == 2), ms = __ballot_sync(kFull, state == 1);
        int slot = 0;
        if (mf) {
            const int leader = __ffs(mf) - 1;
            if (lane == leader) slot = atomicAdd(&S.nq[b], __popc(mf));
            slot = __shfl_sync(kFull, slot, leader) + __popc(mf & ((1u << lane) - 1u));
        }
        if (ms) {
            const int leader = __ffs(ms) - 1;
            int sl = 0;
            if (lane == leader) sl = atomicAdd(&S.nslow[b], __popc(ms));
            sl = __shfl_sync(kFull, sl, leader) + __popc(ms & ((1u << lane) - 1u));
            if (state == 1) slot = kCtaPts - 1 - sl;
        }
        if (state != 0) S.q[slot] = make_int2(local | ((state == 1 ? kCtaSlow : bi.y) << 16), bi.x);
    }
    __syncthreads();
    // B. dense resolution of the queue; the next round's ballots are cleared
    const int nslow = S.nslow[b], nq = S.nq[b] + nslow;
    if (threadIdx.x == 0) {
        S.nq[b ^ 1] = 0;
        S.nslow[b ^ 1] = 0;
    }
    if (threadIdx.x < kCtaWords) {
        S.inl[b ^ 1][threadIdx.x] = 0u;
        S.miss[b ^ 1][threadIdx.x] = 0u;
    }
    // warps take the queue 32 entries at a time: a warp with slow entries
    // (long lists, the exact fallback) takes fewer chunks, so the round's
    // barrier waits less for the slowest thread
    for (int first = 1;; first = 0) {
        // each warp's first chunk is its own (no atomic round trip), the rest
        // are handed out in order of demand
        int e0 = (threadIdx.x >> 5) * 32;
        if (!first) {
            if (lane == 0) e0 = kCtaThreads + atomicAdd(&S.next, 32);
            e0 = __shfl_sync(kFull, e0, 0);
        }
        if (e0 >= nq) break;
        const int e = e0 + lane;
        if (e >= nq) continue;
        const int2 qe = S.q[e < nslow ? kCtaPts - 1 - e : e - nslow];
        const int local = qe.x & 0xffff;
        const int cnt = static_cast<int>(static_cast<unsigned>(qe.x) >> 16);
        const int64_t i = base + local;
        double addend = 0.0;
        bool inl;
        if (cnt == kCtaSlow) {
            inl = eval_point_slow(g, cand_rt_c, src, i, sp, &addend);
        } else {
            const float4 P = __ldg(src.pos32 + i);
            const float qx = fmaf(F.r[0], P.x, fmaf(F.r[1], P.y, fmaf(F.r[2], P.z, F.t[0])));
            const float qy = fmaf(F.r[3], P.x, fmaf(F.r[4], P.y, fmaf(F.r[5], P.z, F.t[1])));
            const float qz = fmaf(F.r[6], P.x, fmaf(F.r[7], P.y, fmaf(F.r[8], P.z, F.t[2])));
            const bool rec = src.pos4 != nullptr && src.nrm32 != nullptr;
            const V3 p = rec ? ld4(src.pos4, i) : ld3(src.pos, i);
            const float4 n32 = rec ? __ldg(src.nrm32 + i) : make_float4(0, 0, 0, 0);
            inl = resolve_fine(g, S.R, S.t, rec ? S.Rf : nullptr, F, src, i, p, n32, qx, qy, qz, qe.y, cnt,
                               sp, addend);
        }
        const int word = local >> 5;  // ballot word w covers points base + 32 w ..
        const uint32_t bit = 1u << (local & 31);
        if (inl) {
            atomicOr(&S.inl[b][word], bit);
            add[i] = addend;
            part += addend;
        } else {
            atomicOr(&S.miss[b][word], bit);
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void cta_body(CtaSmem& S, const SourceView& src, const GridView& g, const ScoreParams& sp,
                                         const double* __restrict__ cand_rt, const int64_t* __restrict__ cand_index,
                                         int64_t sampled, int64_t ns_pad, double* __restrict__ scr_add,
                                         uint32_t* __restrict__ scr_inl, Counters* __restrict__ ctr,
                                         BestRec* __restrict__ block_best, RecordDev* __restrict__ rec,
                                         int64_t unit_cap, int64_t unit_threshold, int n_prev_best) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n_cand = static_cast<int64_t>(ctr->n_candidates);
    // the candidates k_score_units did not take (same rule as there)
    const int64_t cand_begin = n_cand >= unit_threshold ? 0 : (n_cand < unit_cap ? n_cand : unit_cap);
    const int64_t ns = src.n;
    const int32_t n_chunks = static_cast<int32_t>(ns_pad / 32);
    // the CTA's two scratch slots: addends (ns_pad) and ballot words (n_chunks)
    double* slot_add[2] = {scr_add + (2 * static_cast<int64_t>(blockIdx.x)) * ns_pad,
                           scr_add + (2 * static_cast<int64_t>(blockIdx.x) + 1) * ns_pad};
    uint32_t* slot_inl[2] = {scr_inl + (2 * static_cast<int64_t>(blockIdx.x)) * n_chunks,
                             scr_inl + (2 * static_cast<int64_t>(blockIdx.x) + 1) * n_chunks};
    int cur = 0;  // slot of the candidate in progress; the best lives in 1 - cur
    // thread 0's books: the CTA best (fitness exact when best_eb == 0)
    BestRec best{0, 0, 0.0, INT64_MAX, -1};
    double best_eb = 0.0;
    unsigned long long t_qual = 0, t_wref = 0, t_exec = 0;
    for (;;) {
        if (threadIdx.x == 0) S.cand = cand_begin + static_cast<int64_t>(atomicAdd(&ctr->work_next2, 1ull));
        if (threadIdx.x < 2 * kCtaWords) {
            (&S.inl[0][0])[threadIdx.x] = 0u;
            (&S.miss[0][0])[threadIdx.x] = 0u;
        }
        __syncthreads();
        const int64_t cand = S.cand;
        if (cand >= n_cand) break;
        if (threadIdx.x < 12) {
            const double v = __ldg(cand_rt + 12 * cand + threadIdx.x);
            if (threadIdx.x < 9) {
                S.R[threadIdx.x] = v;
                S.Rf[threadIdx.x] = static_cast<float>(v);
            } else {
                S.t[threadIdx.x - 9] = v;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            S.F = make_fast_fine(S.R, S.t, g, sp);
            S.nq[0] = S.nq[1] = 0;
            S.nslow[0] = S.nslow[1] = 0;
        }
        __syncthreads();
        double* add = slot_add[cur];
        uint32_t* inlw = slot_inl[cur];
        double part = 0.0;
        int64_t misses = 0, inliers = 0, visited = ns, done = ns;
        bool exited = false;
        for (int64_t base = 0, r = 0; base < ns; base += kCtaPts, ++r) {
            const int b = static_cast<int>(r & 1);
            score_round_ab(S, src, g, sp, cand_rt + 12 * cand, base, b, ns, add, part);
            // C. the miss budget in point order (word w covers points base + 32 w ..)
            const int rm = round_misses(S.miss[b], base, misses, sp, visited);
            if (misses + rm > sp.miss_budget) {
                exited = true;
                const int64_t end = base + kCtaPts;
                done = end < ns ? end : ns;
                break;
            }
            misses += rm;
            if (warp == 0) {
                unsigned pop = 0;
#pragma unroll
                for (int w = lane; w < kCtaWords; w += 32) {
                    const uint32_t iw = S.inl[b][w];
                    if (base / 32 + w < n_chunks) inlw[base / 32 + w] = iw;
                    pop += __popc(iw);
                }
                inliers += __reduce_add_sync(kFull, pop);
            }
        }
        // the candidate's verdict (thread 0 decides, the CTA runs exact chains on demand)
        if (!exited) {
            double v = part;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
            if (lane == 0) S.red[warp] = v;
        }
        __syncthreads();
        int need = 0;  // bit 0: chain the candidate, bit 1: chain the best
        double fit = 0.0, eb = 0.0;
        bool qual_sure = false;
        if (threadIdx.x == 0) {
            t_wref += static_cast<unsigned long long>(visited);
            t_exec += static_cast<unsigned long long>(done);
            if (!exited) {
                const double ratio = static_cast<double>(inliers) / static_cast<double>(ns);
                if (!(ratio < sp.min_ratio)) {
                    double s = 0.0;
                    for (int w = 0; w < kCtaWarps; ++w) s += S.red[w];
                    fit = inliers > 0 ? s / static_cast<double>(inliers) : 0.0;
                    eb = inliers > 0 ? order_bound(inliers) * fit : 0.0;
                    const bool may = !(fit - eb > sp.max_fitness);
                    qual_sure = fit + eb <= sp.max_fitness;
                    if (may) {
                        need |= 16;
                        if (!qual_sure) need |= 1;
                        if (best.valid && inliers == best.inliers && fabs(fit - best.fitness) <= eb + best_eb) {
                            need |= 1;
                            if (best_eb != 0.0) need |= 2;
                        }
                    }
                }
            }
            S.flag = need;
            S.swap = 0;
        }
        __syncthreads();
        need = S.flag;
        if (need & 1) {
            const double s = cta_chain(inlw, add, n_chunks, S);
            if (threadIdx.x == 0) S.exact[0] = s;
        }
        if (need & 2) {
            const double s = cta_chain(slot_inl[1 - cur], slot_add[1 - cur], n_chunks, S);
            if (threadIdx.x == 0) S.exact[1] = s;
        }
        __syncthreads();
        if (threadIdx.x == 0 && (need & 16)) {
            if (need & 2) {
                best.fitness = S.exact[1] / static_cast<double>(best.inliers);
                best_eb = 0.0;
            }
            bool qual = qual_sure;
            if (need & 1) {
                fit = S.exact[0] / static_cast<double>(inliers);
                eb = 0.0;
                qual = !(fit > sp.max_fitness);
            }
            if (qual) {
                t_qual += 1;
                const BestRec c{1, inliers, fit, __ldg(cand_index + cand), cand};
                bool take;
                if (!best.valid || inliers != best.inliers) take = !best.valid || inliers > best.inliers;
                else if (eb == 0.0 && best_eb == 0.0) take = better(c, best);
                else take = fit < best.fitness;  // bounds disjoint (else both were chained)
                if (take) {
                    best = c;
                    best_eb = eb;
                    S.swap = 1;  // the candidate's slot becomes the best's
                }
            }
        }
        __syncthreads();
        if (S.swap) cur = 1 - cur;
        __syncthreads();
    }
    // the CTA best's exact sum
    if (threadIdx.x == 0) S.flag = (best.valid && best_eb != 0.0) ? 1 : 0;
    __syncthreads();
    if (S.flag) {
        const double s = cta_chain(slot_inl[1 - cur], slot_add[1 - cur], n_chunks, S);
        if (threadIdx.x == 0) best.fitness = s / static_cast<double>(best.inliers);
    }
    // publish the CTA's tallies and best; the last CTA writes the record
    __shared__ unsigned long long s_ticket;
    if (threadIdx.x == 0) {
        if (t_qual) atomicAdd(&ctr->qualified, t_qual);
        if (t_wref) atomicAdd(&ctr->w_ref, t_wref);
        if (t_exec) atomicAdd(&ctr->evals_executed, t_exec);
        block_best[n_prev_best + blockIdx.x] = best;
        __threadfence();
        s_ticket = atomicAdd(&ctr->fin_done, 1ull);
    }
    __syncthreads();
    if (s_ticket != gridDim.x - 1) return;
    __threadfence();
    // every CTA best: the unit scorer's (before) and this kernel's
    BestRec b{0, 0, 0.0, INT64_MAX, -1};
    for (int i = threadIdx.x; i < n_prev_best + static_cast<int>(gridDim.x); i += blockDim.x) {
        BestRec c;
        c.valid = __ldcg(&block_best[i].valid);
        c.inliers = __ldcg(&block_best[i].inliers);
        c.fitness = __ldcg(&block_best[i].fitness);
        c.index = __ldcg(&block_best[i].index);
        c.slot = __ldcg(&block_best[i].slot);
        if (better(c, b)) b = c;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        BestRec c;
        c.valid = __shfl_down_sync(kFull, b.valid, o);
        c.inliers = __shfl_down_sync(kFull, b.inliers, o);
        c.fitness = __shfl_down_sync(kFull, b.fitness, o);
        c.index = __shfl_down_sync(kFull, b.index, o);
        c.slot = __shfl_down_sync(kFull, b.slot, o);
        if (better(c, b)) b = c;
    }
    __shared__ BestRec s_red[kCtaWarps];
    if (lane == 0) s_red[warp] = b;
    __syncthreads();
    if (threadIdx.x != 0) return;
    for (int w = 1; w < kCtaWarps; ++w)
        if (better(s_red[w], b)) b = s_red[w];
    RecordDev r{};
    r.valid = b.valid;
    r.inliers = b.valid ? b.inliers : 0;
    r.fitness = b.valid ? b.fitness : 0.0;
    r.index = b.valid ? b.index : -1;
    for (int q = 0; q < 9; ++q) r.R[q] = b.valid ? cand_rt[12 * b.slot + q] : 0.0;
    for (int q = 0; q < 3; ++q) r.t[q] = b.valid ? cand_rt[12 * b.slot + 9 + q] : 0.0;
    r.sampled = sampled;
    r.prerejected = sampled - static_cast<int64_t>(__ldcg(&ctr->n_survivors));
    r.degenerate = static_cast<int64_t>(__ldcg(&ctr->degenerate));
    r.evaluated = n_cand;
    r.qualified = static_cast<int64_t>(__ldcg(&ctr->qualified));
    r.w_ref = static_cast<int64_t>(__ldcg(&ctr->w_ref));
    r.evals_executed = static_cast<int64_t>(__ldcg(&ctr->evals_executed));
    *rec = r;
}

// ---- round-unit scoring ----------------------------------------------------
// Work unit = (candidate, round of kCtaPts points), taken candidate-major from
// a ticket counter by a persistent grid, so a heavy candidate (nearly every
// point pending) spreads over many CTAs instead of serialising on one -- the
// balance that strong scaling over ranks needs. A unit runs phases A and B of
// the candidate-CTA scorer, then publishes its ballots (per candidate, per
// 32-point word), its inliers' d2 and its partial sum (atomic, any order). The
// CTA that completes a candidate's last unit applies the miss budget in point
// order over the published ballots (exit => the reference's visit count), and
// decides qualification and the comparison with its CTA best by the order
// bound, running the reference's sequential sum (registration.cpp:206) on
// demand; every CTA best ends exact (registration.cpp:272-276). Candidates
// beyond the scratch capacity go to k_score_cta, which writes the record.
__device__ __forceinline__ void units_body(CtaSmem& S, const SourceView& src, const GridView& g,
                                           const ScoreParams& sp, const double* __restrict__ cand_rt,
                                           const int64_t* __restrict__ cand_index, int64_t cap, int64_t ns_pad,
                                           uint32_t* __restrict__ u_miss, uint32_t* __restrict__ u_inl,
                                           double* __restrict__ u_add, double* __restrict__ u_sum,
                                           unsigned* __restrict__ u_done, Counters* __restrict__ ctr,
                                           BestRec* __restrict__ block_best, int64_t unit_threshold) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n_all = static_cast<int64_t>(ctr->n_candidates);
    // units only pay when candidates are too few to keep a CTA each busy
    // (strong scaling over ranks); otherwise k_score_cta takes them all
    const int64_t n_cand = n_all >= unit_threshold ? 0 : (n_all < cap ? n_all : cap);
    const int64_t ns = src.n;
    const int32_t n_chunks = static_cast<int32_t>(ns_pad / 32);
    const int64_t R = (ns + kUnitPts - 1) / kUnitPts;  // units per candidate
    const int64_t n_units = n_cand * R;
    // thread 0's books: the CTA best (fitness exact when best_eb == 0)
    BestRec best{0, 0, 0.0, INT64_MAX, -1};
    double best_eb = 0.0;
    unsigned long long t_qual = 0, t_wref = 0, t_exec = 0;
    for (;;) {
        if (threadIdx.x == 0) {
            S.cand = static_cast<int64_t>(atomicAdd(&ctr->work_next, 1ull));
            S.nq[0] = S.nq[1] = 0;
            S.nslow[0] = S.nslow[1] = 0;
        }
        if (threadIdx.x < kCtaWords) {
            S.inl[0][threadIdx.x] = 0u;
            S.miss[0][threadIdx.x] = 0u;
        }
        __syncthreads();
        const int64_t u = S.cand;
        if (u >= n_units) break;
        // round-major tickets: every candidate's first unit, then the second,
        // ... so a late round usually finds its candidate's earlier rounds done
        const int64_t r = u / n_cand, c = u - r * n_cand;
        const int64_t base = r * kUnitPts;
        const int64_t ns_u = base + kUnitPts < ns ? base + kUnitPts : ns;  // the unit's end
        // u_done: unit count in bits 0-15, completed rounds (r < 16) above.
        // When rounds 0..r-1 are complete and already hold more misses than the
        // budget, the reference's exit lies before this unit: it is skipped
        // (the verdict finds the exit in those rounds' ballots).
        const unsigned inc = 1u + (r < 16 ? (1u << (16 + r)) : 0u);
        if (warp == 0) {
            int skip = 0;
            if (r > 0 && r < 16 && sp.miss_budget != INT64_MAX) {
                const unsigned need = ((1u << r) - 1u) << 16;
                unsigned st = 0;
                if (lane == 0) st = __ldcg(u_done + c);
                st = __shfl_sync(kFull, st, 0);
                if ((st & need) == need) {
                    __threadfence();
                    int64_t misses = 0;
                    const int32_t wend = static_cast<int32_t>(base / 32);
                    for (int32_t w = lane; w < wend; w += 32) misses += __popc(__ldcg(u_miss + c * n_chunks + w));
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) misses += __shfl_xor_sync(kFull, misses, o);
                    skip = misses > sp.miss_budget ? 1 : 0;
                }
            }
            if (lane == 0) S.swap = skip;
        }
        __syncthreads();
        if (S.swap) {
            if (threadIdx.x == 0) S.flag = (atomicAdd(u_done + c, inc) & 0xffffu) == static_cast<unsigned>(R - 1) ? 1 : 0;
            __syncthreads();
            if (!S.flag) continue;
        } else {
        if (threadIdx.x < 12) {
            const double v = __ldg(cand_rt + 12 * c + threadIdx.x);
            if (threadIdx.x < 9) {
                S.R[threadIdx.x] = v;
                S.Rf[threadIdx.x] = static_cast<float>(v);
            } else {
                S.t[threadIdx.x - 9] = v;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) S.F = make_fast_fine(S.R, S.t, g, sp);
        __syncthreads();
        double part = 0.0;
        double* add = u_add + c * ns_pad;
        score_round_ab(S, src, g, sp, cand_rt + 12 * c, base, 0, ns_u, add, part);
        // publish the round: ballots, the partial sum, then the unit count
        const int32_t w0 = static_cast<int32_t>(base / 32);
        if (threadIdx.x < kUnitPts / 32 && w0 + static_cast<int32_t>(threadIdx.x) < n_chunks) {
            u_miss[c * n_chunks + w0 + threadIdx.x] = S.miss[0][threadIdx.x];
            u_inl[c * n_chunks + w0 + threadIdx.x] = S.inl[0][threadIdx.x];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(kFull, part, o);
        if (lane == 0) S.red[warp] = part;
        __syncthreads();
        if (threadIdx.x == 0) {
            double sum = 0.0;
            for (int w = 0; w < kCtaWarps; ++w) sum += S.red[w];
            if (sum != 0.0) atomicAdd(u_sum + c, sum);
        }
        if (threadIdx.x == 0) t_exec += static_cast<unsigned long long>(ns_u - base);
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) S.flag = (atomicAdd(u_done + c, inc) & 0xffffu) == static_cast<unsigned>(R - 1) ? 1 : 0;
        __syncthreads();
        if (!S.flag) continue;
        }
        // ---- the candidate's last unit: its verdict
        __threadfence();
        const uint32_t* mw_c = u_miss + c * n_chunks;
        const uint32_t* iw_c = u_inl + c * n_chunks;
        if (warp == 0) {
            int64_t misses = 0, visited = ns;
            unsigned pop = 0;
            bool exited = false;
            for (int32_t s0 = 0; s0 < n_chunks; s0 += 32) {
                const int32_t w = s0 + lane;
                const uint32_t mw = w < n_chunks ? __ldcg(mw_c + w) : 0u;
                pop += w < n_chunks ? __popc(__ldcg(iw_c + w)) : 0u;
                if (exited) continue;
                const int cnt = __popc(mw);
                int incl = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o) incl += y;
                }
                const unsigned over = __ballot_sync(kFull, misses + incl > sp.miss_budget);
                if (over) {
                    const int L = __ffs(over) - 1;
                    const int64_t before = misses + __shfl_sync(kFull, incl - cnt, L);
                    unsigned m = __shfl_sync(kFull, mw, L);
                    const int need = static_cast<int>(sp.miss_budget - before);
                    for (int q = 0; q < need; ++q) m &= m - 1;
                    visited = static_cast<int64_t>(s0 + L) * 32 + (__ffs(m) - 1) + 1;
                    exited = true;
                }
                misses += __shfl_sync(kFull, incl, 31);
            }
            const int64_t inliers = static_cast<int64_t>(__reduce_add_sync(kFull, pop));
            if (lane == 0) {
                S.exact[0] = static_cast<double>(visited);
                S.exact[1] = static_cast<double>(inliers);
                S.swap = exited ? 1 : 0;
            }
        }
        __syncthreads();
        const bool exited = S.swap != 0;
        const int64_t visited = static_cast<int64_t>(S.exact[0]);
        const int64_t inliers = static_cast<int64_t>(S.exact[1]);
        int need = 0;  // bit 0: chain the candidate, bit 1: chain the best, bit 4: a qualifying verdict
        double fit = 0.0, eb = 0.0;
        bool qual_sure = false;
        if (threadIdx.x == 0) {
            t_wref += static_cast<unsigned long long>(visited);
            if (!exited) {
                const double ratio = static_cast<double>(inliers) / static_cast<double>(ns);
                if (!(ratio < sp.min_ratio)) {
                    const double s = __ldcg(u_sum + c);
                    fit = inliers > 0 ? s / static_cast<double>(inliers) : 0.0;
                    eb = inliers > 0 ? order_bound(inliers) * fit : 0.0;
                    const bool may = !(fit - eb > sp.max_fitness);
                    qual_sure = fit + eb <= sp.max_fitness;
                    if (may) {
                        need |= 16;
                        if (!qual_sure) need |= 1;
                        if (best.valid && inliers == best.inliers && fabs(fit - best.fitness) <= eb + best_eb) {
                            need |= 1;
                            if (best_eb != 0.0) need |= 2;
                        }
                    }
                }
            }
            S.flag = need;
        }
        __syncthreads();
        need = S.flag;
        if (need & 1) {
            const double s = cta_chain(iw_c, u_add + c * ns_pad, n_chunks, S);
            if (threadIdx.x == 0) S.exact[0] = s;
        }
        if (need & 2) {
            const double s = cta_chain(u_inl + best.slot * n_chunks, u_add + best.slot * ns_pad, n_chunks, S);
            if (threadIdx.x == 0) S.exact[1] = s;
        }
        __syncthreads();
        if (threadIdx.x == 0 && (need & 16)) {
            if (need & 2) {
                best.fitness = S.exact[1] / static_cast<double>(best.inliers);
                best_eb = 0.0;
            }
            bool qual = qual_sure;
            if (need & 1) {
                fit = S.exact[0] / static_cast<double>(inliers);
                eb = 0.0;
                qual = !(fit > sp.max_fitness);
            }
            if (qual) {
                t_qual += 1;
                const BestRec cb{1, inliers, fit, __ldg(cand_index + c), c};
                bool take;
                if (!best.valid || inliers != best.inliers) take = !best.valid || inliers > best.inliers;
                else if (eb == 0.0 && best_eb == 0.0) take = better(cb, best);
                else take = fit < best.fitness;  // bounds disjoint (else both were chained)
                if (take) {
                    best = cb;
                    best_eb = eb;
                }
            }
        }
        __syncthreads();
    }
    // every warp has read the final ticket from S.cand before it is reused
    __syncthreads();
    // the CTA best's exact sum (its scratch rows persist)
    if (threadIdx.x == 0) {
        S.flag = (best.valid && best_eb != 0.0) ? 1 : 0;
        S.cand = best.slot;
    }
    __syncthreads();
    if (S.flag) {
        const int64_t bs = S.cand;
        const double s = cta_chain(u_inl + bs * n_chunks, u_add + bs * ns_pad, n_chunks, S);
        if (threadIdx.x == 0) best.fitness = s / static_cast<double>(best.inliers);
    }
    if (threadIdx.x == 0) {
        if (t_qual) atomicAdd(&ctr->qualified, t_qual);
        if (t_wref) atomicAdd(&ctr->w_ref, t_wref);
        if (t_exec) atomicAdd(&ctr->evals_executed, t_exec);
        block_best[blockIdx.x] = best;
    }
}

// The scorer of run_hypotheses, two launches: k_score_units takes round units
// while the candidates are too few to keep a CTA each busy (a rank's share
// under strong scaling) and exits at once otherwise; k_score_cta then takes
// one CTA per candidate for the rest and writes the rank record. Separate
// kernels keep each body's register allocation.
__global__ void __launch_bounds__(kCtaThreads, 4) k_score_units(SourceView src, const __grid_constant__ GridView g,
                                                                 const __grid_constant__ ScoreParams sp,
                                                                 const double* __restrict__ cand_rt,
                                                                 const int64_t* __restrict__ cand_index,
                                                                 int64_t unit_cap, int64_t unit_ns_pad,
                                                                 uint32_t* __restrict__ u_miss,
                                                                 uint32_t* __restrict__ u_inl,
                                                                 double* __restrict__ u_add,
                                                                 double* __restrict__ u_sum,
                                                                 unsigned* __restrict__ u_done,
                                                                 Counters* __restrict__ ctr,
                                                                 BestRec* __restrict__ block_best,
                                                                 int64_t unit_threshold) {
    __shared__ CtaSmem S;
    if (static_cast<int64_t>(ctr->n_candidates) >= unit_threshold) {
        if (threadIdx.x == 0) block_best[blockIdx.x] = BestRec{0, 0, 0.0, INT64_MAX, -1};
        return;
    }
    units_body(S, src, g, sp, cand_rt, cand_index, unit_cap, unit_ns_pad, u_miss, u_inl, u_add, u_sum, u_done, ctr,
               block_best, unit_threshold);
}

__global__ void __launch_bounds__(kCtaThreads, 5) k_score_cta(SourceView src, const __grid_constant__ GridView g,
                                                               const __grid_constant__ ScoreParams sp,
                                                               const double* __restrict__ cand_rt,
                                                               const int64_t* __restrict__ cand_index,
                                                               int64_t sampled, int64_t cta_ns_pad,
                                                               double* __restrict__ scr_add,
                                                               uint32_t* __restrict__ scr_inl, int64_t unit_cap,
                                                               Counters* __restrict__ ctr,
                                                               BestRec* __restrict__ block_best,
                                                               RecordDev* __restrict__ rec, int64_t unit_threshold,
                                                               int n_unit_best) {
    __shared__ CtaSmem S;
    cta_body(S, src, g, sp, cand_rt, cand_index, sampled, cta_ns_pad, scr_add, scr_inl, ctr, block_best, rec,
             unit_cap, unit_threshold, n_unit_best);
}

// ---- explicit candidate lists (evaluate_hypothesis / evaluate_against_grid
// per candidate, registration.cpp:53-78 / 155-219) over an EvalGrid with fine
// lists: one CTA per candidate (persistent grid, ticket), rounds as in the
// candidate-CTA scorer, and the candidate's sum run in point order by warp 0
// round by round (every per-candidate fitness is the reference's own sum);
// the last CTA writes the record of the best (registration.cpp:272-276).
__global__ void __launch_bounds__(kCtaThreads, 4) k_score_list(SourceView src, const __grid_constant__ GridView g,
                                                                const __grid_constant__ ScoreParams sp,
                                                                const double* __restrict__ cand_rt, int64_t C,
                                                                int64_t* __restrict__ out_inliers,
                                                                double* __restrict__ out_sum,
                                                                double* __restrict__ scratch,
                                                                Counters* __restrict__ ctr,
                                                                BestRec* __restrict__ block_best,
                                                                RecordDev* __restrict__ rec) {
    __shared__ CtaSmem S;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t ns = src.n;
    double* my_add = scratch + static_cast<int64_t>(blockIdx.x) * kCtaPts;
    WarpTally wt;  // thread 0's books
    for (;;) {
        if (threadIdx.x == 0) {
            S.cand = static_cast<int64_t>(atomicAdd(&ctr->work_next, 1ull));
            S.nq[0] = S.nq[1] = 0;
            S.nslow[0] = S.nslow[1] = 0;
        }
        if (threadIdx.x < 2 * kCtaWords) {
            (&S.inl[0][0])[threadIdx.x] = 0u;
            (&S.miss[0][0])[threadIdx.x] = 0u;
        }
        __syncthreads();
        const int64_t cand = S.cand;
        if (cand >= C) break;
        if (threadIdx.x < 12) {
            const double v = __ldg(cand_rt + 12 * cand + threadIdx.x);
            if (threadIdx.x < 9) {
                S.R[threadIdx.x] = v;
                S.Rf[threadIdx.x] = static_cast<float>(v);
            } else {
                S.t[threadIdx.x - 9] = v;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) S.F = make_fast_fine(S.R, S.t, g, sp);
        __syncthreads();
        double part = 0.0, sum = 0.0;
        int64_t misses = 0, inliers = 0, visited = ns, done = ns;
        bool exited = false;
        for (int64_t base = 0, r = 0; base < ns; base += kCtaPts, ++r) {
            const int b = static_cast<int>(r & 1);
            score_round_ab(S, src, g, sp, cand_rt + 12 * cand, base, b, ns, my_add - base, part);
            // the miss budget in point order (word w covers points base + 32 w ..)
            const int rm = round_misses(S.miss[b], base, misses, sp, visited);
            if (misses + rm > sp.miss_budget) {
                exited = true;
                const int64_t end = base + kCtaPts;
                done = end < ns ? end : ns;
                break;
            }
            misses += rm;
            // this round's inliers' d2 in point order onto the candidate's sum
            if (warp == 0) {
                const unsigned below = (1u << lane) - 1u;
                int off = 0;
                for (int w = 0; w < kCtaWords; ++w) {
                    const uint32_t m = S.inl[b][w];
                    if ((m >> lane) & 1u) S.chain[off + __popc(m & below)] = my_add[w * 32 + lane];
                    off += __popc(m);
                }
                inliers += off;
                __syncwarp();
                if (lane == 0) {
                    int k = 0;
                    for (; k + 4 <= off; k += 4) {
                        const double x0 = S.chain[k], x1 = S.chain[k + 1], x2 = S.chain[k + 2], x3 = S.chain[k + 3];
                        sum += x0;
                        sum += x1;
                        sum += x2;
                        sum += x3;
                    }
                    for (; k < off; ++k) sum += S.chain[k];
                }
            }
            __syncthreads();  // S.chain aliases the next round's queue
        }
        if (threadIdx.x == 0) {
            out_inliers[cand] = exited ? -1 : inliers;
            out_sum[cand] = exited ? 0.0 : sum;
            wt.w_ref += static_cast<unsigned long long>(visited);
            wt.executed += static_cast<unsigned long long>(done);
            if (!exited) wt.candidate(inliers, sum, ns, sp, cand, cand);
        }
        __syncthreads();
    }
    // publish_cta folds lane 0 of every warp: only warp 0 carries the books
    if (threadIdx.x != 0) wt = WarpTally{};
    const bool last = publish_cta(wt, ctr, block_best, blockIdx.x, true);
    if (last) write_record(block_best, gridDim.x, cand_rt, C, C, ctr, rec);
}

// Explicit lists on a dense EvalGrid target (its fine lists too long to scan):
// the same per-candidate rounds, every point answered by the ring grid
// (lk_ring.cuh: the reference EvalGrid's neighbour within d_max), then the
// normal gate in FP64 (registration.cpp:200-210). Ballots come straight from
// the warps; the sum runs in point order round by round.
// Each round's points are queried in their Morton order (order: per-round
// permutation of the source, spatial_order_blocks) so that a warp's queries
// share ring cells (ring_nn_warp); verdicts land in the round's bit words by
// original index, so the round logic is unchanged.
__global__ void __launch_bounds__(kCtaThreads, 3) k_score_list_ring(SourceView src, const __grid_constant__ RingGrid rg,
                                                                     const int32_t* __restrict__ order,
                                                                     const double* __restrict__ tnrm,
                                                                     const __grid_constant__ ScoreParams sp,
                                                                     const double* __restrict__ cand_rt, int64_t C,
                                                                     int64_t* __restrict__ out_inliers,
                                                                     double* __restrict__ out_sum,
                                                                     double* __restrict__ scratch,
                                                                     Counters* __restrict__ ctr,
                                                                     BestRec* __restrict__ block_best,
                                                                     RecordDev* __restrict__ rec) {
    __shared__ CtaSmem S;
    __shared__ float4 s_buf[kCtaWarps][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t ns = src.n;
    double* my_add = scratch + static_cast<int64_t>(blockIdx.x) * kCtaPts;
    WarpTally wt;  // thread 0's books
    for (;;) {
        if (threadIdx.x == 0) S.cand = static_cast<int64_t>(atomicAdd(&ctr->work_next, 1ull));
        __syncthreads();
        const int64_t cand = S.cand;
        if (cand >= C) break;
        if (threadIdx.x < 12) {
            const double v = __ldg(cand_rt + 12 * cand + threadIdx.x);
            if (threadIdx.x < 9) S.R[threadIdx.x] = v;
            else S.t[threadIdx.x - 9] = v;
        }
        __syncthreads();
        double sum = 0.0;
        int64_t misses = 0, inliers = 0, visited = ns, done = ns;
        bool exited = false;
        for (int64_t base = 0; base < ns; base += kCtaPts) {
            if (threadIdx.x < kCtaWords) {
                S.inl[0][threadIdx.x] = 0u;
                S.miss[0][threadIdx.x] = 0u;
            }
            if (threadIdx.x == 0) S.next = 0;
            __syncthreads();
            // warps take the round's 32-point Morton runs dynamically: walk
            // costs vary by run, so static shares leave warps at the barrier
#pragma unroll 1
            for (;;) {
                int run = 0;
                if (lane == 0) run = atomicAdd(&S.next, 1);
                run = __shfl_sync(0xffffffffu, run, 0);
                if (run >= kCtaPts / 32) break;
                const int64_t t = base + run * 32 + lane;
                const bool act = t < ns;
                const int64_t i = act ? static_cast<int64_t>(__ldg(order + t)) : 0;
                const int local = static_cast<int>(i - base);
                V3 y = mk(0.0, 0.0, 0.0);
                if (act) y = xform(S.R, S.t, src.pos4 ? ld4(src.pos4, i) : ld3(src.pos, i));
                const int32_t j = ring_nn_warp(rg, y, sp.d2_max, act, s_buf[warp]);  // warp-uniform call
                bool inl = false;
                if (j >= 0) {
                    const V3 ns_ = ld3(src.nrm, i);
                    const V3 nt = ld3(tnrm, j);
                    if (!is_zero(ns_) && !is_zero(nt) && dot(rot(S.R, ns_), nt) >= sp.cos_max) {
                        inl = true;
                        my_add[local] = sqnorm(sub(ld4(rg.pos4, j), y));
                    }
                }
                if (act) atomicOr(inl ? &S.inl[0][local >> 5] : &S.miss[0][local >> 5], 1u << (local & 31));
            }
            __syncthreads();
            const int rm = round_misses(S.miss[0], base, misses, sp, visited);
            if (misses + rm > sp.miss_budget) {
                exited = true;
                const int64_t end = base + kCtaPts;
                done = end < ns ? end : ns;
                break;
            }
            misses += rm;
            if (warp == 0) {
                const unsigned below = (1u << lane) - 1u;
                int off = 0;
                for (int w = 0; w < kCtaWords; ++w) {
                    const uint32_t m = S.inl[0][w];
                    if ((m >> lane) & 1u) S.chain[off + __popc(m & below)] = my_add[w * 32 + lane];
                    off += __popc(m);
                }
                inliers += off;
                __syncwarp();
                if (lane == 0) {
                    int k = 0;
                    for (; k + 4 <= off; k += 4) {
                        const double x0 = S.chain[k], x1 = S.chain[k + 1], x2 = S.chain[k + 2], x3 = S.chain[k + 3];
                        sum += x0;
                        sum += x1;
                        sum += x2;
                        sum += x3;
                    }
                    for (; k < off; ++k) sum += S.chain[k];
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            out_inliers[cand] = exited ? -1 : inliers;
            out_sum[cand] = exited ? 0.0 : sum;
            wt.w_ref += static_cast<unsigned long long>(visited);
            wt.executed += static_cast<unsigned long long>(done);
            if (!exited) wt.candidate(inliers, sum, ns, sp, cand, cand);
        }
        __syncthreads();
    }
    if (threadIdx.x != 0) wt = WarpTally{};
    const bool last = publish_cta(wt, ctr, block_best, blockIdx.x, true);
    if (last) write_record(block_best, gridDim.x, cand_rt, C, C, ctr, rec);
}

int blocks_per_sm(const void* fn) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kScoreThreads, 0) != cudaSuccess || b < 1) b = 1;
    return b;
}

int score_blocks_per_sm() {
    static int cached = 0;
    if (!cached) cached = blocks_per_sm(reinterpret_cast<const void*>(k_score));
    return cached;
}

int cand_blocks_per_sm() {
    static int cached = 0;
    if (!cached) cached = blocks_per_sm(reinterpret_cast<const void*>(k_score_cta));
    return cached;
}

}  // namespace

void RunBuffers::release() {
    pool_free(surv_index, stream);
    pool_free(surv_ids, stream);
    pool_free(cand_index, stream);
    pool_free(cand_rt, stream);
    pool_free(counters, stream);
    pool_free(block_best, stream);
    pool_free(cand_fast, stream);
    pool_free(cta_add, stream);
    pool_free(cta_inl, stream);
    pool_free(u_miss, stream);
    pool_free(u_inl, stream);
    pool_free(u_add, stream);
    pool_free(u_sum, stream);
    pool_free(u_done, stream);
    u_miss = u_inl = nullptr;
    u_add = u_sum = nullptr;
    u_done = nullptr;
    u_cap = u_ns_pad = 0;
    cta_add = nullptr;
    cta_inl = nullptr;
    cta_slots = 0;
    cta_ns_pad = 0;
    cand_fast = nullptr;
    fast_capacity = 0;
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
    if (!counters && (e = pool_alloc(&counters, sizeof(Counters), stream)) != cudaSuccess) return e;
    if (score_blocks > n_blocks) {
        pool_free(block_best, stream);
        if ((e = pool_alloc(&block_best, score_blocks * sizeof(BestRec), stream)) != cudaSuccess) return e;
        n_blocks = score_blocks;
    }
    if (cap > capacity) {
        pool_free(surv_index, stream);
        pool_free(surv_ids, stream);
        pool_free(cand_index, stream);
        pool_free(cand_rt, stream);
        surv_index = nullptr;
        surv_ids = nullptr;
        cand_index = nullptr;
        cand_rt = nullptr;
        capacity = 0;
        if ((e = pool_alloc(&surv_index, cap * sizeof(int64_t), stream)) != cudaSuccess) return e;
        if ((e = pool_alloc(&surv_ids, cap * 8 * sizeof(int32_t), stream)) != cudaSuccess) return e;
        if ((e = pool_alloc(&cand_index, cap * sizeof(int64_t), stream)) != cudaSuccess) return e;
        if ((e = pool_alloc(&cand_rt, cap * 12 * sizeof(double), stream)) != cudaSuccess) return e;
        capacity = cap;
    }
    return cudaSuccess;
}

cudaError_t RunBuffers::ensure_cta(int64_t ns, int32_t n_ctas) {
    const int64_t ns_pad = (ns + 31) / 32 * 32;
    if (n_ctas <= cta_slots && ns_pad == cta_ns_pad) return cudaSuccess;
    pool_free(cta_add, stream);
    pool_free(cta_inl, stream);
    pool_free(u_miss, stream);
    pool_free(u_inl, stream);
    pool_free(u_add, stream);
    pool_free(u_sum, stream);
    pool_free(u_done, stream);
    u_miss = u_inl = nullptr;
    u_add = u_sum = nullptr;
    u_done = nullptr;
    u_cap = u_ns_pad = 0;
    cta_add = nullptr;
    cta_inl = nullptr;
    cta_slots = 0;
    cudaError_t e;
    if ((e = pool_alloc(&cta_add, 2 * static_cast<int64_t>(n_ctas) * ns_pad * sizeof(double), stream)) != cudaSuccess)
        return e;
    if ((e = pool_alloc(&cta_inl, 2 * static_cast<int64_t>(n_ctas) * (ns_pad / 32) * sizeof(uint32_t), stream)) !=
        cudaSuccess)
        return e;
    cta_slots = n_ctas;
    cta_ns_pad = ns_pad;
    return cudaSuccess;
}

cudaError_t RunBuffers::ensure_units(int64_t ns, int64_t cap) {
    const int64_t ns_pad = (ns + 31) / 32 * 32;
    if (cap <= u_cap && ns_pad == u_ns_pad) return cudaSuccess;
    pool_free(u_miss, stream);
    pool_free(u_inl, stream);
    pool_free(u_add, stream);
    pool_free(u_sum, stream);
    pool_free(u_done, stream);
    u_miss = u_inl = nullptr;
    u_add = u_sum = nullptr;
    u_done = nullptr;
    u_cap = 0;
    const int64_t words = cap * (ns_pad / 32);
    cudaError_t e;
    if ((e = pool_alloc(&u_miss, words * sizeof(uint32_t), stream)) != cudaSuccess) return e;
    if ((e = pool_alloc(&u_inl, words * sizeof(uint32_t), stream)) != cudaSuccess) return e;
    if ((e = pool_alloc(&u_add, cap * ns_pad * sizeof(double), stream)) != cudaSuccess) return e;
    if ((e = pool_alloc(&u_sum, cap * sizeof(double), stream)) != cudaSuccess) return e;
    if ((e = pool_alloc(&u_done, cap * sizeof(unsigned), stream)) != cudaSuccess) return e;
    u_cap = cap;
    u_ns_pad = ns_pad;
    return cudaSuccess;
}

cudaError_t RunBuffers::ensure_fast(int64_t n) {
    if (n <= fast_capacity) return cudaSuccess;
    pool_free(cand_fast, stream);
    cand_fast = nullptr;
    fast_capacity = 0;
    cudaError_t e = pool_alloc(&cand_fast, n * sizeof(FastRT), stream);
    if (e == cudaSuccess) fast_capacity = n;
    return e;
}

cudaError_t run_hypotheses_range(const SourceView& src, const double* d_tgt_pos, const int32_t* d_cache,
                                 const GridView& grid, const ScoreParams& sp, uint64_t seed, double tau, int64_t begin,
                                 int64_t end, RunBuffers& rb, void* d_record, cudaStream_t stream, int sm_count,
                                 cudaEvent_t* events) {
    const int64_t count = end - begin;
    const int cand_blocks = sm_count * cand_blocks_per_sm();
    cudaError_t e = rb.ensure(count > 0 ? count : 1, 2 * cand_blocks);
    if (e != cudaSuccess) return e;
    if ((e = rb.ensure_cta(src.n, cand_blocks)) != cudaSuccess) return e;
    {
        // unit scratch: a few percent of the hypotheses survive; at most 2 GiB of addends
        const int64_t ns_pad = (src.n + 31) / 32 * 32;
        int64_t ucap = count / 64 > 4096 ? count / 64 : 4096;
        const int64_t byte_cap = (int64_t(2) << 30) / (ns_pad * static_cast<int64_t>(sizeof(double)));
        if (ucap > byte_cap) ucap = byte_cap > 1 ? byte_cap : 1;
        if ((e = rb.ensure_units(src.n, ucap)) != cudaSuccess) return e;
    }
    if ((e = cudaMemsetAsync(rb.counters, 0, sizeof(Counters), stream)) != cudaSuccess) return e;
    const uint32_t ns = static_cast<uint32_t>(src.n);
    const uint32_t thresh = static_cast<uint32_t>(0x100000000ull % ns);
    if (events) cudaEventRecord(events[0], stream);
    if (count > 0) {
        int64_t want = (count + 255) / 256;
        unsigned gs = static_cast<unsigned>(want < sm_count * 16 ? want : sm_count * 16);
        PrefetchList pf{};
        auto add = [&](const void* ptr, int64_t bytes) {
            // 16-byte aligned start (allocations are), whole 16-byte granules
            if (ptr && bytes >= 16 && pf.n < PrefetchList::kMax) {
                pf.ptr[pf.n] = static_cast<const char*>(ptr);
                pf.bytes[pf.n] = static_cast<unsigned long long>(bytes);
                ++pf.n;
            }
        };
        add(grid.fine_info, grid.n_fine * static_cast<int64_t>(sizeof(int2)));
        add(grid.fine_pts, grid.n_fine_entries * static_cast<int64_t>(sizeof(float4)));
        add(grid.pos4_orig, grid.n_points * static_cast<int64_t>(sizeof(double4)));
        add(grid.nrm32_orig, grid.n_points * static_cast<int64_t>(sizeof(float4)));
        add(src.pos32, src.n * static_cast<int64_t>(sizeof(float4)));
        add(src.pos4, src.n * static_cast<int64_t>(sizeof(double4)));
        add(src.nrm32, src.n * static_cast<int64_t>(sizeof(float4)));
        if (static_cast<int64_t>(gs) < pf.n) pf.n = static_cast<int>(gs);
        // measured on B1: the scoring gathers hit L2 without it and the bulk
        // DRAM reads slow k_hyp_sample, so it is opt-in (LK_PREFETCH=1)
        if (const char* v = std::getenv("LK_PREFETCH"); !(v && v[0] == '1')) pf.n = 0;
        k_hyp_sample<<<gs, 256, 0, stream>>>(begin, count, splitmix64(seed), ns, thresh, d_cache, src.pos, d_tgt_pos,
                                             tau, rb.surv_index, rb.surv_ids, rb.counters, pf);
    }
    if (events) cudaEventRecord(events[1], stream);
    if (count > 0) {
        k_kabsch<<<sm_count * 8, 32, 0, stream>>>(src.pos, d_tgt_pos, rb.surv_index, rb.surv_ids, rb.cand_index,
                                                   rb.cand_rt, rb.counters, rb.u_sum, rb.u_done, rb.u_cap);
    }
    if (events) cudaEventRecord(events[2], stream);
    // candidate-CTA scoring: one persistent kernel, record included
    if (events) cudaEventRecord(events[3], stream);
    // few candidates (a rank's share under strong scaling): units for the
    // first u_cap, the candidate-CTA scorer for the rest; many: the
    // candidate-CTA scorer for all. The latter writes the record.
    int64_t unit_threshold = 2 * static_cast<int64_t>(cand_blocks);
    if (const char* v = std::getenv("LK_SCORE_UNITS"); v && v[0] == '1') unit_threshold = INT64_MAX;
    if (const char* v = std::getenv("LK_SCORE_UNITS"); v && v[0] == '0') unit_threshold = 0;
    k_score_units<<<cand_blocks, kCtaThreads, 0, stream>>>(src, grid, sp, rb.cand_rt, rb.cand_index, rb.u_cap,
                                                          rb.u_ns_pad, rb.u_miss, rb.u_inl, rb.u_add, rb.u_sum,
                                                          rb.u_done, rb.counters, rb.block_best, unit_threshold);
    k_score_cta<<<cand_blocks, kCtaThreads, 0, stream>>>(src, grid, sp, rb.cand_rt, rb.cand_index, count,
                                                        rb.cta_ns_pad, rb.cta_add, rb.cta_inl, rb.u_cap, rb.counters,
                                                        rb.block_best, static_cast<RecordDev*>(d_record),
                                                        unit_threshold, cand_blocks);
    if (events) {
        cudaEventRecord(events[4], stream);
        cudaEventRecord(events[5], stream);
        cudaEventRecord(events[6], stream);
    }
    return cudaGetLastError();
}

cudaError_t score_candidates(const SourceView& src, const GridView& grid, const ScoreParams& sp, const double* d_rt,
                             int64_t C, RunBuffers& rb, int64_t* d_out_inliers, double* d_out_sum, void* d_record,
                             cudaStream_t stream, int sm_count, const RingGrid* ring) {
    if (ring && !sp.fitness_from_distance) {
        // dense EvalGrid target: ring-grid queries, CTA per candidate
        const int blocks = sm_count * blocks_per_sm(reinterpret_cast<const void*>(k_score_list_ring));
        cudaError_t e = rb.ensure(1, blocks);
        if (e != cudaSuccess) return e;
        if ((e = rb.ensure_cta(kCtaPts, blocks)) != cudaSuccess) return e;
        if ((e = cudaMemsetAsync(rb.counters, 0, sizeof(Counters), stream)) != cudaSuccess) return e;
        int32_t* order = nullptr;
        if ((e = pool_alloc(&order, (src.n > 0 ? src.n : 1) * sizeof(int32_t), stream)) != cudaSuccess) return e;
        if (src.n > 0 && (e = spatial_order_blocks(src.pos, src.n, kCtaPts, order, stream)) != cudaSuccess) {
            pool_free(order, stream);
            return e;
        }
        k_score_list_ring<<<blocks, kCtaThreads, 0, stream>>>(src, *ring, order, grid.nrm_orig, sp, d_rt, C,
                                                              d_out_inliers, d_out_sum, rb.cta_add, rb.counters,
                                                              rb.block_best, static_cast<RecordDev*>(d_record));
        e = cudaGetLastError();
        pool_free(order, stream);
        return e;
    }
    if (grid.fine_info && sp.fast && !sp.fitness_from_distance) {
        // EvalGrid with fine lists: CTA per candidate over rounds
        const int blocks = sm_count * cand_blocks_per_sm();
        cudaError_t e = rb.ensure(1, blocks);
        if (e != cudaSuccess) return e;
        if ((e = rb.ensure_cta(kCtaPts, blocks)) != cudaSuccess) return e;  // kCtaPts doubles per CTA
        if ((e = cudaMemsetAsync(rb.counters, 0, sizeof(Counters), stream)) != cudaSuccess) return e;
        k_score_list<<<blocks, kCtaThreads, 0, stream>>>(src, grid, sp, d_rt, C, d_out_inliers, d_out_sum, rb.cta_add,
                                                         rb.counters, rb.block_best,
                                                         static_cast<RecordDev*>(d_record));
        return cudaGetLastError();
    }
    const int blocks = sm_count * score_blocks_per_sm();
    cudaError_t e = rb.ensure(1, blocks);
    if (e != cudaSuccess) return e;
    if ((e = rb.ensure_fast(C > 0 ? C : 1)) != cudaSuccess) return e;
    FastRT* cand_fast = static_cast<FastRT*>(rb.cand_fast);
    if ((e = cudaMemsetAsync(rb.counters, 0, sizeof(Counters), stream)) != cudaSuccess) return e;
    if (C > 0) k_prep_fast<<<sm_count * 2, 128, 0, stream>>>(d_rt, C, rb.counters, grid, sp, cand_fast);
    k_score<<<blocks, kScoreThreads, 0, stream>>>(src, grid, sp, d_rt, cand_fast, nullptr, 0, C, C, d_out_inliers,
                                                  d_out_sum,
                                                  rb.counters, rb.block_best, 0, static_cast<RecordDev*>(d_record));
    return cudaGetLastError();
}

}  // namespace lkk
