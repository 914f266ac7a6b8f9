// lk_prepare.cu -- prepare_registration on the device.
//
// voxel_downsample (proj/src/preprocess.cpp:14-59):
//   k_vox_insert   voxel key floor(p / leaf) per point into an open-addressing
//                  hash table; per voxel: first input index (atomicMin), count
//   k_vox_mark     flag the first index of every voxel; an exclusive scan of
//                  the flags gives each voxel its output position, which is the
//                  reference's order (voxels sorted by first input index)
//   k_vox_keys     (output voxel, input index) pairs; a stable radix sort
//                  (cub::DeviceRadixSort) groups members by voxel in input order
//   k_vox_reduce   warp per voxel: the reference's sequential FP64 sums in
//                  input order (lane-0 chain over shuffled members) and the
//                  normalised normal
// compute_fpfh (proj/src/fpfh.cpp:57-141):
//   neighbour lists within r (SearchGrid cell = r, ascending, self excluded),
//   k_spfh    warp per point: pair-angle votes as integer counts; pairs whose
//             frame-source test (std::acos comparison) the device cannot
//             decide, or whose theta (atan2) lies at a bin edge, are deferred
//             to the host's libm (host_pair_bins, k_spfh_resolve_a/b), then
//             k_spfh_scale applies fl(100 / votes) like `v *= 100.0 / votes`
//   k_fpfh    warp per point, lane per bin: acc_b += spfh_j[b] / w_j over the
//             neighbours in ascending order (the reference's summation order)
// Temporaries come from the stream's Scratch buffer and initialisation is
// folded into the first kernel that runs: few stream commands per call (each
// costs the device front end several us while the other cloud's upload holds
// the PCIe link, tools/launch_under_dma.cu).
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "lk_device_math.cuh"
#include "lk_eig3.hpp"
#include "lk_acos_cr.hpp"
#include "lk_kernels.cuh"

namespace lkk {

using namespace lkd;

namespace {

constexpr unsigned long long kEmpty = ~0ull;
constexpr unsigned kFull = 0xffffffffu;

inline unsigned nblocks(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

__device__ __forceinline__ int floor_cell(double q) {
    double f = floor(q);
    if (!(f >= -2147483648.0 && f < 2147483648.0)) return INT32_MIN;
    return static_cast<int>(f);
}

// proj/src/preprocess.cpp:25-29 (pack of grid_index(p, 0, leaf))
__device__ __forceinline__ unsigned long long voxel_key(const double* p, double leaf) {
    const long long off = 1 << 20;
    unsigned long long x = static_cast<unsigned long long>(floor_cell((p[0] - 0.0) / leaf) + off);
    unsigned long long y = static_cast<unsigned long long>(floor_cell((p[1] - 0.0) / leaf) + off);
    unsigned long long z = static_cast<unsigned long long>(floor_cell((p[2] - 0.0) / leaf) + off);
    return (x << 42) | (y << 21) | z;
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k;
}

// the table and the flags to their empty state, the flag scan's leading 0
__global__ void k_vox_init(uint32_t table, int64_t n, unsigned long long* __restrict__ keys,
                           int32_t* __restrict__ first, int32_t* __restrict__ count, int32_t* __restrict__ flags,
                           int32_t* __restrict__ flag_scan, int* __restrict__ bad,
                           unsigned long long* __restrict__ stats) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < table; i += stride) {
        keys[i] = kEmpty;
        first[i] = 0x7f7f7f7f;
        count[i] = 0;
    }
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) flags[i] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        flag_scan[0] = 0;
        *bad = 0;
        stats[0] = stats[1] = 0;
    }
}

// nrm (optional): validate_cloud's normal check (proj/src/geometry.cpp:93-103:
// unit within 1e-6 or exactly zero) on the same pass
__global__ void k_vox_insert(const double* __restrict__ pos, const double* __restrict__ nrm, int64_t n, double leaf,
                             unsigned long long* keys, uint32_t mask, int32_t* __restrict__ point_slot, int32_t* first,
                             int32_t* count, int* __restrict__ bad) {
    int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    if (nrm) {
        const V3 v = ld3(nrm, i);
        const double len = sqrt(sqnorm(v));
        if (len != 0.0 && fabs(len - 1.0) > 1e-6) atomicOr(bad, 1);
    }
    const unsigned long long key = voxel_key(pos + 3 * i, leaf);
    uint32_t h = static_cast<uint32_t>(mix64(key)) & mask;
    while (true) {
        unsigned long long prev = atomicCAS(&keys[h], kEmpty, key);
        if (prev == kEmpty || prev == key) break;
        h = (h + 1) & mask;
    }
    point_slot[i] = static_cast<int32_t>(h);
    atomicMin(&first[h], static_cast<int32_t>(i));
    atomicAdd(&count[h], 1);
}

__global__ void k_vox_mark(const unsigned long long* __restrict__ keys, const int32_t* __restrict__ first,
                           uint32_t table, int32_t* __restrict__ flags) {
    uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h < table && keys[h] != kEmpty) flags[first[h]] = 1;
}

__global__ void k_vox_out(const unsigned long long* __restrict__ keys, const int32_t* __restrict__ first,
                          const int32_t* __restrict__ count, uint32_t table, const int32_t* __restrict__ flag_scan,
                          int32_t* __restrict__ slot_out, int32_t* __restrict__ cnt_out,
                          int32_t* __restrict__ member_start) {
    uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= table || keys[h] == kEmpty) return;
    const int32_t o = flag_scan[first[h]];
    slot_out[h] = o;
    cnt_out[o] = count[h];
    if (o == 0) member_start[0] = 0;  // the member scan's leading 0
}

// sort keys for the members: each point's output voxel, value = its index
__global__ void k_vox_keys(const int32_t* __restrict__ point_slot, int64_t n, const int32_t* __restrict__ slot_out,
                           int32_t* __restrict__ keys, int32_t* __restrict__ vals) {
    int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    keys[i] = slot_out[point_slot[i]];
    vals[i] = static_cast<int32_t>(i);
}

// Sorts seg[0..k) ascending with the 32 lanes of a warp: in shared memory
// (bitonic network) when k <= cap, else in place by lane 0 (rare, slow, exact).
// Returns the sorted array to read (shared buffer or seg itself).
__device__ int32_t* warp_sort_segment(int32_t* seg, int k, int32_t* sbuf, int cap) {
    const int lane = threadIdx.x & 31;
    if (k <= cap) {
        int P = 1;
        while (P < k) P <<= 1;
        for (int a = lane; a < P; a += 32) sbuf[a] = a < k ? seg[a] : INT32_MAX;
        __syncwarp();
        for (int size = 2; size <= P; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int t = lane; t < (P >> 1); t += 32) {
                    const int i = 2 * stride * (t / stride) + (t % stride);
                    const int j = i + stride;
                    const bool up = (i & size) == 0;
                    const int32_t a = sbuf[i], b = sbuf[j];
                    if ((a > b) == up) {
                        sbuf[i] = b;
                        sbuf[j] = a;
                    }
                }
                __syncwarp();
            }
        }
        return sbuf;
    }
    if (lane == 0) {
        for (int a = 1; a < k; ++a) {
            int32_t v = seg[a];
            int b = a - 1;
            while (b >= 0 && seg[b] > v) {
                seg[b + 1] = seg[b];
                --b;
            }
            seg[b + 1] = v;
        }
    }
    __syncwarp();
    return seg;
}

constexpr int kSortWarps = 4;
constexpr int kSortCap = 2048;

// proj/src/preprocess.cpp:30-58, warp per voxel: members sorted by input
// index, then the sums in that order (lane order within 32-member chunks).
// A skipped (zero) normal contributes +0.0, which leaves the sum unchanged.
// stats (optional, zeroed by k_vox_init): cloud_stats of the output -- usable
// normals and max |p|, k_cloud_stats' arithmetic on the stored values --
// one atomic pair per block, so the prepare needs no separate stats pass.
__global__ void __launch_bounds__(32 * kSortWarps) k_vox_reduce(const int32_t* __restrict__ members,
                                                                const int32_t* __restrict__ member_start, int64_t n_out,
                                                                const double* __restrict__ pos,
                                                                const double* __restrict__ nrm,
                                                                double* __restrict__ out_pos,
                                                                double* __restrict__ out_nrm,
                                                                unsigned long long* __restrict__ stats) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t o = blockIdx.x * static_cast<int64_t>(kSortWarps) + warp;
    __shared__ double s_v[kSortWarps][6][32];
    __shared__ unsigned long long s_usable[kSortWarps], s_max[kSortWarps];
    unsigned long long usable = 0, max_bits = 0;
    if (o < n_out) {
        const int32_t s0 = member_start[o], s1 = member_start[o + 1];
        const int k = s1 - s0;
        const int32_t* sorted = members + s0;  // ascending input index (stable radix sort)
        // lanes gather 32 members at a time (the next chunk's loads in flight
        // while lane 0 runs the sequential sums over the current one from smem)
        auto fetch = [&](int c0, V3& p, V3& nv) {
            p = mk(0.0, 0.0, 0.0);
            nv = mk(0.0, 0.0, 0.0);
            if (c0 + lane < k) {
                const int64_t i = sorted[c0 + lane];
                p = ld3(pos, i);
                if (nrm) {
                    nv = ld3(nrm, i);
                    if (is_zero(nv)) nv = mk(0.0, 0.0, 0.0);
                }
            }
        };
        // lane q < 6 runs component q's sequential chain (x, y, z of the
        // positions, then of the normals): six chains side by side
        double acc = 0.0;
        V3 p, nv;
        // chunk c + 2's members pulled into L1 while chunk c + 1 is loaded
        // into registers (their indices loaded one iteration earlier)
        auto l1_prefetch = [&](int j) {
            asm volatile("prefetch.global.L1 [%0];" ::"l"(pos + 3 * static_cast<int64_t>(j)));
            if (nrm) asm volatile("prefetch.global.L1 [%0];" ::"l"(nrm + 3 * static_cast<int64_t>(j)));
        };
        int32_t ahead = 64 + lane < k ? sorted[64 + lane] : -1;
        fetch(0, p, nv);
        for (int c0 = 0; c0 < k; c0 += 32) {
            if (ahead >= 0) l1_prefetch(ahead);
            ahead = c0 + 96 + lane < k ? sorted[c0 + 96 + lane] : -1;
            s_v[warp][0][lane] = p.x;
            s_v[warp][1][lane] = p.y;
            s_v[warp][2][lane] = p.z;
            s_v[warp][3][lane] = nv.x;
            s_v[warp][4][lane] = nv.y;
            s_v[warp][5][lane] = nv.z;
            __syncwarp();
            if (c0 + 32 < k) fetch(c0 + 32, p, nv);
            if (lane < 6) {
                const int m = k - c0 < 32 ? k - c0 : 32;
                const double* col = s_v[warp][lane];
#pragma unroll 8
                for (int L = 0; L < m; ++L) acc += col[L];
            }
            __syncwarp();
        }
        const V3 ps = mk(__shfl_sync(kFull, acc, 0), __shfl_sync(kFull, acc, 1), __shfl_sync(kFull, acc, 2));
        const V3 nsum = mk(__shfl_sync(kFull, acc, 3), __shfl_sync(kFull, acc, 4), __shfl_sync(kFull, acc, 5));
        if (lane == 0) {
            const double cnt = static_cast<double>(k);
            const double x = ps.x / cnt, y = ps.y / cnt, z = ps.z / cnt;
            out_pos[3 * o] = x;
            out_pos[3 * o + 1] = y;
            out_pos[3 * o + 2] = z;
            const double r = sqrt(x * x + y * y + z * z);
            if (r == r) max_bits = static_cast<unsigned long long>(__double_as_longlong(r));  // fmax drops NaN
            if (nrm) {
                const double len = sqrt(sqnorm(nsum));
                V3 nn = mk(0.0, 0.0, 0.0);
                if (len > 1e-12) nn = mk(nsum.x / len, nsum.y / len, nsum.z / len);
                out_nrm[3 * o] = nn.x;
                out_nrm[3 * o + 1] = nn.y;
                out_nrm[3 * o + 2] = nn.z;
                usable = is_zero(nn) ? 0 : 1;
            }
        }
    }
    if (!stats) return;
    if (lane == 0) {
        s_usable[warp] = usable;
        s_max[warp] = max_bits;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long u = 0, m = 0;
        for (int w = 0; w < kSortWarps; ++w) {
            u += s_usable[w];
            m = s_max[w] > m ? s_max[w] : m;
        }
        atomicAdd(&stats[0], u);
        atomicMax(&stats[1], m);  // non-negative doubles order like their bit patterns
    }
}

// ---- FPFH --------------------------------------------------------------------

__device__ __forceinline__ V3 cross(V3 a, V3 b) {
    return mk(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}

// The reference's frame-source test is acos(|a1|) > acos(|a2|) evaluated with
// the host libm's acos, which is not correctly rounded but within 0.522 ulp
// (lk_acos_cr.hpp). When |a1| and |a2| are more than 2.5e-16 apart the libm
// values are certainly ordered like the arguments (acos is decreasing with
// |slope| >= 1 and ulp(acos) <= 2.22e-16 on [0, pi/2], so the exact values
// are more than 2 x 0.522 ulp apart). Closer pairs -- common on noisy planar
// faces, where normals agree to the last bits -- go to list A: k_spfh_decide_a
// settles those whose outcome does not depend on how glibc rounds near a
// midpoint (lk_acos_cr.hpp), the rest (~5 % of the ties) are decided on the
// host with the reference's libm (compute_fpfh below). Returns 0 no swap,
// 1 swap, 2 undecided.
__device__ __forceinline__ int swap_decision(double x1, double x2) {
    if (!(x1 <= 1.0 && x2 <= 1.0)) return 0;  // acos of |a| > 1 is NaN: never greater
    if (fabs(x1 - x2) > 2.5e-16) return x1 < x2 ? 1 : 0;
    if (x1 == x2) return 0;
    return 2;
}

// proj/src/fpfh.cpp:50-53
__device__ __forceinline__ int bin_index(double value, double lo, double hi) {
    int b = floor_cell(11 * (value - lo) / (hi - lo));
    return b < 0 ? 0 : (b > 10 ? 10 : b);
}

// proj/src/fpfh.cpp:17-48, split at the frame-source test: pair_setup forms
// d, dist and the two cosines; pair_bins finishes the Darboux frame for a
// given test outcome and returns the three histogram bins (false = no vote).
struct PairSetup {
    V3 d;
    double dist, a1, a2;
};
__device__ __forceinline__ bool pair_setup(V3 p1, V3 n1, V3 p2, V3 n2, PairSetup& s) {
    s.d = sub(p2, p1);
    s.dist = sqrt(sqnorm(s.d));
    if (s.dist <= 0.0) return false;
    s.a1 = dot(n1, s.d) / s.dist;
    s.a2 = dot(n2, s.d) / s.dist;
    return true;
}
// theta = atan2(w.nt, u.nt) comes from CUDA's atan2 (<= 2 ulp) where the
// reference uses glibc's; its bin floor(11 (theta + pi) / 2 pi) is decided
// here only when that value is more than 1e-12 from an inner bin edge (the
// two libms put it within ~1e-14 of each other); otherwise theta_edge is set
// and the pair goes to the host (k_spfh's deferred list). Most pairs are
// settled by an FP32 atan2 with a 1e-4 margin before any FP64 atan2. alpha and phi are
// plain IEEE arithmetic, identical on both sides.
__device__ __forceinline__ bool pair_bins(const PairSetup& s, V3 n1, V3 n2, int swap, int3& bins, bool& theta_edge) {
    V3 ns = n1, nt = n2, line = s.d;
    double cos_line = s.a1;
    if (swap == 1) {
        ns = n2;
        nt = n1;
        line = mk(-s.d.x, -s.d.y, -s.d.z);
        cos_line = -s.a2;
    }
    V3 u = ns;
    V3 v = cross(line, u);
    double v_len = sqrt(sqnorm(v));
    theta_edge = false;
    if (v_len <= 1e-12 * s.dist) return false;
    v = mk(v.x / v_len, v.y / v_len, v.z / v_len);
    V3 w = cross(u, v);
    const double alpha = dot(v, nt);
    const double phi = cos_line;
    const double ty = dot(w, nt), tx = dot(u, nt);
    // theta's bin from FP32 first: its tv is within 1e-5 of the exact value
    // (atan2f, the float rounding of tx and ty -- both normal floats near an
    // inner edge, where |sin|, |cos| >= 0.14 -- and the float arithmetic), so
    // more than 1e-4 from every integer it is the bin of glibc's theta too,
    // and not within 1e-12 of an inner edge. Otherwise the FP64 path below.
    const double m = fmax(fabs(tx), fabs(ty));
    int tb = -1;
    if (m >= 1e-30 && m <= 1e30) {
        const float tf = atan2f(static_cast<float>(ty), static_cast<float>(tx));
        const float tvf = 11.0f * (tf + 3.14159265f) / 6.28318531f;
        if (fabsf(tvf - rintf(tvf)) > 1e-4f) {
            const int b = static_cast<int>(floorf(tvf));
            tb = b < 0 ? 0 : (b > 10 ? 10 : b);
            theta_edge = false;
        }
    }
    if (tb < 0) {
        const double theta = atan2(ty, tx);
        const double tv = 11 * (theta - -M_PI) / (M_PI - -M_PI);
        const double edge = rint(tv);
        theta_edge = edge >= 1.0 && edge <= 10.0 && fabs(tv - edge) < 1e-12;
        tb = bin_index(theta, -M_PI, M_PI);
    }
    bins = make_int3(bin_index(alpha, -1.0, 1.0), 11 + bin_index(phi, -1.0, 1.0), 22 + tb);
    return true;
}

// neighbours within r (inclusive), self excluded (proj/src/fpfh.cpp:66-74)
// warp per point: lanes over the slots of each cell row, ballot counts
__global__ void __launch_bounds__(32 * kSortWarps) k_nbr_count(const double* __restrict__ pos, int64_t n, GridView g,
                                                               double r2, int32_t* __restrict__ counts) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i = blockIdx.x * static_cast<int64_t>(kSortWarps) + warp;
    if (i >= n) return;
    const V3 p = ld3(pos, i);
    const int kx = floor_cell((p.x - g.ox) / g.cell) - g.offx;
    const int ky = floor_cell((p.y - g.oy) / g.cell) - g.offy;
    const int kz = floor_cell((p.z - g.oz) / g.cell) - g.offz;
    int32_t c = 0;
    for (int x = max(kx - g.radius, 0); x <= min(kx + g.radius, g.nx - 1); ++x)
        for (int y = max(ky - g.radius, 0); y <= min(ky + g.radius, g.ny - 1); ++y) {
            const int64_t row = (static_cast<int64_t>(x) * g.ny + y) * g.nz;
            const int32_t s0 = g.start[row + max(kz - g.radius, 0)];
            const int32_t s1 = g.start[row + min(kz + g.radius, g.nz - 1) + 1];
            for (int32_t b = s0; b < s1; b += 32) {
                const int32_t s = b + lane;
                const bool hit = s < s1 && g.index[s] != i && sqnorm(sub(ld3(g.slot_pos, s), p)) <= r2;
                c += __popc(__ballot_sync(kFull, hit));
            }
        }
    if (lane == 0) counts[i] = c;
}

// Small clouds: radius_search by a warp-per-point scan of the whole cloud in
// index order (ascending output, no grid, no sort). A pair counts when the
// reference's SearchGrid would visit it -- cells (floor(p / cell), center 0)
// within the block radius of the query's -- and d2 <= r2, so the lists equal
// the grid's to the bit even where rounding puts a point within r two cells away.
constexpr int64_t kBruteMax = 24576;

// Cells packed 10 bits per axis (mod 1024: x 22-31, y 11-20, z 0-9) with
// guard bits 10 and 21 set: for a query key ki (guards clear),
//   t = (((kj | G) - ki) & ~G) + ONE
// holds (dc + 1) mod 1024 in each field without carries between fields, and
// (t & kCellNearMask) == 0 iff every dc mod 1024 is in {-1, 0, 1, 2} -- a
// superset of the block-radius-1 test, which the exact int4 test then
// decides. Four ALU operations per pair instead of a dozen.
constexpr uint32_t kCellGuards = (1u << 10) | (1u << 21);
constexpr uint32_t kCellOne = 1u | (1u << 11) | (1u << 22);
constexpr uint32_t kCellNearMask = (0x3fcu << 22) | (0x3fcu << 11) | 0x3fcu;
__device__ __forceinline__ uint32_t pack_cell(int4 c) {
    return ((static_cast<uint32_t>(c.x) & 1023u) << 22) | ((static_cast<uint32_t>(c.y) & 1023u) << 11) |
           (static_cast<uint32_t>(c.z) & 1023u);
}
__device__ __forceinline__ bool cell_near(uint32_t kj_guarded, uint32_t ki) {
    return ((((kj_guarded - ki) & ~kCellGuards) + kCellOne) & kCellNearMask) == 0;
}

// zero (optional): off[0], the deferred-list counts and the overflow flag;
// keys (optional): the packed cells with their guard bits
__global__ void k_search_cells(const double* __restrict__ pos, int64_t n, double cell, int4* __restrict__ out,
                               int32_t* __restrict__ off = nullptr, int32_t* __restrict__ n_def = nullptr,
                               int32_t* __restrict__ overflow = nullptr, uint32_t* __restrict__ keys = nullptr) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i == 0 && off) {
        off[0] = 0;
        n_def[0] = n_def[1] = n_def[2] = n_def[3] = 0;
        *overflow = 0;
    }
    if (i >= n) return;
    const int4 c = make_int4(floor_cell((pos[3 * i] - 0.0) / cell), floor_cell((pos[3 * i + 1] - 0.0) / cell),
                             floor_cell((pos[3 * i + 2] - 0.0) / cell), 0);
    out[i] = c;
    if (keys) keys[i] = pack_cell(c) | kCellGuards;
}

template <bool kFill>
__global__ void __launch_bounds__(32 * kSortWarps) k_nbr_brute(const double* __restrict__ pos,
                                                               const int4* __restrict__ cells, int64_t n, int rad,
                                                               double r2, int32_t* __restrict__ counts,
                                                               const int32_t* __restrict__ off,
                                                               int32_t* __restrict__ nbr, int64_t cap) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i = blockIdx.x * static_cast<int64_t>(kSortWarps) + warp;
    if (i >= n) return;
    if (kFill && off[n] > cap) return;  // lists exceed the speculative capacity: the host redoes the fill
    const V3 p = ld3(pos, i);
    const int4 ci = cells[i];
    int32_t o = kFill ? off[i] : 0;
    for (int64_t b = 0; b < n; b += 32) {
        const int64_t j = b + lane;
        bool hit = false;
        if (j < n && j != i) {
            const int4 cj = __ldg(cells + j);
            hit = abs(cj.x - ci.x) <= rad && abs(cj.y - ci.y) <= rad && abs(cj.z - ci.z) <= rad &&
                  sqnorm(sub(ld3(pos, j), p)) <= r2;
        }
        const unsigned m = __ballot_sync(kFull, hit);
        if (kFill && hit) nbr[o + __popc(m & ((1u << lane) - 1u))] = static_cast<int32_t>(j);
        o += __popc(m);
    }
    if (!kFill && lane == 0) counts[i] = o;
}

// One pass of k_nbr_brute that counts and keeps the first kNbrSlots
// neighbours of each point in a fixed-stride table (ascending j); points with
// more set *overflow (the host then runs the exact two-pass fill).
constexpr int kNbrSlots = 192;

__global__ void __launch_bounds__(32 * kSortWarps) k_nbr_brute_once(const double* __restrict__ pos,
                                                                    const int4* __restrict__ cells,
                                                                    const uint32_t* __restrict__ keys, int64_t n,
                                                                    int rad, double r2, int32_t* __restrict__ counts,
                                                                    int32_t* __restrict__ slots,
                                                                    int32_t* __restrict__ overflow) {
    // per warp: candidates that pass the packed-cell filter, queued in index
    // order and tested 32 at a time (exact cell test + distance), so the
    // lanes stay busy although only a few percent of the cloud are candidates
    __shared__ int32_t s_q[kSortWarps][64];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i64 = blockIdx.x * static_cast<int64_t>(kSortWarps) + warp;
    if (i64 >= n) return;
    const int i = static_cast<int>(i64), ni = static_cast<int>(n);  // n <= kBruteMax
    const V3 p = ld3(pos, i);
    const int4 ci = cells[i];
    const uint32_t ki = pack_cell(ci);
    int32_t* row = slots + i64 * kNbrSlots;
    int32_t* q = s_q[warp];
    int o = 0, qn = 0;
    const unsigned lt = (1u << lane) - 1u;
    auto test = [&](int m) {  // the first m queued candidates, in order (i itself is one)
        bool hit = false;
        int j = 0;
        if (lane < m) {
            j = q[lane];
            const int4 cj = __ldg(cells + j);
            hit = j != i && abs(cj.x - ci.x) <= rad && abs(cj.y - ci.y) <= rad && abs(cj.z - ci.z) <= rad &&
                  sqnorm(sub(ld3(pos, j), p)) <= r2;
        }
        const unsigned hm = __ballot_sync(kFull, hit);
        const int at = o + __popc(hm & lt);
        if (hit && at < kNbrSlots) row[at] = j;
        o += __popc(hm);
    };
    auto enqueue = [&](bool cand, int j) {
        const unsigned m = __ballot_sync(kFull, cand);
        if (m == 0u) return;  // the common case: one vote per 32 points
        if (cand) q[qn + __popc(m & lt)] = j;
        qn += __popc(m);
        if (qn >= 32) {
            __syncwarp();
            test(32);
            __syncwarp();
            const int32_t rest = lane + 32 < qn ? q[lane + 32] : 0;
            __syncwarp();
            q[lane] = rest;
            __syncwarp();
            qn -= 32;
        }
    };
    constexpr int kU = 4;  // four 32-point chunks per step: their key loads issued together
    int b0 = 0;
    for (; b0 + 32 * kU <= ni; b0 += 32 * kU) {
        uint32_t kj[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) kj[u] = __ldg(keys + b0 + 32 * u + lane);
#pragma unroll
        for (int u = 0; u < kU; ++u) enqueue(cell_near(kj[u], ki), b0 + 32 * u + lane);
    }
    for (; b0 < ni; b0 += 32) {
        const int j = b0 + lane;
        enqueue(j < ni && cell_near(__ldg(keys + j), ki), j);
    }
    __syncwarp();
    test(qn);
    if (lane == 0) {
        counts[i] = o;
        if (o > kNbrSlots) atomicExch(overflow, 1);
    }
}

// fixed-stride table -> CSR at the scanned offsets (warp per point)
__global__ void k_nbr_compact(const int32_t* __restrict__ slots, const int32_t* __restrict__ off, int64_t n,
                              const int32_t* __restrict__ overflow, int32_t* __restrict__ nbr, int64_t cap) {
    const int lane = threadIdx.x & 31;
    const int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (i >= n || *overflow || off[n] > cap) return;
    const int32_t o0 = off[i], k = off[i + 1] - o0;
    for (int a = lane; a < k; a += 32) nbr[o0 + a] = slots[i * kNbrSlots + a];
}

// warp per point: gather the neighbours (row by row, lanes over slots,
// ballot-compacted), then sort ascending (radius_search sorts its output)
__global__ void __launch_bounds__(32 * kSortWarps) k_nbr_fill(const double* __restrict__ pos, int64_t n, GridView g,
                                                              double r2, const int32_t* __restrict__ off,
                                                              int32_t* __restrict__ nbr, int64_t cap) {
    __shared__ int32_t s_buf[kSortWarps][kSortCap];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i = blockIdx.x * static_cast<int64_t>(kSortWarps) + warp;
    if (i >= n) return;
    if (off[n] > cap) return;  // lists exceed the speculative capacity: the host redoes the fill
    const V3 p = ld3(pos, i);
    const int kx = floor_cell((p.x - g.ox) / g.cell) - g.offx;
    const int ky = floor_cell((p.y - g.oy) / g.cell) - g.offy;
    const int kz = floor_cell((p.z - g.oz) / g.cell) - g.offz;
    const int32_t o0 = off[i];
    int32_t o = o0;
    for (int x = max(kx - g.radius, 0); x <= min(kx + g.radius, g.nx - 1); ++x)
        for (int y = max(ky - g.radius, 0); y <= min(ky + g.radius, g.ny - 1); ++y) {
            const int64_t row = (static_cast<int64_t>(x) * g.ny + y) * g.nz;
            const int32_t s0 = g.start[row + max(kz - g.radius, 0)];
            const int32_t s1 = g.start[row + min(kz + g.radius, g.nz - 1) + 1];
            for (int32_t b = s0; b < s1; b += 32) {
                const int32_t s = b + lane;
                const bool hit = s < s1 && g.index[s] != i && sqnorm(sub(ld3(g.slot_pos, s), p)) <= r2;
                const unsigned m = __ballot_sync(kFull, hit);
                if (hit) nbr[o + __popc(m & ((1u << lane) - 1u))] = g.index[s];
                o += __popc(m);
            }
        }
    __syncwarp();
    const int k = o - o0;
    const int32_t* sorted = warp_sort_segment(nbr + o0, k, s_buf[warp], kSortCap);
    if (sorted != nbr + o0)
        for (int a = lane; a < k; a += 32) nbr[o0 + a] = sorted[a];
}

constexpr int kFpfhWarps = 4;
constexpr int kRows = 8;  // spfh rows in flight per step of k_fpfh

// a / b correctly rounded from r = RN(1 / b): q = RN(a r) is within one ulp,
// the residual a - b q is exact in one FMA, and RN(q + residual * r) is the
// correctly rounded quotient (Markstein; no over/underflow for the FPFH
// ranges: a in [0, 100], b in (0, radius]). One reciprocal per neighbour
// instead of 33 divisions.
__device__ __forceinline__ double div_by(double a, double b, double r) {
    const double q = a * r;
    const double e = fma(-q, b, a);
    return fma(e, r, q);
}

// pass 1 (proj/src/fpfh.cpp:76-100): warp per point, integer vote counts in
// counts[i][0..32], votes in counts[i][33]. Pairs whose frame-source test the
// device cannot decide are appended to the deferred list (k_spfh_resolve_b).
// Pairs the device cannot settle go to the host's libm on two lists:
//   A  the frame-source test acos(|a1|) > acos(|a2|) is undecided here and
//      the bins depend on it (common on planar faces): (i, j) and (|a1|,
//      |a2|); the host decides the swap, k_spfh_resolve_a recomputes the bins;
//   B  theta (atan2) lies at a bin edge for an outcome the pair can take
//      (astronomically rare): (i, j) and the two points and normals; the host
//      evaluates pair_angles whole (host_pair_bins), k_spfh_resolve_b votes.
struct DeferredPair {
    double v[12];  // p1, n1, p2, n2
};
struct DeferLists {
    int2* a_ij;
    double2* a_x;
    int2* b_ij;
    DeferredPair* b_x;
    int32_t* n;  // n[0] = list A, n[1] = list B, n[2] = list A2
    int64_t a_cap, b_cap;
    int32_t* a_dec;  // list A decisions: 0 / 1, or 2 + the entry's list A2 slot (the host decides)
    double4* a2_x;   // (|a1|, |a2|, v1, v2): v = glibc's acos when certain, else NaN
};

// compute_fpfh's one device->host copy before the host decides the deferred
// pairs: the counts, list B's first entries and, from a[], list A2's (|a1|,
// |a2|, v1, v2) -- dl.a2_x points at a[0] and runs on past the struct
constexpr int kStageA = 2048;
constexpr int kStageB = 64;
struct FpfhHead {
    int32_t total, n_a, n_b, n_a2, overflow, pad[3];
    DeferredPair b[kStageB];
    double4 a[kStageA];
};
static_assert(offsetof(FpfhHead, b) == 32 && offsetof(FpfhHead, a) % 32 == 0, "FpfhHead layout");

// List A's frame-source tests settled on the device where glibc's outcome is
// certain (lk_acos_cr.hpp acos_greater); the rest go to list A2 for the host.
__global__ void k_spfh_decide_a(DeferLists dl, const int32_t* __restrict__ total, const int32_t* __restrict__ overflow,
                                FpfhHead* __restrict__ head) {
    const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < dl.n[0]) {
        const double2 x = dl.a_x[k];
        double l1, h1, l2, h2;
        const int r1 = lkacos::acos_bracket(x.x, &l1, &h1), r2 = lkacos::acos_bracket(x.y, &l2, &h2);
        if (r1 && r2 && (l1 > h2 || h1 <= l2)) {  // lkacos::acos_greater, certain
            dl.a_dec[k] = l1 > h2 ? 1 : 0;
        } else {
            // the host evaluates only the values whose rounding is in doubt
            const double nan = __longlong_as_double(0x7ff8000000000000ll);
            const int32_t slot = atomicAdd(dl.n + 2, 1);
            dl.a_dec[k] = 2 + slot;
            dl.a2_x[slot] = make_double4(x.x, x.y, r1 == 1 ? l1 : nan, r2 == 1 ? l2 : nan);
        }
    }
    // the last block to finish writes the head's counts and list B's first
    // entries (dl.n[3]: blocks done, zeroed with the counts)
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(dl.n + 3, 1) == static_cast<int32_t>(gridDim.x) - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const volatile int32_t* vn = dl.n;
    const int32_t n_b = vn[1];
    if (threadIdx.x == 0) {
        head->total = *total;
        head->n_a = vn[0];
        head->n_b = n_b;
        head->n_a2 = vn[2];
        head->overflow = overflow ? *overflow : 0;
    }
    const int nb = n_b < kStageB ? n_b : kStageB;
    for (int t = threadIdx.x; t < nb * 12; t += blockDim.x) head->b[t / 12].v[t % 12] = dl.b_x[t / 12].v[t % 12];
}

__global__ void __launch_bounds__(32 * kFpfhWarps) k_spfh(const double* __restrict__ pos,
                                                          const double* __restrict__ nrm, int64_t n,
                                                          const int32_t* __restrict__ off,
                                                          const int32_t* __restrict__ nbr, int32_t* __restrict__ counts,
                                                          DeferLists dl, int64_t cap,
                                                          const int32_t* __restrict__ skip) {
    __shared__ int hist[kFpfhWarps][34];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i = blockIdx.x * static_cast<int64_t>(kFpfhWarps) + warp;
    if (i >= n) return;
    if (off[n] > cap || (skip && *skip)) return;  // the neighbour lists overflowed: redone by the host
    for (int b = lane; b < 34; b += 32) hist[warp][b] = 0;
    __syncwarp();
    const V3 p = ld3(pos, i), np = ld3(nrm, i);
    int votes = 0;
    if (!is_zero(np)) {
        for (int32_t k = off[i] + lane; k < off[i + 1]; k += 32) {
            const int32_t j = nbr[k];
            const V3 nq = ld3(nrm, j);
            if (is_zero(nq)) continue;
            const V3 q = ld3(pos, j);
            PairSetup s;
            if (!pair_setup(p, np, q, nq, s)) continue;
            const int dec = swap_decision(fabs(s.a1), fabs(s.a2));
            int3 bins;
            bool valid, edge;
            int list = -1;  // 0 = A, 1 = B
            if (dec == 2) {
                // undecidable here: settle it only if the outcome depends on it
                int3 b1;
                bool edge1;
                valid = pair_bins(s, np, nq, 0, bins, edge);
                const bool valid1 = pair_bins(s, np, nq, 1, b1, edge1);
                if ((valid && edge) || (valid1 && edge1))
                    list = 1;
                else if (valid != valid1 || (valid && (bins.x != b1.x || bins.y != b1.y || bins.z != b1.z)))
                    list = 0;
            } else {
                valid = pair_bins(s, np, nq, dec, bins, edge);
                if (valid && edge) list = 1;
            }
            if (list == 0) {
                const int32_t slot = atomicAdd(dl.n, 1);
                if (slot < dl.a_cap) {  // full: the host sees the count over capacity and redoes the pass
                    dl.a_ij[slot] = make_int2(static_cast<int32_t>(i), j);
                    dl.a_x[slot] = make_double2(fabs(s.a1), fabs(s.a2));
                }
                continue;
            }
            if (list == 1) {
                const int32_t slot = atomicAdd(dl.n + 1, 1);
                if (slot < dl.b_cap) {
                    dl.b_ij[slot] = make_int2(static_cast<int32_t>(i), j);
                    DeferredPair& d = dl.b_x[slot];
                    d.v[0] = p.x, d.v[1] = p.y, d.v[2] = p.z, d.v[3] = np.x, d.v[4] = np.y, d.v[5] = np.z;
                    d.v[6] = q.x, d.v[7] = q.y, d.v[8] = q.z, d.v[9] = nq.x, d.v[10] = nq.y, d.v[11] = nq.z;
                }
                continue;
            }
            if (!valid) continue;
            atomicAdd(&hist[warp][bins.x], 1);
            atomicAdd(&hist[warp][bins.y], 1);
            atomicAdd(&hist[warp][bins.z], 1);
            votes += 1;
        }
    }
    for (int o = 16; o > 0; o >>= 1) votes += __shfl_xor_sync(kFull, votes, o);
    __syncwarp();
    for (int b = lane; b < 33; b += 32) counts[34 * i + b] = hist[warp][b];
    if (lane == 0) counts[34 * i + 33] = votes;
}

// list A with the host's decisions (0/1) of the frame-source test (no theta
// edge for either outcome: checked in k_spfh)
__global__ void k_spfh_resolve_a(const double* __restrict__ pos, const double* __restrict__ nrm,
                                 const int2* __restrict__ deferred, const int32_t* __restrict__ decision,
                                 const uint8_t* __restrict__ host_dec, int32_t m, int32_t* __restrict__ counts) {
    const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    const int2 ij = deferred[k];
    int32_t dec = decision[k];
    if (dec >= 2) dec = host_dec[dec - 2];  // page-locked host memory, read in place
    const V3 n1 = ld3(nrm, ij.x), n2 = ld3(nrm, ij.y);
    PairSetup s;
    int3 bins;
    bool edge;
    if (!pair_setup(ld3(pos, ij.x), n1, ld3(pos, ij.y), n2, s) || !pair_bins(s, n1, n2, dec, bins, edge))
        return;
    int32_t* c = counts + 34 * static_cast<int64_t>(ij.x);
    atomicAdd(c + bins.x, 1);
    atomicAdd(c + bins.y, 1);
    atomicAdd(c + bins.z, 1);
    atomicAdd(c + 33, 1);
}

// list B with the host's bins: (alpha bin, 11 + phi bin, 22 + theta bin) as
// bytes 0-2, byte 3 = 1 for a vote (0: the pair casts none)
__global__ void k_spfh_resolve_b(const int2* __restrict__ deferred, const uint32_t* __restrict__ decision, int32_t m,
                                 int32_t* __restrict__ counts) {
    const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    const uint32_t d = decision[k];
    if (!(d >> 24)) return;
    int32_t* c = counts + 34 * static_cast<int64_t>(deferred[k].x);
    atomicAdd(c + (d & 0xff), 1);
    atomicAdd(c + ((d >> 8) & 0xff), 1);
    atomicAdd(c + ((d >> 16) & 0xff), 1);
    atomicAdd(c + 33, 1);
}

// h[b] accumulates 1.0 per vote exactly, then h[b] *= 100.0 / votes
__global__ void k_spfh_scale(const int32_t* __restrict__ counts, int64_t n, double* __restrict__ spfh) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= 33 * n) return;
    const int64_t i = t / 33, b = t - 33 * i;
    const int32_t votes = counts[34 * i + 33];
    spfh[t] = votes > 0 ? static_cast<double>(counts[34 * i + b]) * (100.0 / static_cast<double>(votes)) : 0.0;
}

// pass 2 (proj/src/fpfh.cpp:102-139): warp per point, lane per bin
__global__ void __launch_bounds__(32 * kFpfhWarps) k_fpfh(const double* __restrict__ pos,
                                                          const double* __restrict__ nrm, int64_t n,
                                                          const int32_t* __restrict__ off,
                                                          const int32_t* __restrict__ nbr,
                                                          const double* __restrict__ spfh, float* __restrict__ out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i = blockIdx.x * static_cast<int64_t>(kFpfhWarps) + warp;
    if (i >= n) return;
    if (is_zero(ld3(nrm, i))) {
        for (int b = lane; b < 33; b += 32) out[33 * i + b] = 0.0f;
        return;
    }
    const V3 p = ld3(pos, i);
    double acc0 = 0.0, acc1 = 0.0;  // bin lane, and bin 32 on lane 0
    int k_count = 0;
    const int32_t k1 = off[i + 1];
    for (int32_t base = off[i]; base < k1; base += 32) {
        // lane t: neighbour base + t -- its usability, weight, the correctly
        // rounded reciprocal of the weight and its bin-32 term
        const int32_t kk = base + lane;
        int32_t j = 0;
        double w = 1.0, r = 1.0, q32 = 0.0;
        bool ok = false;
        if (kk < k1) {
            j = nbr[kk];
            if (!is_zero(ld3(nrm, j))) {
                w = sqrt(sqnorm(sub(ld3(pos, j), p)));
                ok = w > 0.0;
            }
            if (ok) {
                r = 1.0 / w;
                q32 = div_by(spfh[33 * static_cast<int64_t>(j) + 32], w, r);
            } else {
                w = 1.0;
            }
        }
        unsigned m = __ballot_sync(kFull, ok);
        k_count += __popc(m);
        // the usable ones in neighbour order, kRows rows of spfh in flight
        while (m) {
            int src[kRows];
            bool use[kRows];
#pragma unroll
            for (int t = 0; t < kRows; ++t) {
                use[t] = m != 0;
                src[t] = use[t] ? __ffs(m) - 1 : 0;
                if (use[t]) m &= m - 1;
            }
            double sv[kRows], wv[kRows], rv[kRows], q32v[kRows];
#pragma unroll
            for (int t = 0; t < kRows; ++t) {
                const int32_t jt = __shfl_sync(kFull, j, src[t]);
                wv[t] = __shfl_sync(kFull, w, src[t]);
                rv[t] = __shfl_sync(kFull, r, src[t]);
                q32v[t] = __shfl_sync(kFull, q32, src[t]);
                sv[t] = use[t] ? spfh[33 * static_cast<int64_t>(jt) + lane] : 0.0;
            }
#pragma unroll
            for (int t = 0; t < kRows; ++t) {
                if (use[t]) {
                    acc0 += div_by(sv[t], wv[t], rv[t]);
                    acc1 += q32v[t];  // lane 0's value is the one used
                }
            }
        }
    }
    {
        double blended = spfh[33 * i + lane];
        if (k_count > 0) blended += acc0 / static_cast<double>(k_count);
        out[33 * i + lane] = static_cast<float>(blended);
    }
    if (lane == 0) {
        double blended = spfh[33 * i + 32];
        if (k_count > 0) blended += acc1 / static_cast<double>(k_count);
        out[33 * i + 32] = static_cast<float>(blended);
    }
}

// estimate_normals (proj/src/preprocess.cpp:61-96), warp per point: the
// radius_search neighbours (grid.cpp:153-174 with cell = radius: the +-1 cell
// window and d2 <= r^2, self included, ascending index) are found by a brute
// scan in index order; the mean and then the covariance are the reference's
// sequential sums (each hit broadcast to the warp in order); the eigenvector
// of the smallest eigenvalue (lk_eig3.hpp) is normalised and oriented to the
// viewpoint. Fewer than 3 neighbours or a non-finite length: zero normal.
// The normal of one point from a warp-uniform scan(use) that calls use(q) for
// each radius_search neighbour q in ascending index order (self included).
template <class Scan>
__device__ __forceinline__ void normal_of(V3 p, double vx, double vy, double vz, Scan&& scan, double* out3) {
    const int lane = threadIdx.x & 31;
    V3 mean = mk(0.0, 0.0, 0.0);
    int64_t cnt = 0;
    scan([&](V3 q) {
        mean = mk(mean.x + q.x, mean.y + q.y, mean.z + q.z);
        ++cnt;
    });
    double nv[3] = {0.0, 0.0, 0.0};
    if (cnt >= 3) {
        const double c = static_cast<double>(cnt);
        mean = mk(mean.x / c, mean.y / c, mean.z / c);
        double a00 = 0.0, a10 = 0.0, a20 = 0.0, a11 = 0.0, a21 = 0.0, a22 = 0.0;
        scan([&](V3 q) {  // cov += d d^T (lower triangle)
            const V3 d = sub(q, mean);
            a00 = a00 + d.x * d.x;
            a10 = a10 + d.y * d.x;
            a20 = a20 + d.z * d.x;
            a11 = a11 + d.y * d.y;
            a21 = a21 + d.z * d.y;
            a22 = a22 + d.z * d.z;
        });
        double v[3];
        lkeig::smallest_eigenvector(a00, a10, a20, a11, a21, a22, v);
        const double len = sqrt(sqnorm(mk(v[0], v[1], v[2])));
        if (len > 0.0 && isfinite(len)) {
            V3 nn = mk(v[0] / len, v[1] / len, v[2] / len);
            if (dot(nn, mk(vx - p.x, vy - p.y, vz - p.z)) < 0.0) nn = mk(-nn.x, -nn.y, -nn.z);
            nv[0] = nn.x;
            nv[1] = nn.y;
            nv[2] = nn.z;
        }
    }
    if (lane == 0) {
        out3[0] = nv[0];
        out3[1] = nv[1];
        out3[2] = nv[2];
    }
}

// estimate_normals (proj/src/preprocess.cpp:61-96), warp per point: the
// radius_search neighbours (grid.cpp:153-174 with cell = radius: the +-1 cell
// window and d2 <= r^2, self included, ascending index) are found by a brute
// scan in index order; the mean and then the covariance are the reference's
// sequential sums (each hit broadcast to the warp in order); the eigenvector
// of the smallest eigenvalue (lk_eig3.hpp) is normalised and oriented to the
// viewpoint. Fewer than 3 neighbours or a non-finite length: zero normal.
__global__ void __launch_bounds__(32 * kSortWarps) k_estimate_normals(const double* __restrict__ pos,
                                                                      const int4* __restrict__ cells, int64_t n,
                                                                      double r2, double vx, double vy, double vz,
                                                                      double* __restrict__ out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i = blockIdx.x * static_cast<int64_t>(kSortWarps) + warp;
    if (i >= n) return;
    const V3 p = ld3(pos, i);
    const int4 ci = cells[i];
    auto scan = [&](auto&& use) {
        for (int64_t b = 0; b < n; b += 32) {
            const int64_t j = b + lane;
            V3 q = mk(0.0, 0.0, 0.0);
            bool hit = false;
            if (j < n) {
                const int4 cj = __ldg(cells + j);
                if (abs(cj.x - ci.x) <= 1 && abs(cj.y - ci.y) <= 1 && abs(cj.z - ci.z) <= 1) {
                    q = ld3(pos, j);
                    hit = sqnorm(sub(q, p)) <= r2;
                }
            }
            unsigned m = __ballot_sync(kFull, hit);
            while (m) {
                const int k = __ffs(m) - 1;
                m &= m - 1;
                use(mk(__shfl_sync(kFull, q.x, k), __shfl_sync(kFull, q.y, k), __shfl_sync(kFull, q.z, k)));
            }
        }
    };
    normal_of(p, vx, vy, vz, scan, out + 3 * i);
}

// The same from the SearchGrid neighbour lists of the FPFH path (sorted
// ascending, self excluded; self is visited at its place in the order).
__global__ void __launch_bounds__(32 * kSortWarps) k_estimate_normals_lists(const double* __restrict__ pos,
                                                                            int64_t n,
                                                                            const int32_t* __restrict__ off,
                                                                            const int32_t* __restrict__ nbr,
                                                                            double vx, double vy, double vz,
                                                                            double* __restrict__ out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i = blockIdx.x * static_cast<int64_t>(kSortWarps) + warp;
    if (i >= n) return;
    const V3 p = ld3(pos, i);
    const int32_t o0 = off[i], k = off[i + 1] - o0;
    // self's place: the number of listed neighbours below i
    int below = 0;
    for (int a = lane; a < k; a += 32) below += nbr[o0 + a] < i ? 1 : 0;
    below = __reduce_add_sync(kFull, below);
    auto scan = [&](auto&& use) {
        for (int b = 0; b <= k; b += 32) {
            const int v = b + lane;  // position in the list with self inserted
            V3 q = mk(0.0, 0.0, 0.0);
            if (v <= k) q = ld3(pos, v < below ? nbr[o0 + v] : (v == below ? static_cast<int32_t>(i) : nbr[o0 + v - 1]));
            const int cnt = k + 1 - b < 32 ? k + 1 - b : 32;
            for (int t = 0; t < cnt; ++t)
                use(mk(__shfl_sync(kFull, q.x, t), __shfl_sync(kFull, q.y, t), __shfl_sync(kFull, q.z, t)));
        }
    };
    normal_of(p, vx, vy, vz, scan, out + 3 * i);
}

// usable (non-zero) normals and max |p| of a cloud
__global__ void k_cloud_stats(const double* __restrict__ pos, const double* __restrict__ nrm, int64_t n,
                              unsigned long long* __restrict__ out) {
    unsigned long long usable = 0;
    double m = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (nrm && !is_zero(ld3(nrm, i))) ++usable;
        const double x = pos[3 * i], y = pos[3 * i + 1], z = pos[3 * i + 2];
        m = fmax(m, sqrt(x * x + y * y + z * z));
    }
    // non-negative doubles order like their bit patterns
    atomicAdd(&out[0], usable);
    atomicMax(&out[1], static_cast<unsigned long long>(__double_as_longlong(m)));
}

#define LK_TRY(x)                         \
    do {                                  \
        cudaError_t e_ = (x);             \
        if (e_ != cudaSuccess) return e_; \
    } while (0)

}  // namespace

cudaError_t estimate_normals(const double* d_pos, int64_t n, double radius, const double* viewpoint, double* d_out,
                             cudaStream_t stream) {
    if (n <= 0 || !(radius > 0.0)) return cudaErrorInvalidValue;
    const double r2 = radius * radius;
    if (n <= kBruteMax) {
        int4* cells = nullptr;
        LK_TRY(cudaMallocAsync(&cells, n * sizeof(int4), stream));
        k_search_cells<<<nblocks(n, 256), 256, 0, stream>>>(d_pos, n, radius, cells);
        k_estimate_normals<<<nblocks(n, kSortWarps), 32 * kSortWarps, 0, stream>>>(
            d_pos, cells, n, r2, viewpoint[0], viewpoint[1], viewpoint[2], d_out);
        cudaFreeAsync(cells, stream);
        return cudaGetLastError();
    }
    // larger clouds: the FPFH path's SearchGrid lists (exact size, one readback)
    GridStorage g;
    int32_t *counts = nullptr, *off = nullptr, *nbr = nullptr;
    LK_TRY(build_grid(g, 1, d_pos, nullptr, n, radius, radius, stream, false));
    LK_TRY(cudaMallocAsync(&counts, n * sizeof(int32_t), stream));
    LK_TRY(cudaMallocAsync(&off, (n + 1) * sizeof(int32_t), stream));
    k_nbr_count<<<nblocks(n, kSortWarps), 32 * kSortWarps, 0, stream>>>(d_pos, n, g.view, r2, counts);
    LK_TRY(exclusive_scan(counts, n, off, stream));
    int32_t* h_total = static_cast<int32_t*>(host_scratch(sizeof(int32_t)));
    if (!h_total) return cudaErrorMemoryAllocation;
    LK_TRY(cudaMemcpyAsync(h_total, off + n, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
    LK_TRY(cudaStreamSynchronize(stream));
    const int64_t total = *h_total;
    LK_TRY(cudaMallocAsync(&nbr, (total > 0 ? total : 1) * sizeof(int32_t), stream));
    k_nbr_fill<<<nblocks(n, kSortWarps), 32 * kSortWarps, 0, stream>>>(d_pos, n, g.view, r2, off, nbr,
                                                                       total > 0 ? total : 1);
    k_estimate_normals_lists<<<nblocks(n, kSortWarps), 32 * kSortWarps, 0, stream>>>(
        d_pos, n, off, nbr, viewpoint[0], viewpoint[1], viewpoint[2], d_out);
    cudaFreeAsync(counts, stream);
    cudaFreeAsync(off, stream);
    cudaFreeAsync(nbr, stream);
    g.release();
    return cudaGetLastError();
}

cudaError_t voxel_downsample(const double* d_pos, const double* d_nrm, int64_t n, double leaf, double* d_out_pos,
                             double* d_out_nrm, int64_t* out_count, int* status, cudaStream_t stream,
                             unsigned long long* h_stats) {
    *status = 0;
    *out_count = 0;
    if (n <= 0) {
        *status = 2;
        return cudaSuccess;
    }
    if (n > INT32_MAX / 2) return cudaErrorInvalidValue;
    uint32_t table = 1024;
    while (table < 2 * n) table <<= 1;
    // members grouped by output voxel, ascending input index inside each: a
    // stable LSD radix sort on the voxel ordinal (< n_out <= n)
    int max_bit = 1;
    while ((int64_t(1) << max_bit) < n) ++max_bit;
    size_t sort_bytes = 0;
    LK_TRY(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, static_cast<const int32_t*>(nullptr),
                                           static_cast<int32_t*>(nullptr), static_cast<const int32_t*>(nullptr),
                                           static_cast<int32_t*>(nullptr), static_cast<int>(n), 0, max_bit, stream));
    const size_t scan_bytes = scan_temp_bytes(n);
    using S = Scratch;
    const size_t tb = S::round(table * sizeof(unsigned long long)) + 3 * S::round(table * sizeof(int32_t));
    const size_t nb = S::round(n * sizeof(int32_t));
    Scratch sc(stream, tb + 8 * nb + 3 * S::round((n + 2) * sizeof(int32_t)) +
                           S::round(scan_bytes) + S::round(sort_bytes) + S::round(2 * sizeof(unsigned long long)));
    unsigned long long* keys = sc.take<unsigned long long>(table);
    int32_t* first = sc.take<int32_t>(table);
    int32_t* count = sc.take<int32_t>(table);
    int32_t* slot_out = sc.take<int32_t>(table);
    int32_t* point_slot = sc.take<int32_t>(n);
    int32_t* flags = sc.take<int32_t>(n);
    int32_t* flag_scan = sc.take<int32_t>(n + 2);
    int32_t* bad = flag_scan + n + 1;  // read back with the total in one copy
    void* scan_temp = sc.take<char>(scan_bytes);
    int32_t* cnt_out = sc.take<int32_t>(n + 1);
    int32_t* member_start = sc.take<int32_t>(n + 1);
    int32_t* members = sc.take<int32_t>(n);
    int32_t* skeys = sc.take<int32_t>(n);
    int32_t* svals = sc.take<int32_t>(n);
    int32_t* skeys_out = sc.take<int32_t>(n);
    void* sort_temp = sc.take<char>(sort_bytes);
    unsigned long long* d_stats = sc.take<unsigned long long>(2);
    LK_TRY(sc.status());
    const int64_t init_n = std::max<int64_t>(table, n);
    k_vox_init<<<static_cast<unsigned>(std::min<int64_t>(nblocks(init_n, 256), 148 * 8)), 256, 0, stream>>>(
        table, n, keys, first, count, flags, flag_scan, bad, d_stats);
    k_vox_insert<<<nblocks(n, 256), 256, 0, stream>>>(d_pos, d_nrm, n, leaf, keys, table - 1, point_slot, first,
                                                     count, bad);
    k_vox_mark<<<nblocks(table, 256), 256, 0, stream>>>(keys, first, table, flags);
    LK_TRY(exclusive_scan(flags, n, flag_scan, stream, scan_temp, scan_bytes, false));
    trace_point("vox scan", stream);
    int32_t* host = static_cast<int32_t*>(host_scratch(2 * sizeof(int32_t)));
    if (!host) return cudaErrorMemoryAllocation;
    LK_TRY(cudaMemcpyAsync(host, flag_scan + n, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
    LK_TRY(cudaStreamSynchronize(stream));
    if (host[1]) {
        *status = 5;
        return cudaSuccess;
    }
    const int64_t n_out = host[0];
    trace_point("vox count back", stream);
    k_vox_out<<<nblocks(table, 256), 256, 0, stream>>>(keys, first, count, table, flag_scan, slot_out, cnt_out,
                                                       member_start);
    LK_TRY(exclusive_scan(cnt_out, n_out, member_start, stream, scan_temp, scan_bytes, false));
    k_vox_keys<<<nblocks(n, 256), 256, 0, stream>>>(point_slot, n, slot_out, skeys, svals);
    int end_bit = 1;
    while ((int64_t(1) << end_bit) < n_out) ++end_bit;
    size_t sort_need = 0;
    LK_TRY(cub::DeviceRadixSort::SortPairs(nullptr, sort_need, skeys, skeys_out, svals, members, static_cast<int>(n),
                                           0, end_bit, stream));
    if (sort_need > sort_bytes) return cudaErrorInvalidValue;  // fewer bits never need more storage
    LK_TRY(cub::DeviceRadixSort::SortPairs(sort_temp, sort_bytes, skeys, skeys_out, svals, members,
                                           static_cast<int>(n), 0, end_bit, stream));
    trace_point("vox sorted", stream);
    k_vox_reduce<<<nblocks(n_out, kSortWarps), 32 * kSortWarps, 0, stream>>>(
        members, member_start, n_out, d_pos, d_nrm, d_out_pos, d_out_nrm, h_stats ? d_stats : nullptr);
    if (h_stats)
        LK_TRY(cudaMemcpyAsync(h_stats, d_stats, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream));
    *out_count = n_out;
    return cudaGetLastError();
}

// proj/src/fpfh.cpp:17-53 on the host with the reference's libm (std::acos,
// std::atan2) for the pairs k_spfh defers. Same IEEE operation order as the
// device (-ffp-contract=off), so everything but the two libm calls agrees
// bit for bit. Returns the packed bins of k_spfh_resolve_b.
static uint32_t host_pair_bins(const double* v) {
    struct H {
        double x, y, z;
    };
    auto sub3 = [](H a, H b) { return H{a.x - b.x, a.y - b.y, a.z - b.z}; };
    auto dot3 = [](H a, H b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; };
    auto cross3 = [](H a, H b) { return H{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; };
    auto bin = [](double value, double lo, double hi) {
        int b = static_cast<int>(std::floor(11 * (value - lo) / (hi - lo)));
        return std::clamp(b, 0, 10);
    };
    const H p1{v[0], v[1], v[2]}, n1{v[3], v[4], v[5]}, p2{v[6], v[7], v[8]}, n2{v[9], v[10], v[11]};
    const H d = sub3(p2, p1);
    const double dist = std::sqrt(dot3(d, d));
    if (dist <= 0.0) return 0;
    const double angle1 = dot3(n1, d) / dist;
    const double angle2 = dot3(n2, d) / dist;
    H ns = n1, nt = n2, line = d;
    double cos_line = angle1;
    if (std::acos(std::abs(angle1)) > std::acos(std::abs(angle2))) {
        ns = n2;
        nt = n1;
        line = H{-d.x, -d.y, -d.z};
        cos_line = -angle2;
    }
    const H u = ns;
    H w3 = cross3(line, u);
    const double v_len = std::sqrt(dot3(w3, w3));
    if (v_len <= 1e-12 * dist) return 0;
    const H vv{w3.x / v_len, w3.y / v_len, w3.z / v_len};
    const H w = cross3(u, vv);
    const double alpha = dot3(vv, nt);
    const double theta = std::atan2(dot3(w, nt), dot3(u, nt));
    const uint32_t b0 = static_cast<uint32_t>(bin(alpha, -1.0, 1.0));
    const uint32_t b1 = 11u + static_cast<uint32_t>(bin(cos_line, -1.0, 1.0));
    const uint32_t b2 = 22u + static_cast<uint32_t>(bin(theta, -M_PI, M_PI));
    return b0 | (b1 << 8) | (b2 << 16) | (1u << 24);
}

// Pinned host staging of compute_fpfh, one per host thread (each prepare side
// runs on its own thread): the FpfhHead comes back in one copy; the host's
// decisions are written here and read by the resolve kernels in place.
// Reused only after the caller's stream has synchronised.
struct FpfhStage {
    FpfhHead* head = nullptr;
    double4* more_a = nullptr;  // list A2 beyond kStageA (rare)
    size_t more_cap = 0;
    uint8_t* dec_a = nullptr;
    uint32_t* dec_b = nullptr;
    size_t dec_a_cap = 0, dec_b_cap = 0;
    ~FpfhStage() {
        if (head) cudaFreeHost(head);
        if (more_a) cudaFreeHost(more_a);
        if (dec_a) cudaFreeHost(dec_a);
        if (dec_b) cudaFreeHost(dec_b);
    }
};
thread_local FpfhStage t_stage;

cudaError_t compute_fpfh(const double* d_pos, const double* d_nrm, int64_t n, double radius, float* d_out,
                         cudaStream_t stream) {
    if (n <= 0) return cudaErrorInvalidValue;
    FpfhStage& st = t_stage;
    if (!st.head) LK_TRY(cudaHostAlloc(reinterpret_cast<void**>(&st.head), sizeof(FpfhHead), 0));
    GridStorage g;
    const double r2 = radius * radius;
    const bool brute = n <= kBruteMax;
    // speculative capacity (no host round trip for the total): 192 neighbours
    // per point; an overflow turns the fill and the votes into no-ops and is
    // redone below with the exact size (pool allocations, rare)
    int64_t cap = std::max<int64_t>(192 * n, 4096);
    int64_t a_cap = std::max<int64_t>(8 * n, 65536);  // list A: acos ties (planar faces: ~4 per point)
    int64_t b_cap = 4096;                            // list B: theta bin edges (essentially never)
    using S = Scratch;
    const size_t scan_bytes = scan_temp_bytes(n);
    const size_t lists_bytes = S::round(cap * sizeof(int32_t)) + S::round(a_cap * sizeof(int2)) +
                               S::round(a_cap * sizeof(double2)) + S::round(b_cap * sizeof(int2)) +
                               S::round(b_cap * sizeof(DeferredPair)) + S::round(a_cap * sizeof(int32_t)) +
                               S::round(offsetof(FpfhHead, a) + a_cap * sizeof(double4));
    Scratch sc(stream, 2 * S::round((n + 1) * sizeof(int32_t)) + S::round(33 * n * sizeof(double)) +
                           S::round(34 * n * sizeof(int32_t)) + 2 * S::round(4 * sizeof(int32_t)) + S::round(scan_bytes) +
                           (brute ? S::round(n * sizeof(int4)) + S::round(n * sizeof(uint32_t)) +
                                      S::round(n * kNbrSlots * sizeof(int32_t))
                                : 0) +
                           lists_bytes);
    int32_t* counts = sc.take<int32_t>(n + 1);
    int32_t* off = sc.take<int32_t>(n + 1);
    double* spfh = sc.take<double>(33 * n);
    int32_t* votes = sc.take<int32_t>(34 * n);
    int32_t* n_def = sc.take<int32_t>(4);
    int32_t* d_overflow = sc.take<int32_t>(4);
    void* scan_temp = sc.take<char>(scan_bytes);
    int4* cells = brute ? sc.take<int4>(n) : nullptr;
    uint32_t* cell_keys = brute ? sc.take<uint32_t>(n) : nullptr;
    int32_t* slots = brute ? sc.take<int32_t>(n * kNbrSlots) : nullptr;
    LK_TRY(sc.status());
    if (brute) {
        // SearchGrid(cell = radius): block radius ceil(radius / cell) = 1;
        // one pass counts and keeps the lists in a fixed-stride table
        k_search_cells<<<nblocks(n, 256), 256, 0, stream>>>(d_pos, n, radius, cells, off, n_def, d_overflow,
                                                            cell_keys);
        k_nbr_brute_once<<<nblocks(n, kSortWarps), 32 * kSortWarps, 0, stream>>>(d_pos, cells, cell_keys, n, 1, r2,
                                                                                 counts, slots, d_overflow);
    } else {
        LK_TRY(build_grid(g, 1, d_pos, nullptr, n, radius, radius, stream, false));
        k_nbr_count<<<nblocks(n, kSortWarps), 32 * kSortWarps, 0, stream>>>(d_pos, n, g.view, r2, counts);
    }
    LK_TRY(exclusive_scan(counts, n, off, stream, scan_temp, scan_bytes, !brute));
    trace_point("fpfh nbr", stream);
    int32_t* nbr = nullptr;
    DeferLists dl{};
    FpfhHead* head_dev = nullptr;  // dl.a2_x = head_dev->a
    bool pooled = false;  // this attempt's lists come from the pool (the retry)
    auto free_lists = [&] {
        if (!pooled) return;
        cudaFreeAsync(nbr, stream);
        cudaFreeAsync(dl.a_ij, stream);
        cudaFreeAsync(dl.a_x, stream);
        cudaFreeAsync(dl.b_ij, stream);
        cudaFreeAsync(dl.b_x, stream);
        cudaFreeAsync(dl.a_dec, stream);
        cudaFreeAsync(head_dev, stream);
    };
    for (int attempt = 0; attempt < 2; ++attempt) {
        if (attempt == 0) {
            nbr = sc.take<int32_t>(cap);
            dl.a_ij = sc.take<int2>(a_cap);
            dl.a_x = sc.take<double2>(a_cap);
            dl.b_ij = sc.take<int2>(b_cap);
            dl.b_x = sc.take<DeferredPair>(b_cap);
            dl.a_dec = sc.take<int32_t>(a_cap);
            head_dev = reinterpret_cast<FpfhHead*>(sc.take<char>(offsetof(FpfhHead, a) + a_cap * sizeof(double4)));
            LK_TRY(sc.status());
        } else {
            pooled = true;
            LK_TRY(cudaMallocAsync(&nbr, cap * sizeof(int32_t), stream));
            LK_TRY(cudaMallocAsync(&dl.a_ij, a_cap * sizeof(int2), stream));
            LK_TRY(cudaMallocAsync(&dl.a_x, a_cap * sizeof(double2), stream));
            LK_TRY(cudaMallocAsync(&dl.b_ij, b_cap * sizeof(int2), stream));
            LK_TRY(cudaMallocAsync(&dl.b_x, b_cap * sizeof(DeferredPair), stream));
            LK_TRY(cudaMallocAsync(&dl.a_dec, a_cap * sizeof(int32_t), stream));
            LK_TRY(cudaMallocAsync(&head_dev, offsetof(FpfhHead, a) + a_cap * sizeof(double4), stream));
        }
        if (!head_dev) return cudaErrorMemoryAllocation;
        dl.a2_x = head_dev->a;
        dl.n = n_def;
        dl.a_cap = a_cap;
        dl.b_cap = b_cap;
        // zeroed by k_search_cells on the brute path's first attempt
        if (!brute || attempt > 0) LK_TRY(cudaMemsetAsync(n_def, 0, 4 * sizeof(int32_t), stream));
        if (brute && attempt == 0)
            k_nbr_compact<<<nblocks(32 * n, 256), 256, 0, stream>>>(slots, off, n, d_overflow, nbr, cap);
        else if (brute)
            k_nbr_brute<true><<<nblocks(n, kSortWarps), 32 * kSortWarps, 0, stream>>>(d_pos, cells, n, 1, r2, nullptr,
                                                                                      off, nbr, cap);
        else
            k_nbr_fill<<<nblocks(n, kSortWarps), 32 * kSortWarps, 0, stream>>>(d_pos, n, g.view, r2, off, nbr, cap);
        // an overflowed slot table leaves nbr unfilled: the votes are skipped too
        k_spfh<<<nblocks(n, kFpfhWarps), 32 * kFpfhWarps, 0, stream>>>(d_pos, d_nrm, n, off, nbr, votes, dl, cap,
                                                                       (brute && attempt == 0) ? d_overflow : nullptr);
        trace_point("fpfh spfh", stream);
        k_spfh_decide_a<<<nblocks(a_cap, 256), 256, 0, stream>>>(dl, off + n,
                                                                 (brute && attempt == 0) ? d_overflow : nullptr,
                                                                 head_dev);
        // one round trip: the counts and the heads of lists A2 and B
        LK_TRY(cudaMemcpyAsync(st.head, head_dev, sizeof(FpfhHead), cudaMemcpyDeviceToHost, stream));
        LK_TRY(cudaStreamSynchronize(stream));
        if (st.head->total <= cap && !st.head->overflow && st.head->n_a <= a_cap && st.head->n_b <= b_cap) break;
        free_lists();
        cap = std::max<int64_t>(cap, st.head->total);
        a_cap = std::max<int64_t>(a_cap, st.head->n_a);
        b_cap = std::max<int64_t>(b_cap, st.head->n_b);
    }
    // pairs the device cannot settle, decided with the reference's libm:
    // list A2 by its acos comparison (fpfh.cpp:28), list B whole (host_pair_bins)
    const int32_t na = st.head->n_a, ma = st.head->n_a2, mb = st.head->n_b;
    trace_point("fpfh head back", stream);
    if (const char* tr = std::getenv("LK_TRACE"); tr && tr[0] == '1')
        std::fprintf(stderr, "[lk fpfh] n %lld neighbours %d deferred: acos ties %d (host %d), theta edges %d\n",
                     static_cast<long long>(n), st.head->total, na, ma, mb);
    if (ma > 0) {
        const double4* xs = st.head->a;
        if (ma > kStageA) {
            if (static_cast<size_t>(ma) > st.more_cap) {
                if (st.more_a) cudaFreeHost(st.more_a);
                st.more_a = nullptr;
                st.more_cap = 0;
                LK_TRY(cudaHostAlloc(reinterpret_cast<void**>(&st.more_a), ma * sizeof(double4), 0));
                st.more_cap = ma;
            }
            LK_TRY(cudaMemcpyAsync(st.more_a + kStageA, dl.a2_x + kStageA,
                                   (ma - kStageA) * sizeof(double4), cudaMemcpyDeviceToHost, stream));
            std::memcpy(st.more_a, st.head->a, kStageA * sizeof(double4));
            LK_TRY(cudaStreamSynchronize(stream));
            xs = st.more_a;
        }
        if (static_cast<size_t>(ma) > st.dec_a_cap) {
            if (st.dec_a) cudaFreeHost(st.dec_a);
            st.dec_a = nullptr;
            st.dec_a_cap = 0;
            LK_TRY(cudaHostAlloc(reinterpret_cast<void**>(&st.dec_a), ma, 0));
            st.dec_a_cap = ma;
        }
#pragma omp parallel for schedule(static) if (ma > 4096)
        for (int32_t k = 0; k < ma; ++k) {
            const double g1 = std::isnan(xs[k].z) ? std::acos(xs[k].x) : xs[k].z;
            const double g2 = std::isnan(xs[k].w) ? std::acos(xs[k].y) : xs[k].w;
            st.dec_a[k] = g1 > g2 ? 1 : 0;
        }
    }
    // the host's decisions are read by the kernels from the page-locked
    // staging in place (a few bytes each: no copy command)
    if (na > 0)
        k_spfh_resolve_a<<<nblocks(na, 256), 256, 0, stream>>>(d_pos, d_nrm, dl.a_ij, dl.a_dec, st.dec_a, na, votes);
    if (mb > 0) {
        std::vector<DeferredPair> more;
        const DeferredPair* xs = st.head->b;
        if (mb > kStageB) {
            more.resize(mb);
            LK_TRY(cudaMemcpyAsync(more.data(), dl.b_x, mb * sizeof(DeferredPair), cudaMemcpyDeviceToHost, stream));
            LK_TRY(cudaStreamSynchronize(stream));
            xs = more.data();
        }
        if (static_cast<size_t>(mb) > st.dec_b_cap) {
            if (st.dec_b) cudaFreeHost(st.dec_b);
            st.dec_b = nullptr;
            st.dec_b_cap = 0;
            LK_TRY(cudaHostAlloc(reinterpret_cast<void**>(&st.dec_b), mb * sizeof(uint32_t), 0));
            st.dec_b_cap = mb;
        }
        for (int32_t k = 0; k < mb; ++k) st.dec_b[k] = host_pair_bins(xs[k].v);
        k_spfh_resolve_b<<<nblocks(mb, 256), 256, 0, stream>>>(dl.b_ij, st.dec_b, mb, votes);
    }
    trace_point("fpfh resolved", stream);
    k_spfh_scale<<<nblocks(33 * n, 256), 256, 0, stream>>>(votes, n, spfh);
    k_fpfh<<<nblocks(n, kFpfhWarps), 32 * kFpfhWarps, 0, stream>>>(d_pos, d_nrm, n, off, nbr, spfh, d_out);
    LK_TRY(cudaGetLastError());
    // stream-ordered frees: nothing here waits for the device (the pinned
    // staging is reused only after the caller synchronises this stream)
    free_lists();
    g.release();
    return cudaGetLastError();
}

cudaError_t cloud_stats_async(const double* d_pos, const double* d_nrm, int64_t n, unsigned long long* h_out2,
                              cudaStream_t stream) {
    Scratch sc(stream, Scratch::round(2 * sizeof(unsigned long long)));
    unsigned long long* d = sc.take<unsigned long long>(2);
    LK_TRY(sc.status());
    LK_TRY(cudaMemsetAsync(d, 0, 2 * sizeof(unsigned long long), stream));
    k_cloud_stats<<<nblocks(n, 256) < 64 ? nblocks(n, 256) : 64, 256, 0, stream>>>(d_pos, d_nrm, n, d);
    LK_TRY(cudaMemcpyAsync(h_out2, d, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream));
    return cudaGetLastError();
}

void cloud_stats_decode(const unsigned long long* h2, int64_t* usable, double* max_norm) {
    *usable = static_cast<int64_t>(h2[0]);
    const long long bits = static_cast<long long>(h2[1]);
    std::memcpy(max_norm, &bits, sizeof(double));
}

cudaError_t cloud_stats(const double* d_pos, const double* d_nrm, int64_t n, int64_t* usable, double* max_norm,
                        cudaStream_t stream) {
    unsigned long long h[2] = {0, 0};
    LK_TRY(cloud_stats_async(d_pos, d_nrm, n, h, stream));
    LK_TRY(cudaStreamSynchronize(stream));
    cloud_stats_decode(h, usable, max_norm);
    return cudaGetLastError();
}

}  // namespace lkk
