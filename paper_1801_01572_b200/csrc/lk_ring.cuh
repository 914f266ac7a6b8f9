// lk_ring.cuh -- device query of the ring grid (lk_ring.cu): the reference
// EvalGrid's nearest neighbour within d_max (registration.cpp:165-199
// semantics) for dense targets. See lk_ring.cu for the exactness argument.
#pragma once

#include <cstdint>

#include "lk_device_math.cuh"
#include "lk_kernels.cuh"

namespace lkk {

// Cells c along one axis whose entries ([c - delta, c + 1 + delta]) can lie
// within h of q: c in [lo, hi]. h carries a relative and an absolute slack
// over sqrt(rem) so that every cell the per-cell FP32 test
// (gap^2 + rest <= bound) would pass is inside: the range is a superset.
__device__ __forceinline__ void ring_reach(float q, float dl, float rem, float bnd, int& lo, int& hi) {
    // sqrt.approx (relative error ~2^-22) is far inside the slack
    float h;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(h) : "f"(fmaxf(rem, 0.0f) * 1.0001f + bnd * 1e-5f));
    h += 1e-3f;
    lo = static_cast<int>(ceilf(q - dl - h - 1.0f));
    hi = static_cast<int>(floorf(q + dl + h));
}

// Visits the entries of the cells of the cube shell of radius r around
// (cx, cy, cz) that can hold a point within sqrt(bound()) cells of q: a
// cell's entries lie within [c - delta, c + 1 + delta] per axis, so a row or
// cell whose box is farther than that from q is skipped without loading it;
// a row's reachable cells are one contiguous CSR range. The bound is re-read
// row by row (it shrinks as the best improves).
template <class B, class F>
__device__ __forceinline__ void ring_shell(const RingGrid& rg, float qx, float qy, float qz, int cx, int cy, int cz,
                                           int r, B&& bound, F&& f) {
    const float dl = rg.delta;
    auto gap = [dl](float q, int c) {  // distance from q to [c - dl, c + 1 + dl]
        const float lo = static_cast<float>(c) - dl, hi = static_cast<float>(c + 1) + dl;
        return q < lo ? lo - q : (q > hi ? q - hi : 0.0f);
    };
    for (int dx = -r; dx <= r; ++dx) {
        const int x = cx + dx;
        if (x < 0 || x >= rg.nx) continue;
        const float gx = gap(qx, x);
        if (gx * gx > bound()) continue;
        for (int dy = -r; dy <= r; ++dy) {
            const int y = cy + dy;
            if (y < 0 || y >= rg.ny) continue;
            const float gy = gap(qy, y);
            const float gxy = gx * gx + gy * gy;
            if (gxy > bound()) continue;
            const int64_t row = (static_cast<int64_t>(x) * rg.ny + y) * rg.nz;
            const bool edge = dx == -r || dx == r || dy == -r || dy == r;
            // the cells of the row the bound reaches (a superset of the
            // per-cell test): one contiguous CSR range per row
            int lz, hz;
            ring_reach(qz, dl, bound() - gxy, bound(), lz, hz);
            if (edge) {
                int z0 = cz - r > lz ? cz - r : lz, z1 = cz + r < hz ? cz + r : hz;
                z0 = z0 > 0 ? z0 : 0;
                z1 = z1 < rg.nz - 1 ? z1 : rg.nz - 1;
                if (z0 <= z1) {
                    const int32_t s0 = __ldg(rg.start + row + z0), s1 = __ldg(rg.start + row + z1 + 1);
                    for (int32_t e = s0; e < s1; ++e) f(e);
                }
            } else {
                for (int z = cz - r; z <= cz + r; z += 2 * r) {  // r > 0 here: the shell's two caps
                    if (z < 0 || z >= rg.nz || z < lz || z > hz) continue;
                    const int32_t s0 = __ldg(rg.start + row + z), s1 = __ldg(rg.start + row + z + 1);
                    for (int32_t e = s0; e < s1; ++e) f(e);
                }
            }
        }
    }
}

__device__ __forceinline__ int ecell_axis(double v, double o, double c) { return static_cast<int>(floor((v - o) / c)); }

// exact scan of the reference window (the +-ewin reference cells of y's cell)
static __device__ __noinline__ int32_t ring_window_scan(const RingGrid& rg, lkd::V3 y, double d2_max, int ex, int ey,
                                                 int ez) {
    using namespace lkd;
    const int w = rg.ewin;
    const double lx = rg.eox + (ex - w) * rg.ecell, hx = rg.eox + (ex + w + 1) * rg.ecell;
    const double ly = rg.eoy + (ey - w) * rg.ecell, hy = rg.eoy + (ey + w + 1) * rg.ecell;
    const double lz = rg.eoz + (ez - w) * rg.ecell, hz = rg.eoz + (ez + w + 1) * rg.ecell;
    auto clampc = [](double v, int n) {
        return v < 0.0 ? 0 : (v >= static_cast<double>(n) ? n - 1 : static_cast<int>(v));
    };
    const int x0 = clampc(floor((lx - rg.ox) / rg.cell) - 1.0, rg.nx);
    const int x1 = clampc(floor((hx - rg.ox) / rg.cell) + 1.0, rg.nx);
    const int y0 = clampc(floor((ly - rg.oy) / rg.cell) - 1.0, rg.ny);
    const int y1 = clampc(floor((hy - rg.oy) / rg.cell) + 1.0, rg.ny);
    const int z0 = clampc(floor((lz - rg.oz) / rg.cell) - 1.0, rg.nz);
    const int z1 = clampc(floor((hz - rg.oz) / rg.cell) + 1.0, rg.nz);
    double best_d2 = __longlong_as_double(0x7ff0000000000000ll);
    int32_t best = INT32_MAX;
    for (int x = x0; x <= x1; ++x)
        for (int yy = y0; yy <= y1; ++yy) {
            const int64_t row = (static_cast<int64_t>(x) * rg.ny + yy) * rg.nz;
            for (int32_t e = rg.start[row + z0]; e < rg.start[row + z1 + 1]; ++e) {
                const int32_t o = __float_as_int(rg.pts[e].w);
                const V3 q = ld4(rg.pos4, o);
                const int qx = ecell_axis(q.x, rg.eox, rg.ecell), qy = ecell_axis(q.y, rg.eoy, rg.ecell),
                          qz = ecell_axis(q.z, rg.eoz, rg.ecell);
                if (qx < ex - w || qx > ex + w || qy < ey - w || qy > ey + w || qz < ez - w || qz > ez + w) continue;
                const double d2 = sqnorm(sub(q, y));
                if (d2 > d2_max) continue;
                if (d2 < best_d2 || (d2 == best_d2 && o < best)) {
                    best_d2 = d2;
                    best = o;
                }
            }
        }
    return best == INT32_MAX ? -1 : best;
}

__device__ __forceinline__ void ring_top3(float d2, int32_t o, float& f1, float& f2, float& f3, int32_t& o1,
                                          int32_t& o2) {
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

// FP32 d2 up to which an entry may still be the FP64 nearest (or tie it),
// given the FP32 best f1: the guard band of lk_ring.cu's ring_frame, but for
// distances up to D = sqrt(f1 + band) (every such entry, and the FP32 best
// itself, is within D) instead of the walk's worst case rmax + 1 cells -- so
// the FP64 candidate set, and the re-scans when it exceeds two, stay small.
__device__ __forceinline__ float ring_lim(const RingGrid& rg, float f1) {
    if (!(rg.band < 1e29f)) return f1 + 2.0f * rg.band;  // FP64-only mode: every entry within d_max
    const float D = sqrtf(f1 + rg.band) * 1.001f + 1e-4f;
    const float e = 4.0f * (2.0f * 1.7320508f * D * rg.delta + 3.0f * rg.delta * rg.delta +
                            4.0f * 5.9604645e-8f * D * D) + 1e-6f;
    return f1 + 2.02f * e;
}

// Original index of the reference EvalGrid neighbour of y within d_max, or -1.
__device__ __forceinline__ int32_t ring_nn(const RingGrid& rg, lkd::V3 y, double d2_max) {
    using namespace lkd;
    // the reference's cell of y; an EvalGrid query outside the grid misses
    // (registration.cpp:167-172)
    const double fx = floor((y.x - rg.eox) / rg.ecell), fy = floor((y.y - rg.eoy) / rg.ecell),
                 fz = floor((y.z - rg.eoz) / rg.ecell);
    if (rg.ebounded && !(fx >= 0.0 && fy >= 0.0 && fz >= 0.0 && fx < rg.enx && fy < rg.eny && fz < rg.enz))
        return -1;
    const float qx = static_cast<float>((y.x - rg.ox) / rg.cell);
    const float qy = static_cast<float>((y.y - rg.oy) / rg.cell);
    const float qz = static_cast<float>((y.z - rg.oz) / rg.cell);
    const int cx = static_cast<int>(floorf(qx)), cy = static_cast<int>(floorf(qy)), cz = static_cast<int>(floorf(qz));
    // shells below the cell's distance to the nearest occupied cell are empty;
    // every entry lies >= k0 - 1 - delta cells away on some axis
    int k0 = 0;
    if (rg.dt && cx >= 0 && cx < rg.nx && cy >= 0 && cy < rg.ny && cz >= 0 && cz < rg.nz) {
        k0 = __ldg(rg.dt + (static_cast<int64_t>(cx) * rg.ny + cy) * rg.nz + cz);
        const float m = static_cast<float>(k0 - 1) - rg.delta;
        if (m > 0.0f && m * m > rg.thr + 2.0f * rg.band) return -1;
    }
    const float inf = __int_as_float(0x7f800000);
    float f1 = inf, f2 = inf, f3 = inf;
    int32_t o1 = -1, o2 = -1;
    int r_end = k0;
    // entries farther than this (squared cells) can be neither the nearest,
    // nor tied with it, nor within d_max
    auto bound = [&]() { return fminf(f1 + 2.0f * rg.band, rg.thr + rg.band); };
    for (int r = k0; r <= rg.rmax; ++r) {
        ring_shell(rg, qx, qy, qz, cx, cy, cz, r, bound, [&](int32_t e) {
            const float4 A = __ldg(rg.pts + e);
            const float dx = qx - A.x, dy = qy - A.y, dz = qz - A.z;
            ring_top3(fmaf(dx, dx, fmaf(dy, dy, dz * dz)), __float_as_int(A.w), f1, f2, f3, o1, o2);
        });
        r_end = r;
        // every entry outside the scanned cube lies >= r - delta cells away
        const float m = static_cast<float>(r) - rg.delta;
        if (m > 0.0f && m * m > bound()) break;
    }
    if (f1 > rg.thr + rg.band) return -1;
    double best_d2 = __longlong_as_double(0x7ff0000000000000ll);
    int32_t best = INT32_MAX;
    auto consider = [&](int32_t o) {
        const V3 q = ld4(rg.pos4, o);
        const double d2 = sqnorm(sub(q, y));
        if (d2 > d2_max) return;
        if (d2 < best_d2 || (d2 == best_d2 && o < best)) {
            best_d2 = d2;
            best = o;
        }
    };
    const float lim = ring_lim(rg, f1);
    if (f3 <= lim) {
        auto lim_bound = [&]() { return lim; };
        for (int r = k0; r <= r_end; ++r)
            ring_shell(rg, qx, qy, qz, cx, cy, cz, r, lim_bound, [&](int32_t e) {
                const float4 A = __ldg(rg.pts + e);
                const float dx = qx - A.x, dy = qy - A.y, dz = qz - A.z;
                if (fmaf(dx, dx, fmaf(dy, dy, dz * dz)) <= lim) consider(__float_as_int(A.w));
            });
    } else {
        consider(o1);
        if (f2 <= lim) consider(o2);
    }
    if (best == INT32_MAX) return -1;
    // the reference only sees its window: a nearest point outside it (a
    // division rounded across a face) sends the query to the exact window scan
    const V3 q = ld4(rg.pos4, best);
    const int ex = static_cast<int>(fx), ey = static_cast<int>(fy), ez = static_cast<int>(fz);
    const int wx = ecell_axis(q.x, rg.eox, rg.ecell), wy = ecell_axis(q.y, rg.eoy, rg.ecell),
              wz = ecell_axis(q.z, rg.eoz, rg.ecell);
    const int w = rg.ewin;
    if (wx < ex - w || wx > ex + w || wy < ey - w || wy > ey + w || wz < ez - w || wz > ez + w)
        return ring_window_scan(rg, y, d2_max, ex, ey, ez);
    return best;
}

// ---- warp-cooperative query ---------------------------------------------
// All 32 lanes call ring_nn_warp together, each with its own query (active =
// false: no query, -1). When the live queries' cells span at most
// kWarpSpan cells per axis (queries in a spatially coherent order), the warp
// scans cube shells around their common cell box instead of one walk per
// lane: a cell is visited when any live lane's guard-banded bound reaches it,
// its entries are loaded once (coalesced) and broadcast, and every lane keeps
// its own FP32 top three. Scanning a superset of a lane's own walk keeps each
// decision of ring_nn: the same stop rule per lane (every unscanned entry is
// >= margin - delta cells away), the same band re-scan and FP64 choice, the
// same window check. Wider warps fall back to ring_nn per lane.
constexpr int kWarpSpan = 24;  // row hulls make wide boxes cheap (B2: 24 beats 6 by ~15%)

__device__ __forceinline__ void ring_top3_sel(float d2, int32_t o, float& f1, float& f2, float& f3, int32_t& o1,
                                              int32_t& o2) {
    const bool c1 = d2 < f1, c2 = d2 < f2, c3 = d2 < f3;
    f3 = c2 ? f2 : (c3 ? d2 : f3);
    o2 = c1 ? o1 : (c2 ? o : o2);
    f2 = c1 ? f1 : (c2 ? d2 : f2);
    o1 = c1 ? o : o1;
    f1 = c1 ? d2 : f1;
}

// Visits the cells of shell r around the box [b0, b1] (r = 0: the box) that
// some participating lane's bound reaches; visit(chunk, cnt) per staged chunk
// of up to 32 entries (chunk: x[32] y[32] z[32] index[32] in shared memory).
// Row by row: each lane turns its bound into the z range of cells it can
// reach in the (x, y) row, the warp takes the hull of those ranges, and the
// hull's entries -- contiguous in the CSR -- are streamed with two start[]
// reads per row instead of a box test and two reads per cell (empty cells
// cost nothing). Rows strictly inside the shell only add their Z0 / Z1 cells.
// The y range per x is pruned the same way. Hulls are supersets of the
// per-cell test, which keeps every decision (see ring_nn_warp).
template <class B, class F>
__device__ __forceinline__ void warp_shell(const RingGrid& rg, float qx, float qy, float qz, bool part, const int* b0,
                                           const int* b1, int r, float4* wbuf, B&& bound, F&& visit) {
    constexpr unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const float dl = rg.delta;
    auto gap = [dl](float q, int c) {
        const float lo = static_cast<float>(c) - dl, hi = static_cast<float>(c + 1) + dl;
        return q < lo ? lo - q : (q > hi ? q - hi : 0.0f);
    };
    float* xs = reinterpret_cast<float*>(wbuf);  // staged chunk, SoA: x[32] y[32] z[32] index[32]
    auto scan = [&](int64_t row, int za, int zb) {
        const int32_t s0 = __ldg(rg.start + row + za), s1 = __ldg(rg.start + row + zb + 1);
        // stage 32 entries (one coalesced load), read back as broadcasts; the
        // next chunk's load is in flight while this one is visited
        float4 A = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        if (s0 + lane < s1) A = __ldg(rg.pts + s0 + lane);
        for (int32_t base = s0; base < s1; base += 32) {
            const int32_t e = base + lane;
            __syncwarp();
            if (e < s1) {
                xs[lane] = A.x;
                xs[32 + lane] = A.y;
                xs[64 + lane] = A.z;
                xs[96 + lane] = A.w;
            }
            __syncwarp();
            if (e + 32 < s1) A = __ldg(rg.pts + e + 32);
            visit(xs, s1 - base < 32 ? s1 - base : 32);
        }
    };
    const int X0 = b0[0] - r, X1 = b1[0] + r, Y0 = b0[1] - r, Y1 = b1[1] + r, Z0 = b0[2] - r, Z1 = b1[2] + r;
    const int xa = X0 > 0 ? X0 : 0, xb = X1 < rg.nx - 1 ? X1 : rg.nx - 1;
    const int ya = Y0 > 0 ? Y0 : 0, yb = Y1 < rg.ny - 1 ? Y1 : rg.ny - 1;
    const int za = Z0 > 0 ? Z0 : 0, zb = Z1 < rg.nz - 1 ? Z1 : rg.nz - 1;
    if (za > zb) return;
    for (int x = xa; x <= xb; ++x) {
        const float gx = gap(qx, x);
        const float bx = bound();
        const bool okx = part && gx * gx <= bx;
        if (!__any_sync(full, okx)) continue;
        const bool xe = r == 0 || x == X0 || x == X1;
        int ly, hy;
        ring_reach(qy, dl, bx - gx * gx, bx, ly, hy);
        int y0 = __reduce_min_sync(full, okx ? ly : INT32_MAX), y1 = __reduce_max_sync(full, okx ? hy : INT32_MIN);
        y0 = y0 > ya ? y0 : ya;
        y1 = y1 < yb ? y1 : yb;
        for (int y = y0; y <= y1; ++y) {
            const float gy = gap(qy, y);
            const float gxy = gx * gx + gy * gy;
            const float bxy = bound();
            const bool ok = part && gxy <= bxy;
            if (!__any_sync(full, ok)) continue;
            int lz, hz;
            ring_reach(qz, dl, bxy - gxy, bxy, lz, hz);
            const int64_t row = (static_cast<int64_t>(x) * rg.ny + y) * rg.nz;
            if (xe || y == Y0 || y == Y1) {
                int z0 = __reduce_min_sync(full, ok ? lz : INT32_MAX), z1 = __reduce_max_sync(full, ok ? hz : INT32_MIN);
                z0 = z0 > za ? z0 : za;
                z1 = z1 < zb ? z1 : zb;
                if (z0 <= z1) scan(row, z0, z1);
            } else {
                if (Z0 >= 0 && __any_sync(full, ok && lz <= Z0 && Z0 <= hz)) scan(row, Z0, Z0);
                if (Z1 < rg.nz && __any_sync(full, ok && lz <= Z1 && Z1 <= hz)) scan(row, Z1, Z1);
            }
        }
    }
}

// FP32 d2 of staged entries k and k + 1 (chunk SoA) from the negated query:
// fl(a - q) = -fl(q - a), so this is fmaf(dx, dx, fmaf(dy, dy, dz * dz)) bit
// for bit, two lanes of FFMA2 / FADD2 / FMUL2 per instruction.
__device__ __forceinline__ float2 ring_d2x2(const float2* nq, const float* ch, int k) {
    const float2 dx = __fadd2_rn(*reinterpret_cast<const float2*>(ch + k), nq[0]);
    const float2 dy = __fadd2_rn(*reinterpret_cast<const float2*>(ch + 32 + k), nq[1]);
    const float2 dz = __fadd2_rn(*reinterpret_cast<const float2*>(ch + 64 + k), nq[2]);
    return __ffma2_rn(dx, dx, __ffma2_rn(dy, dy, __fmul2_rn(dz, dz)));
}

// wbuf: 32 float4 of shared memory owned by the calling warp. hint: an entry
// (original index) likely near y -- e.g. the previous ICP iteration's match --
// or -1. It seeds the top three, so the bound starts at its distance instead
// of d_max and the box scan is pruned from the first row; any entry is a
// valid seed (it is a real candidate, and the walk skips it once).
__device__ __forceinline__ int32_t ring_nn_warp(const RingGrid& rg, lkd::V3 y, double d2_max, bool active,
                                                float4* wbuf, int32_t hint = -1) {
    using namespace lkd;
    constexpr unsigned full = 0xffffffffu;
    bool live = active;
    double fx = 0.0, fy = 0.0, fz = 0.0;
    if (live) {
        fx = floor((y.x - rg.eox) / rg.ecell);
        fy = floor((y.y - rg.eoy) / rg.ecell);
        fz = floor((y.z - rg.eoz) / rg.ecell);
        if (rg.ebounded && !(fx >= 0.0 && fy >= 0.0 && fz >= 0.0 && fx < rg.enx && fy < rg.eny && fz < rg.enz))
            live = false;
    }
    float qx = 0.0f, qy = 0.0f, qz = 0.0f;
    int c[3] = {0, 0, 0};
    if (live) {
        qx = static_cast<float>((y.x - rg.ox) / rg.cell);
        qy = static_cast<float>((y.y - rg.oy) / rg.cell);
        qz = static_cast<float>((y.z - rg.oz) / rg.cell);
        c[0] = static_cast<int>(floorf(qx));
        c[1] = static_cast<int>(floorf(qy));
        c[2] = static_cast<int>(floorf(qz));
        // every entry lies inside the grid's cells: a query more than rmax
        // cells outside has nothing within d_max
        if (c[0] < -rg.rmax || c[0] >= rg.nx + rg.rmax || c[1] < -rg.rmax || c[1] >= rg.ny + rg.rmax ||
            c[2] < -rg.rmax || c[2] >= rg.nz + rg.rmax)
            live = false;
    }
    if (live && rg.dt && c[0] >= 0 && c[0] < rg.nx && c[1] >= 0 && c[1] < rg.ny && c[2] >= 0 && c[2] < rg.nz) {
        const int k0 = __ldg(rg.dt + (static_cast<int64_t>(c[0]) * rg.ny + c[1]) * rg.nz + c[2]);
        const float m = static_cast<float>(k0 - 1) - rg.delta;
        if (m > 0.0f && m * m > rg.thr + 2.0f * rg.band) live = false;
    }
    if (!__any_sync(full, live)) return -1;
    int b0[3], b1[3];
    bool wide = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        b0[a] = __reduce_min_sync(full, live ? c[a] : INT32_MAX);
        b1[a] = __reduce_max_sync(full, live ? c[a] : INT32_MIN);
        wide = wide || b1[a] - b0[a] > kWarpSpan;
    }
    if (wide) return live ? ring_nn(rg, y, d2_max) : -1;
    const float inf = __int_as_float(0x7f800000);
    float f1 = inf, f2 = inf, f3 = inf;
    int32_t o1 = -1, o2 = -1;
    const int32_t seed = live && hint >= 0 && hint < rg.npoints ? hint : -1;
    if (seed >= 0) {  // the same FP32 cell coordinates as the entry's (k_ring_scatter)
        const V3 p = ld4(rg.pos4, seed);
        const float dx = qx - static_cast<float>((p.x - rg.ox) / rg.cell);
        const float dy = qy - static_cast<float>((p.y - rg.oy) / rg.cell);
        const float dz = qz - static_cast<float>((p.z - rg.oz) / rg.cell);
        f1 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
        o1 = seed;
    }
    auto bound = [&]() { return fminf(f1 + 2.0f * rg.band, rg.thr + rg.band); };
    const float2 nq[3] = {make_float2(-qx, -qx), make_float2(-qy, -qy), make_float2(-qz, -qz)};
    int r_end = 0;
    // r = rmax covers every lane's own walk (its cell +- rmax)
    for (int r = 0; r <= rg.rmax; ++r) {
        warp_shell(rg, qx, qy, qz, live, b0, b1, r, wbuf, bound, [&](const float* ch, int cnt) {
            // two entries per step in packed FP32 (the same roundings as the
            // scalar fmaf(dx, dx, fmaf(dy, dy, dz * dz))); the top three are
            // only touched when some live lane sees an entry below its third
            int k = 0;
            for (; k + 4 <= cnt; k += 4) {
                const float2 da = ring_d2x2(nq, ch, k), db = ring_d2x2(nq, ch, k + 2);
                if (__any_sync(full, live && fminf(fminf(da.x, da.y), fminf(db.x, db.y)) < f3)) {
                    const int4 o = *reinterpret_cast<const int4*>(ch + 96 + k);
                    ring_top3_sel(o.x == seed ? inf : da.x, o.x, f1, f2, f3, o1, o2);
                    ring_top3_sel(o.y == seed ? inf : da.y, o.y, f1, f2, f3, o1, o2);
                    ring_top3_sel(o.z == seed ? inf : db.x, o.z, f1, f2, f3, o1, o2);
                    ring_top3_sel(o.w == seed ? inf : db.y, o.w, f1, f2, f3, o1, o2);
                }
            }
            for (; k + 2 <= cnt; k += 2) {
                const float2 d2 = ring_d2x2(nq, ch, k);
                if (__any_sync(full, live && fminf(d2.x, d2.y) < f3)) {
                    const int2 o = *reinterpret_cast<const int2*>(ch + 96 + k);
                    ring_top3_sel(o.x == seed ? inf : d2.x, o.x, f1, f2, f3, o1, o2);
                    ring_top3_sel(o.y == seed ? inf : d2.y, o.y, f1, f2, f3, o1, o2);
                }
            }
            if (k < cnt) {
                const float dx = qx - ch[k], dy = qy - ch[32 + k], dz = qz - ch[64 + k];
                const int32_t o = __float_as_int(ch[96 + k]);
                ring_top3_sel(o == seed ? inf : fmaf(dx, dx, fmaf(dy, dy, dz * dz)), o, f1, f2, f3, o1, o2);
            }
        });
        r_end = r;
        // entries outside the scanned box lie >= m - delta cells from the query
        const float mx = fminf(qx - static_cast<float>(b0[0] - r), static_cast<float>(b1[0] + r + 1) - qx);
        const float my = fminf(qy - static_cast<float>(b0[1] - r), static_cast<float>(b1[1] + r + 1) - qy);
        const float mz = fminf(qz - static_cast<float>(b0[2] - r), static_cast<float>(b1[2] + r + 1) - qz);
        const float m = fminf(mx, fminf(my, mz)) - rg.delta;
        if (__all_sync(full, !live || (m > 0.0f && m * m > bound()))) break;
    }
    const bool hit = live && f1 <= rg.thr + rg.band;
    const float lim = ring_lim(rg, f1);
    double best_d2 = __longlong_as_double(0x7ff0000000000000ll);
    int32_t best = INT32_MAX;
    auto consider = [&](int32_t o) {
        const V3 q = ld4(rg.pos4, o);
        const double d2 = sqnorm(sub(q, y));
        if (d2 > d2_max) return;
        if (d2 < best_d2 || (d2 == best_d2 && o < best)) {
            best_d2 = d2;
            best = o;
        }
    };
    const bool resc = hit && f3 <= lim;
    if (__any_sync(full, resc)) {
        auto lim_bound = [&]() { return lim; };
        for (int r = 0; r <= r_end; ++r)
            warp_shell(rg, qx, qy, qz, resc, b0, b1, r, wbuf, lim_bound, [&](const float* ch, int cnt) {
                int k = 0;
                for (; k + 2 <= cnt; k += 2) {
                    const float2 d2 = ring_d2x2(nq, ch, k);
                    if (__any_sync(full, resc && fminf(d2.x, d2.y) <= lim)) {
                        const int2 o = *reinterpret_cast<const int2*>(ch + 96 + k);
                        if (resc && d2.x <= lim) consider(o.x);
                        if (resc && d2.y <= lim) consider(o.y);
                    }
                }
                if (k < cnt) {
                    const float dx = qx - ch[k], dy = qy - ch[32 + k], dz = qz - ch[64 + k];
                    if (resc && fmaf(dx, dx, fmaf(dy, dy, dz * dz)) <= lim) consider(__float_as_int(ch[96 + k]));
                }
            });
    }
    if (hit && !resc) {
        consider(o1);
        if (f2 <= lim) consider(o2);
    }
    if (!hit || best == INT32_MAX) return -1;
    const V3 q = ld4(rg.pos4, best);
    const int ex = static_cast<int>(fx), ey = static_cast<int>(fy), ez = static_cast<int>(fz);
    const int wx = ecell_axis(q.x, rg.eox, rg.ecell), wy = ecell_axis(q.y, rg.eoy, rg.ecell),
              wz = ecell_axis(q.z, rg.eoz, rg.ecell);
    const int w = rg.ewin;
    if (wx < ex - w || wx > ex + w || wy < ey - w || wy > ey + w || wz < ez - w || wz > ez + w)
        return ring_window_scan(rg, y, d2_max, ex, ey, ez);
    return best;
}

}  // namespace lkk
