// lk_oracle.cpp -- TEST INFRASTRUCTURE ONLY (see lk_oracle.h).
//
// A line-by-line FP64 CPU restatement of the reference registration path.
// Every function cites the reference file:line it restates (paths relative to
// /root/reference/proj). Eigen is absent, so its expression evaluation order
// is restated explicitly:
//   * dot / squaredNorm of 3-vectors:   (a0 + a1) + a2
//   * Matrix3d * Vector3d, row r<2:     ((m_r0 v0 + m_r1 v1) + m_r2 v2)
//                              row 2:   m_20 v0 + (m_21 v1 + m_22 v2)
//   * Matrix3d * Matrix3d: per result column, the same row rule.
// Built with -O2 -fopenmp -ffp-contract=off and no -march (as the reference
// build: proj/CMakeLists.txt:8-10,34), so no FMA contraction.

#include "lk_oracle.h"

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include <omp.h>

namespace orc {

// ---------------------------------------------------------------- errors
// proj/include/loopkit/errors.hpp:9-74
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] static void fail(int code, const std::string& m) { throw Error(code, m); }

static thread_local std::string g_last_error;

// ---------------------------------------------------------------- vec3
struct V3 {
    double x = 0, y = 0, z = 0;
    double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
    double& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
};
static inline V3 v3(double a, double b, double c) { return V3{a, b, c}; }
static inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
static inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
static inline V3 neg(V3 a) { return {-a.x, -a.y, -a.z}; }
static inline V3 divs(V3 a, double s) { return {a.x / s, a.y / s, a.z / s}; }
static inline double dot(V3 a, V3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
static inline double sqnorm(V3 a) { return (a.x * a.x + a.y * a.y) + a.z * a.z; }
static inline double norm(V3 a) { return std::sqrt(sqnorm(a)); }
static inline bool is_zero(V3 a) { return a.x == 0.0 && a.y == 0.0 && a.z == 0.0; }
// Eigen cross3 (scalar path)
static inline V3 cross(V3 a, V3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
static inline V3 load3(const double* p, int64_t i) { return {p[3 * i], p[3 * i + 1], p[3 * i + 2]}; }
static inline void store3(double* p, int64_t i, V3 v) {
    p[3 * i] = v.x;
    p[3 * i + 1] = v.y;
    p[3 * i + 2] = v.z;
}

// ---------------------------------------------------------------- mat3
struct M3 {
    double m[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};  // m[row][col]
};
static inline M3 ident() {
    M3 r;
    r.m[0][0] = r.m[1][1] = r.m[2][2] = 1.0;
    return r;
}
static inline M3 load_m(const double* R9) {
    M3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[i][j] = R9[3 * i + j];
    return r;
}
static inline void store_m(double* R9, const M3& r) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) R9[3 * i + j] = r.m[i][j];
}
static inline M3 transpose(const M3& a) {
    M3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[j][i];
    return r;
}
// Matrix3d * Vector3d (Appendix A.3)
static inline V3 mul(const M3& a, V3 v) {
    V3 r;
    r.x = (a.m[0][0] * v.x + a.m[0][1] * v.y) + a.m[0][2] * v.z;
    r.y = (a.m[1][0] * v.x + a.m[1][1] * v.y) + a.m[1][2] * v.z;
    r.z = a.m[2][0] * v.x + (a.m[2][1] * v.y + a.m[2][2] * v.z);
    return r;
}
// Matrix3d * Matrix3d: per column j, rows 0-1 packet order, row 2 scalar order.
static inline M3 mul(const M3& a, const M3& b) {
    M3 r;
    for (int j = 0; j < 3; ++j) {
        for (int i = 0; i < 2; ++i)
            r.m[i][j] = (a.m[i][0] * b.m[0][j] + a.m[i][1] * b.m[1][j]) + a.m[i][2] * b.m[2][j];
        r.m[2][j] = a.m[2][0] * b.m[0][j] + (a.m[2][1] * b.m[1][j] + a.m[2][2] * b.m[2][j]);
    }
    return r;
}
// Eigen determinant_impl<3> (bruteforce_det3_helper)
static inline double det(const M3& a) {
    auto h = [&](int x, int y, int z) { return a.m[0][x] * (a.m[1][y] * a.m[2][z] - a.m[1][z] * a.m[2][y]); };
    return h(0, 1, 2) - h(1, 0, 2) + h(2, 0, 1);
}

struct Rigid {
    M3 R = ident();
    V3 t{};
};
// RigidTransform::operator* (geometry.hpp:26): rotation * p + translation
static inline V3 apply(const Rigid& T, V3 p) { return add(mul(T.R, p), T.t); }
static inline Rigid load_rigid(const double* R9, const double* t3) {
    Rigid T;
    T.R = load_m(R9);
    T.t = v3(t3[0], t3[1], t3[2]);
    return T;
}

// ---------------------------------------------------------------- RNG
// proj/include/loopkit/rng.hpp:14-46
static inline uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
struct Rng {
    uint64_t state;
    uint64_t counter = 0;
    Rng(uint64_t seed, uint64_t stream) : state(splitmix64(splitmix64(seed) ^ (stream * 0xd1342543de82ef95ull))) {}
    uint64_t next_u64() {
        counter += 1;
        return splitmix64(state ^ (counter * 0x2545f4914f6cdd1dull));
    }
    uint32_t next_bounded(uint32_t bound) {
        while (true) {
            uint64_t x = next_u64() >> 32;
            unsigned __int128 m = static_cast<unsigned __int128>(x) * bound;
            uint64_t lo = static_cast<uint64_t>(m & 0xffffffffull);
            if (lo >= bound || lo >= (0x100000000ull % bound)) return static_cast<uint32_t>(m >> 32);
        }
    }
    double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
};

// ---------------------------------------------------------------- sampling
// registration.cpp:21-40
static void sample_quadruple(int source_size, const int32_t* cache, int64_t cache_len, Rng& rng, int src[4],
                             int tgt[4]) {
    if (source_size < 4) fail(OR_TOO_FEW_POINTS, "sample_quadruple: need >= 4 source points");
    if (cache_len != source_size) fail(OR_MISSING_DATA, "sample_quadruple: cache size mismatch");
    for (int k = 0; k < 4; ++k) {
        while (true) {
            int idx = static_cast<int>(rng.next_bounded(static_cast<uint32_t>(source_size)));
            bool dup = false;
            for (int m = 0; m < k; ++m) dup = dup || src[m] == idx;
            if (!dup) {
                src[k] = idx;
                break;
            }
        }
        tgt[k] = cache[src[k]];
    }
}

// registration.cpp:42-51
static bool prerejected(const V3 src[4], const V3 dst[4], double tau) {
    for (int a = 0; a < 4; ++a) {
        int b = (a + 1) & 3;
        double es = norm(sub(src[a], src[b]));
        double ed = norm(sub(dst[a], dst[b]));
        if (es < tau * ed || ed < tau * es) return true;
    }
    return false;
}

// ---------------------------------------------------------------- Jacobi SVD
// Restatement of Eigen 3.4 JacobiSVD<Matrix3d> (ComputeFullU|ComputeFullV) for a
// square real 3x3 matrix: no QR preconditioner, scale by max|a_ij|, two-sided
// Jacobi sweeps (real_2x2_jacobi_svd + JacobiRotation::makeJacobi), sign fix,
// descending sort. Called from kabsch (geometry.cpp:77).
struct Rot {
    double c = 1, s = 0;
};
static inline Rot rot_t(Rot j) { return {j.c, -j.s}; }
static inline Rot rot_mul(Rot a, Rot b) { return {a.c * b.c - a.s * b.s, a.c * b.s + a.s * b.c}; }
// apply_rotation_in_the_plane(x, y, j)
static inline void rot_apply(double& x, double& y, Rot j) {
    double xi = x, yi = y;
    x = j.c * xi + j.s * yi;
    y = -j.s * xi + j.c * yi;
}
static inline void apply_left(double w[3][3], int p, int q, Rot j) {  // rows p,q
    if (j.c == 1.0 && j.s == 0.0) return;
    for (int i = 0; i < 3; ++i) rot_apply(w[p][i], w[q][i], j);
}
static inline void apply_right(double w[3][3], int p, int q, Rot j) {  // cols p,q with j^T
    Rot jt = rot_t(j);
    if (jt.c == 1.0 && jt.s == 0.0) return;
    for (int i = 0; i < 3; ++i) rot_apply(w[i][p], w[i][q], jt);
}
static Rot make_jacobi(double x, double y, double z) {
    Rot r;
    double deno = 2.0 * std::abs(y);
    if (deno < std::numeric_limits<double>::min()) {
        r.c = 1.0;
        r.s = 0.0;
        return r;
    }
    double tau = (x - z) / deno;
    double w = std::sqrt(tau * tau + 1.0);
    double t;
    if (tau > 0.0)
        t = 1.0 / (tau + w);
    else
        t = 1.0 / (tau - w);
    double sign_t = t > 0.0 ? 1.0 : -1.0;
    double n = 1.0 / std::sqrt(t * t + 1.0);
    r.s = -sign_t * (y / std::abs(y)) * std::abs(t) * n;
    r.c = n;
    return r;
}
static void real_2x2_jacobi_svd(double w[3][3], int p, int q, Rot* j_left, Rot* j_right) {
    double m[2][2] = {{w[p][p], w[p][q]}, {w[q][p], w[q][q]}};
    Rot rot1;
    double t = m[0][0] + m[1][1];
    double d = m[1][0] - m[0][1];
    if (std::abs(d) < std::numeric_limits<double>::min()) {
        rot1.s = 0.0;
        rot1.c = 1.0;
    } else {
        double u = t / d;
        double tmp = std::sqrt(1.0 + u * u);
        rot1.s = 1.0 / tmp;
        rot1.c = u / tmp;
    }
    if (!(rot1.c == 1.0 && rot1.s == 0.0)) {
        for (int i = 0; i < 2; ++i) rot_apply(m[0][i], m[1][i], rot1);
    }
    *j_right = make_jacobi(m[0][0], m[0][1], m[1][1]);
    *j_left = rot_mul(rot1, rot_t(*j_right));
}
static void jacobi_svd3(const M3& A, M3& U, double S[3], M3& V) {
    const double consider_as_zero = std::numeric_limits<double>::min();
    const double precision = 2.0 * std::numeric_limits<double>::epsilon();
    double scale = 0.0;
    bool first = true;
    for (int j = 0; j < 3; ++j)
        for (int i = 0; i < 3; ++i) {
            double a = std::abs(A.m[i][j]);
            if (first || a > scale) scale = a;
            first = false;
        }
    if (scale == 0.0) scale = 1.0;
    double w[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) w[i][j] = A.m[i][j] / scale;
    double u[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    double v[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    double max_diag = std::abs(w[0][0]);
    for (int i = 1; i < 3; ++i) max_diag = std::max(max_diag, std::abs(w[i][i]));  // maxCoeff: strict >
    bool finished = false;
    int sweeps = 0;
    while (!finished) {
        finished = true;
        for (int p = 1; p < 3; ++p) {
            for (int q = 0; q < p; ++q) {
                double threshold = std::max(consider_as_zero, precision * max_diag);
                if (std::abs(w[p][q]) > threshold || std::abs(w[q][p]) > threshold) {
                    finished = false;
                    Rot jl, jr;
                    real_2x2_jacobi_svd(w, p, q, &jl, &jr);
                    apply_left(w, p, q, jl);
                    apply_right(u, p, q, rot_t(jl));
                    apply_right(w, p, q, jr);
                    apply_right(v, p, q, jr);
                    max_diag = std::max(max_diag, std::max(std::abs(w[p][p]), std::abs(w[q][q])));
                }
            }
        }
        if (++sweeps > 1000) break;  // unreachable for finite input; guards NaN loops
    }
    for (int i = 0; i < 3; ++i) {
        double a = w[i][i];
        S[i] = std::abs(a);
        if (a < 0.0)
            for (int r = 0; r < 3; ++r) u[r][i] = -u[r][i];
    }
    for (int i = 0; i < 3; ++i) S[i] *= scale;
    for (int i = 0; i < 3; ++i) {
        int pos = i;
        double mx = S[i];
        for (int k = i + 1; k < 3; ++k)
            if (S[k] > mx) {
                mx = S[k];
                pos = k;
            }
        if (mx == 0.0) break;
        if (pos != i) {
            std::swap(S[i], S[pos]);
            for (int r = 0; r < 3; ++r) {
                std::swap(u[r][i], u[r][pos]);
                std::swap(v[r][i], v[r][pos]);
            }
        }
    }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            U.m[i][j] = u[i][j];
            V.m[i][j] = v[i][j];
        }
}

// geometry.cpp:62-91
static Rigid kabsch(const V3* src, const V3* dst, int64_t n) {
    if (n < 3) fail(OR_TOO_FEW_POINTS, "kabsch: need >= 3 point pairs of equal count");
    V3 cs{}, cd{};
    for (int64_t i = 0; i < n; ++i) cs = add(cs, src[i]);
    for (int64_t i = 0; i < n; ++i) cd = add(cd, dst[i]);
    cs = divs(cs, static_cast<double>(n));
    cd = divs(cd, static_cast<double>(n));
    M3 h;
    for (int64_t i = 0; i < n; ++i) {
        V3 a = sub(src[i], cs), b = sub(dst[i], cd);
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) h.m[r][c] = h.m[r][c] + a[r] * b[c];
    }
    M3 U, V;
    double S[3];
    jacobi_svd3(h, U, S, V);
    double scale = std::max(S[0], 1.0);
    if (S[1] <= 1e-12 * scale) fail(OR_DEGENERATE, "kabsch: covariance rank < 2");
    M3 d = ident();
    d.m[2][2] = det(mul(V, transpose(U))) < 0 ? -1.0 : 1.0;
    M3 R = mul(mul(V, d), transpose(U));
    Rigid T;
    T.R = R;
    T.t = sub(cd, mul(R, cs));
    return T;
}

// ---------------------------------------------------------------- SearchGrid
// grid.cpp:15-30 (pack_key, grid_index), :32-66 (build_grid)
struct I3 {
    int x, y, z;
};
static inline uint64_t pack_key(int x, int y, int z) {
    constexpr int64_t off = 1 << 20;
    return (static_cast<uint64_t>(x + off) << 42) | (static_cast<uint64_t>(y + off) << 21) |
           static_cast<uint64_t>(z + off);
}
// static_cast<int>(std::floor(q)); NaN / out-of-range follow x86 cvttsd2si
// (INT_MIN), which is what the reference binary produces for them.
static inline int floor_int(double q) {
    double f = std::floor(q);
    if (!(f >= -2147483648.0 && f < 2147483648.0)) return std::numeric_limits<int>::min();
    return static_cast<int>(f);
}
static inline I3 grid_index(V3 p, V3 center, double cell) {
    V3 q = divs(sub(p, center), cell);
    return {floor_int(q.x), floor_int(q.y), floor_int(q.z)};
}

struct SearchGrid {
    double cell = 1.0;
    V3 center{};
    std::vector<V3> points;
    std::vector<int> cell_points;
    std::unordered_map<uint64_t, std::pair<int, int>> cells;
    I3 cmin{0, 0, 0}, cmax{0, 0, 0};

    const int* cell_span(int x, int y, int z, int& count) const {
        auto it = cells.find(pack_key(x, y, z));
        if (it == cells.end()) {
            count = 0;
            return nullptr;
        }
        count = it->second.second;
        return cell_points.data() + it->second.first;
    }
};

static SearchGrid build_grid(const std::vector<V3>& pts, double cell, V3 center) {
    if (pts.empty()) fail(OR_EMPTY_CLOUD, "build_grid: empty cloud");
    if (!(cell > 0.0)) fail(OR_INVALID_ARGUMENT, "build_grid: cell_length must be positive");
    SearchGrid g;
    g.cell = cell;
    g.center = center;
    g.points = pts;
    const int n = static_cast<int>(pts.size());
    std::vector<uint64_t> keys(n);
    g.cmin = {std::numeric_limits<int>::max(), std::numeric_limits<int>::max(), std::numeric_limits<int>::max()};
    g.cmax = {std::numeric_limits<int>::min(), std::numeric_limits<int>::min(), std::numeric_limits<int>::min()};
    for (int i = 0; i < n; ++i) {
        I3 c = grid_index(pts[i], center, cell);
        g.cmin = {std::min(g.cmin.x, c.x), std::min(g.cmin.y, c.y), std::min(g.cmin.z, c.z)};
        g.cmax = {std::max(g.cmax.x, c.x), std::max(g.cmax.y, c.y), std::max(g.cmax.z, c.z)};
        keys[i] = pack_key(c.x, c.y, c.z);
        auto it = g.cells.try_emplace(keys[i], 0, 0).first;
        it->second.second += 1;
    }
    int start = 0;
    for (auto& kv : g.cells) {
        kv.second.first = start;
        start += kv.second.second;
        kv.second.second = 0;
    }
    g.cell_points.resize(n);
    for (int i = 0; i < n; ++i) {
        auto& r = g.cells[keys[i]];
        g.cell_points[r.first + r.second] = i;
        r.second += 1;
    }
    return g;
}

// grid.cpp:78-97
static void scan_block(const SearchGrid& g, V3 q, int c, double d2_max, double& best_d2, int& best_idx) {
    I3 qc = grid_index(q, g.center, g.cell);
    int lx = std::max(qc.x - c, g.cmin.x), ly = std::max(qc.y - c, g.cmin.y), lz = std::max(qc.z - c, g.cmin.z);
    int hx = std::min(qc.x + c, g.cmax.x), hy = std::min(qc.y + c, g.cmax.y), hz = std::min(qc.z + c, g.cmax.z);
    for (int x = lx; x <= hx; ++x)
        for (int y = ly; y <= hy; ++y)
            for (int z = lz; z <= hz; ++z) {
                int cnt;
                const int* ids = g.cell_span(x, y, z, cnt);
                for (int k = 0; k < cnt; ++k) {
                    int idx = ids[k];
                    double d2 = sqnorm(sub(g.points[idx], q));
                    if (d2 > d2_max) continue;
                    if (d2 < best_d2 || (d2 == best_d2 && idx < best_idx)) {
                        best_d2 = d2;
                        best_idx = idx;
                    }
                }
            }
}

struct Nn {
    int index = -1;
    double distance = 0.0;
};

// grid.cpp:101-109
static bool nn_within(const SearchGrid& g, V3 q, double d_max, Nn* out) {
    if (g.points.empty()) return false;
    int c = static_cast<int>(std::ceil(d_max / g.cell));
    double best_d2 = std::numeric_limits<double>::infinity();
    int best_idx = std::numeric_limits<int>::max();
    scan_block(g, q, c, d_max * d_max, best_d2, best_idx);
    if (best_idx == std::numeric_limits<int>::max()) return false;
    out->index = best_idx;
    out->distance = std::sqrt(best_d2);
    return true;
}

// grid.cpp:111-151
static Nn nn_nearest(const SearchGrid& g, V3 q) {
    if (g.points.empty()) fail(OR_EMPTY_CLOUD, "nn_nearest: empty grid");
    I3 qc = grid_index(q, g.center, g.cell);
    int max_ring = 0;
    int qa[3] = {qc.x, qc.y, qc.z}, mn[3] = {g.cmin.x, g.cmin.y, g.cmin.z}, mx[3] = {g.cmax.x, g.cmax.y, g.cmax.z};
    for (int a = 0; a < 3; ++a) {
        max_ring = std::max(max_ring, qa[a] - mn[a]);
        max_ring = std::max(max_ring, mx[a] - qa[a]);
    }
    double best_d2 = std::numeric_limits<double>::infinity();
    int best_idx = std::numeric_limits<int>::max();
    for (int ring = 0; ring <= max_ring; ++ring) {
        if (best_idx != std::numeric_limits<int>::max() &&
            best_d2 < std::pow(static_cast<double>(ring - 1) * g.cell, 2.0))
            break;
        for (int x = qc.x - ring; x <= qc.x + ring; ++x)
            for (int y = qc.y - ring; y <= qc.y + ring; ++y)
                for (int z = qc.z - ring; z <= qc.z + ring; ++z) {
                    bool on_shell = x == qc.x - ring || x == qc.x + ring || y == qc.y - ring || y == qc.y + ring ||
                                    z == qc.z - ring || z == qc.z + ring;
                    if (!on_shell && ring > 0) continue;
                    int cnt;
                    const int* ids = g.cell_span(x, y, z, cnt);
                    for (int k = 0; k < cnt; ++k) {
                        int idx = ids[k];
                        double d2 = sqnorm(sub(g.points[idx], q));
                        if (d2 < best_d2 || (d2 == best_d2 && idx < best_idx)) {
                            best_d2 = d2;
                            best_idx = idx;
                        }
                    }
                }
    }
    return {best_idx, std::sqrt(best_d2)};
}

// grid.cpp:153-174
static std::vector<int> radius_search(const SearchGrid& g, V3 q, double radius) {
    std::vector<int> out;
    if (g.points.empty()) return out;
    int c = static_cast<int>(std::ceil(radius / g.cell));
    double r2 = radius * radius;
    I3 qc = grid_index(q, g.center, g.cell);
    int lx = std::max(qc.x - c, g.cmin.x), ly = std::max(qc.y - c, g.cmin.y), lz = std::max(qc.z - c, g.cmin.z);
    int hx = std::min(qc.x + c, g.cmax.x), hy = std::min(qc.y + c, g.cmax.y), hz = std::min(qc.z + c, g.cmax.z);
    for (int x = lx; x <= hx; ++x)
        for (int y = ly; y <= hy; ++y)
            for (int z = lz; z <= hz; ++z) {
                int cnt;
                const int* ids = g.cell_span(x, y, z, cnt);
                for (int k = 0; k < cnt; ++k)
                    if (sqnorm(sub(g.points[ids[k]], q)) <= r2) out.push_back(ids[k]);
            }
    std::sort(out.begin(), out.end());
    return out;
}

// ---------------------------------------------------------------- clouds
struct Cloud {
    std::vector<V3> pos;
    std::vector<V3> nrm;  // empty or parallel
    size_t size() const { return pos.size(); }
    bool has_normals() const { return !nrm.empty(); }
};
static Cloud make_cloud(const double* xyz, const double* n3, int64_t n) {
    Cloud c;
    c.pos.resize(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) c.pos[i] = load3(xyz, i);
    if (n3) {
        c.nrm.resize(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) c.nrm[i] = load3(n3, i);
    }
    return c;
}
// geometry.cpp:93-103
static void validate_cloud(const Cloud& c) {
    if (!c.nrm.empty() && c.nrm.size() != c.pos.size())
        fail(OR_MISSING_NORMALS, "normals array must be empty or match positions");
    for (const V3& n : c.nrm) {
        double len = norm(n);
        if (len != 0.0 && std::abs(len - 1.0) > 1e-6)
            fail(OR_MISSING_NORMALS, "normals must be unit length or exactly zero");
    }
}

// ---------------------------------------------------------------- EvalGrid
// registration.hpp:68-79, registration.cpp:80-148
struct EvalGrid {
    V3 origin{};
    double cell = 1.0;
    int nx = 0, ny = 0, nz = 0;
    std::vector<int32_t> start, index;
    std::vector<V3> slot_position, slot_normal;
    std::vector<uint8_t> near_occupied;
};

static EvalGrid build_eval_grid(const Cloud& target, double d_max) {
    if (target.pos.empty()) fail(OR_EMPTY_CLOUD, "build_eval_grid: empty target");
    EvalGrid g;
    g.cell = d_max;
    V3 lo = target.pos[0], hi = target.pos[0];
    for (const V3& p : target.pos) {
        lo = {p.x < lo.x ? p.x : lo.x, p.y < lo.y ? p.y : lo.y, p.z < lo.z ? p.z : lo.z};
        hi = {hi.x < p.x ? p.x : hi.x, hi.y < p.y ? p.y : hi.y, hi.z < p.z ? p.z : hi.z};
    }
    g.origin = sub(lo, v3(g.cell, g.cell, g.cell));
    V3 extent = add(sub(hi, g.origin), v3(g.cell, g.cell, g.cell));
    g.nx = static_cast<int>(std::floor(extent.x / g.cell)) + 2;
    g.ny = static_cast<int>(std::floor(extent.y / g.cell)) + 2;
    g.nz = static_cast<int>(std::floor(extent.z / g.cell)) + 2;
    const size_t ncells = static_cast<size_t>(g.nx) * g.ny * g.nz;
    auto cell_of = [&](V3 p, int& ix, int& iy, int& iz) {
        ix = static_cast<int>(std::floor((p.x - g.origin.x) / g.cell));
        iy = static_cast<int>(std::floor((p.y - g.origin.y) / g.cell));
        iz = static_cast<int>(std::floor((p.z - g.origin.z) / g.cell));
    };
    auto flat = [&](int ix, int iy, int iz) {
        return (static_cast<size_t>(ix) * g.ny + static_cast<size_t>(iy)) * g.nz + static_cast<size_t>(iz);
    };
    const int n = static_cast<int>(target.size());
    std::vector<int32_t> counts(ncells + 1, 0);
    std::vector<size_t> cidx(n);
    for (int i = 0; i < n; ++i) {
        int ix, iy, iz;
        cell_of(target.pos[i], ix, iy, iz);
        cidx[i] = flat(ix, iy, iz);
        counts[cidx[i] + 1] += 1;
    }
    g.start.resize(ncells + 1);
    g.start[0] = 0;
    for (size_t c = 0; c < ncells; ++c) g.start[c + 1] = g.start[c] + counts[c + 1];
    g.index.resize(n);
    g.slot_position.resize(n);
    g.slot_normal.assign(n, V3{});
    std::vector<int32_t> cursor(g.start.begin(), g.start.end() - 1);
    for (int i = 0; i < n; ++i) {
        int32_t slot = cursor[cidx[i]]++;
        g.index[slot] = i;
        g.slot_position[slot] = target.pos[i];
        if (target.has_normals()) g.slot_normal[slot] = target.nrm[i];
    }
    g.near_occupied.assign(ncells, 0);
    for (int i = 0; i < n; ++i) {
        int ix, iy, iz;
        cell_of(target.pos[i], ix, iy, iz);
        for (int dx = -1; dx <= 1; ++dx)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dz = -1; dz <= 1; ++dz) {
                    int x = ix + dx, y = iy + dy, z = iz + dz;
                    if (x < 0 || y < 0 || z < 0 || x >= g.nx || y >= g.ny || z >= g.nz) continue;
                    g.near_occupied[flat(x, y, z)] = 1;
                }
    }
    return g;
}

struct WorkCounters {
    int64_t visited = 0, near = 0, slots = 0, hits = 0;
};

// registration.cpp:155-219. Returns true if fully scored.
static bool evaluate_against_grid(const EvalGrid& g, const Cloud& source, const Rigid& t, double d_max,
                                  double cos_max, int64_t miss_budget, double& ratio, double& fitness,
                                  int64_t& inliers_out, WorkCounters* wc) {
    const double d2_max = d_max * d_max;
    const int64_t n = static_cast<int64_t>(source.size());
    int64_t inliers = 0, misses = 0;
    double sq_sum = 0.0;
    const size_t plane = static_cast<size_t>(g.ny) * g.nz;
    for (int64_t i = 0; i < n; ++i) {
        if (wc) wc->visited += 1;
        V3 y = apply(t, source.pos[i]);
        int ix = floor_int((y.x - g.origin.x) / g.cell);
        int iy = floor_int((y.y - g.origin.y) / g.cell);
        int iz = floor_int((y.z - g.origin.z) / g.cell);
        bool miss = true;
        if (ix >= 0 && iy >= 0 && iz >= 0 && ix < g.nx && iy < g.ny && iz < g.nz) {
            size_t c = static_cast<size_t>(ix) * plane + static_cast<size_t>(iy) * g.nz + static_cast<size_t>(iz);
            if (g.near_occupied[c]) {
                if (wc) wc->near += 1;
                double best_d2 = std::numeric_limits<double>::infinity();
                int32_t best_slot = -1;
                int best_index = std::numeric_limits<int>::max();
                int x0 = std::max(ix - 1, 0), x1 = std::min(ix + 1, g.nx - 1);
                int y0 = std::max(iy - 1, 0), y1 = std::min(iy + 1, g.ny - 1);
                int z0 = std::max(iz - 1, 0), z1 = std::min(iz + 1, g.nz - 1);
                for (int x = x0; x <= x1; ++x) {
                    for (int yy = y0; yy <= y1; ++yy) {
                        size_t row = static_cast<size_t>(x) * plane + static_cast<size_t>(yy) * g.nz;
                        int32_t s0 = g.start[row + z0];
                        int32_t s1 = g.start[row + z1 + 1];
                        if (wc) wc->slots += s1 - s0;
                        for (int32_t s = s0; s < s1; ++s) {
                            double d2 = sqnorm(sub(g.slot_position[s], y));
                            if (d2 > d2_max) continue;
                            int orig = g.index[s];
                            if (d2 < best_d2 || (d2 == best_d2 && orig < best_index)) {
                                best_d2 = d2;
                                best_slot = s;
                                best_index = orig;
                            }
                        }
                    }
                }
                if (best_slot >= 0) {
                    if (wc) wc->hits += 1;
                    const V3& ns = source.nrm[i];
                    const V3& nt = g.slot_normal[best_slot];
                    if (!is_zero(ns) && !is_zero(nt) && dot(mul(t.R, ns), nt) >= cos_max) {
                        miss = false;
                        inliers += 1;
                        sq_sum += best_d2;
                    }
                }
            }
        }
        if (miss) {
            misses += 1;
            if (misses > miss_budget) return false;
        }
    }
    ratio = static_cast<double>(inliers) / static_cast<double>(n);
    fitness = inliers > 0 ? sq_sum / static_cast<double>(inliers) : 0.0;
    inliers_out = inliers;
    return true;
}

// registration.cpp:53-78
static void evaluate_hypothesis(const Rigid& t, const Cloud& source, const Cloud& target, const SearchGrid& grid,
                                double d_max, double normal_angle_max, double& ratio, double& fitness,
                                int64_t& inliers_out) {
    if (source.pos.empty() || target.pos.empty()) fail(OR_EMPTY_CLOUD, "evaluate_hypothesis: empty cloud");
    if (!source.has_normals() || !target.has_normals())
        fail(OR_MISSING_NORMALS, "evaluate_hypothesis: both clouds need normals");
    const double cos_max = std::cos(normal_angle_max);
    int64_t inliers = 0;
    double sq_sum = 0.0;
    for (size_t i = 0; i < source.size(); ++i) {
        V3 y = apply(t, source.pos[i]);
        Nn nn;
        if (!nn_within(grid, y, d_max, &nn)) continue;
        V3 ns = source.nrm[i];
        const V3& nt = target.nrm[nn.index];
        if (is_zero(ns) || is_zero(nt)) continue;
        if (dot(mul(t.R, ns), nt) < cos_max) continue;
        inliers += 1;
        sq_sum += nn.distance * nn.distance;
    }
    ratio = static_cast<double>(inliers) / static_cast<double>(source.size());
    fitness = inliers > 0 ? sq_sum / static_cast<double>(inliers) : 0.0;
    inliers_out = inliers;
}

// ---------------------------------------------------------------- preprocessing
// preprocess.cpp:14-59
static Cloud voxel_downsample(const Cloud& cloud, double leaf) {
    if (cloud.pos.empty()) fail(OR_EMPTY_CLOUD, "voxel_downsample: empty cloud");
    if (!(leaf > 0.0)) fail(OR_INVALID_ARGUMENT, "voxel_downsample: leaf must be positive");
    validate_cloud(cloud);
    struct Accum {
        V3 pos_sum{}, normal_sum{};
        int count = 0;
        int min_index = 0;
    };
    std::unordered_map<uint64_t, Accum> voxels;
    voxels.reserve(cloud.size());
    for (size_t i = 0; i < cloud.size(); ++i) {
        I3 c = grid_index(cloud.pos[i], V3{}, leaf);
        uint64_t key = pack_key(c.x, c.y, c.z);
        auto ins = voxels.try_emplace(key);
        Accum& a = ins.first->second;
        if (ins.second) a.min_index = static_cast<int>(i);
        a.pos_sum = add(a.pos_sum, cloud.pos[i]);
        if (cloud.has_normals() && !is_zero(cloud.nrm[i])) a.normal_sum = add(a.normal_sum, cloud.nrm[i]);
        a.count += 1;
    }
    std::vector<const Accum*> order;
    order.reserve(voxels.size());
    for (const auto& kv : voxels) order.push_back(&kv.second);
    std::sort(order.begin(), order.end(), [](const Accum* a, const Accum* b) { return a->min_index < b->min_index; });
    Cloud out;
    out.pos.reserve(order.size());
    for (const Accum* a : order) {
        out.pos.push_back(divs(a->pos_sum, static_cast<double>(a->count)));
        if (cloud.has_normals()) {
            double len = norm(a->normal_sum);
            out.nrm.push_back(len > 1e-12 ? divs(a->normal_sum, len) : V3{});
        }
    }
    return out;
}

// fpfh.cpp:17-48
static bool pair_angles(V3 p1, V3 n1, V3 p2, V3 n2, double& alpha, double& phi, double& theta) {
    V3 d = sub(p2, p1);
    double dist = norm(d);
    if (dist <= 0.0) return false;
    double angle1 = dot(n1, d) / dist;
    double angle2 = dot(n2, d) / dist;
    V3 ns = n1, nt = n2, line = d;
    double cos_line = angle1;
    if (std::acos(std::abs(angle1)) > std::acos(std::abs(angle2))) {
        ns = n2;
        nt = n1;
        line = neg(d);
        cos_line = -angle2;
    }
    V3 u = ns;
    V3 v = cross(line, u);
    double v_len = norm(v);
    if (v_len <= 1e-12 * dist) return false;
    v = divs(v, v_len);
    V3 w = cross(u, v);
    alpha = dot(v, nt);
    phi = cos_line;
    theta = std::atan2(dot(w, nt), dot(u, nt));
    return true;
}
// fpfh.cpp:50-53
static int bin_index(double value, double lo, double hi) {
    int b = floor_int(11 * (value - lo) / (hi - lo));
    return std::clamp(b, 0, 10);
}
// fpfh.cpp:57-141
// ---- estimate_normals (proj/src/preprocess.cpp:61-96) ----------------------
// Eigen::SelfAdjointEigenSolver<Matrix3d> restated (Eigen 3.4 source order;
// Eigen is absent here, so this is the builder's statement of it -- the
// normals' parity with the reference binary is unpinned):
// SelfAdjointEigenSolver::compute, tridiagonalization_inplace_selector<3>,
// computeFromTridiagonal_impl, tridiagonal_qr_step, JacobiRotation::makeGivens,
// applyOnTheRight (rotation transposed), numext::hypot.
namespace eig3 {
static double eabs(double x) { return std::fabs(x); }
static double ehypot(double x, double y) {
    x = eabs(x);
    y = eabs(y);
    if (std::isinf(x) || std::isinf(y)) return HUGE_VAL;
    if (std::isnan(x) || std::isnan(y)) return x + y;
    const double p = std::max(x, y);
    if (p == 0.0) return 0.0;
    const double qp = std::min(y, x) / p;
    return p * std::sqrt(1.0 + qp * qp);
}
static void givens(double p, double q, double& c, double& s) {
    if (q == 0.0) {
        c = p < 0.0 ? -1.0 : 1.0;
        s = 0.0;
    } else if (p == 0.0) {
        c = 0.0;
        s = q < 0.0 ? 1.0 : -1.0;
    } else if (eabs(p) > eabs(q)) {
        const double t = q / p;
        double u = std::sqrt(1.0 + t * t);
        if (p < 0.0) u = -u;
        c = 1.0 / u;
        s = -t * c;
    } else {
        const double t = p / q;
        double u = std::sqrt(1.0 + t * t);
        if (q < 0.0) u = -u;
        s = -1.0 / u;
        c = -t * s;
    }
}
// eivec: column-major, e[col][row]
static void qr_step(double* d, double* e, int start, int end, double ev[3][3]) {
    const double td = (d[end - 1] - d[end]) * 0.5;
    const double ee = e[end - 1];
    double mu = d[end];
    if (td == 0.0) {
        mu -= eabs(ee);
    } else if (ee != 0.0) {
        const double e2 = ee * ee;
        const double h = ehypot(td, ee);
        if (e2 == 0.0) mu -= ee / ((td + (td > 0.0 ? h : -h)) / ee);
        else mu -= e2 / (td + (td > 0.0 ? h : -h));
    }
    double x = d[start] - mu, z = e[start];
    for (int k = start; k < end && z != 0.0; ++k) {
        double c, s;
        givens(x, z, c, s);
        const double sdk = s * d[k] + c * e[k];
        const double dkp1 = s * e[k] + c * d[k + 1];
        d[k] = c * (c * d[k] - s * e[k]) - s * (c * e[k] - s * d[k + 1]);
        d[k + 1] = s * sdk + c * dkp1;
        e[k] = c * sdk - s * dkp1;
        if (k > start) e[k - 1] = c * e[k - 1] - s * z;
        x = e[k];
        if (k < end - 1) {
            z = -s * e[k + 1];
            e[k + 1] = c * e[k + 1];
        }
        // Q = Q * G: applyOnTheRight(k, k+1, rot) = rotation in the plane with (c, -s)
        for (int r = 0; r < 3; ++r) {
            const double xi = ev[k][r], yi = ev[k + 1][r];
            ev[k][r] = c * xi + -s * yi;
            ev[k + 1][r] = -(-s) * xi + c * yi;
        }
    }
}
// column 0 of the eigenvector matrix of the symmetric A (lower triangle used)
static V3 smallest_eigenvector(const double A[3][3]) {
    double m[3][3];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) m[r][c] = c <= r ? A[r][c] : 0.0;  // triangularView<Lower>
    double scale = 0.0;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c <= r; ++c) scale = std::max(scale, eabs(m[r][c]));
    if (scale == 0.0) scale = 1.0;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c <= r; ++c) m[r][c] /= scale;
    double d[3], e[2], ev[3][3];
    d[0] = m[0][0];
    const double v1norm2 = m[2][0] * m[2][0];
    if (v1norm2 <= std::numeric_limits<double>::min()) {
        d[1] = m[1][1];
        d[2] = m[2][2];
        e[0] = m[1][0];
        e[1] = m[2][1];
        for (int c = 0; c < 3; ++c)
            for (int r = 0; r < 3; ++r) ev[c][r] = r == c ? 1.0 : 0.0;
    } else {
        const double beta = std::sqrt(m[1][0] * m[1][0] + v1norm2);
        const double inv = 1.0 / beta;
        const double m01 = m[1][0] * inv, m02 = m[2][0] * inv;
        const double q = 2.0 * m01 * m[2][1] + m02 * (m[2][2] - m[1][1]);
        d[1] = m[1][1] + m02 * q;
        d[2] = m[2][2] - m02 * q;
        e[0] = beta;
        e[1] = m[2][1] - m01 * q;
        const double Q[3][3] = {{1, 0, 0}, {0, m01, m02}, {0, m02, -m01}};  // rows; symmetric
        for (int c = 0; c < 3; ++c)
            for (int r = 0; r < 3; ++r) ev[c][r] = Q[r][c];
    }
    const int n = 3;
    int end = n - 1, start = 0, iter = 0;
    const double considerAsZero = std::numeric_limits<double>::min();
    const double precision_inv = 1.0 / std::numeric_limits<double>::epsilon();
    while (end > 0) {
        for (int i = start; i < end; ++i) {
            if (eabs(e[i]) < considerAsZero) {
                e[i] = 0.0;
            } else {
                const double sc = precision_inv * e[i];
                if (sc * sc <= (eabs(d[i]) + eabs(d[i + 1]))) e[i] = 0.0;
            }
        }
        while (end > 0 && e[end - 1] == 0.0) end--;
        if (end <= 0) break;
        iter++;
        if (iter > 30 * n) break;
        start = end - 1;
        while (start > 0 && e[start - 1] != 0.0) start--;
        qr_step(d, e, start, end, ev);
    }
    if (iter <= 30 * n) {
        for (int i = 0; i < n - 1; ++i) {
            int k = 0;
            for (int j = 1; j < n - i; ++j)
                if (d[i + j] < d[i + k]) k = j;
            if (k > 0) {
                std::swap(d[i], d[k + i]);
                for (int r = 0; r < 3; ++r) std::swap(ev[i][r], ev[k + i][r]);
            }
        }
    }
    return V3{ev[0][0], ev[0][1], ev[0][2]};
}
}  // namespace eig3

static Cloud estimate_normals(const Cloud& cloud, double radius, V3 viewpoint, int threads) {
    if (cloud.pos.empty()) fail(OR_EMPTY_CLOUD, "estimate_normals: empty cloud");
    if (!(radius > 0.0)) fail(OR_INVALID_ARGUMENT, "build_grid: cell_length must be positive");
    SearchGrid grid = build_grid(cloud.pos, radius, V3{});
    Cloud out;
    out.pos = cloud.pos;
    out.nrm.assign(cloud.size(), V3{});
    const int n = static_cast<int>(cloud.size());
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int i = 0; i < n; ++i) {
        const V3 p = cloud.pos[static_cast<size_t>(i)];
        std::vector<int> nbrs = radius_search(grid, p, radius);
        if (nbrs.size() < 3) continue;
        V3 mean{};
        for (int j : nbrs) mean = add(mean, cloud.pos[static_cast<size_t>(j)]);
        mean = divs(mean, static_cast<double>(nbrs.size()));
        double cov[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        for (int j : nbrs) {
            const V3 dd = sub(cloud.pos[static_cast<size_t>(j)], mean);
            const double dv[3] = {dd.x, dd.y, dd.z};
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) cov[r][c] = cov[r][c] + dv[r] * dv[c];
        }
        V3 normal = eig3::smallest_eigenvector(cov);
        const double len = norm(normal);
        if (!(len > 0.0) || !std::isfinite(len)) continue;
        normal = divs(normal, len);
        if (dot(normal, sub(viewpoint, p)) < 0.0) normal = neg(normal);
        out.nrm[static_cast<size_t>(i)] = normal;
    }
    return out;
}

static std::vector<std::array<float, 33>> compute_fpfh(const Cloud& cloud, double radius, int threads) {
    if (cloud.pos.empty()) fail(OR_EMPTY_CLOUD, "compute_fpfh: empty cloud");
    if (!cloud.has_normals()) fail(OR_MISSING_NORMALS, "compute_fpfh: cloud has no normals");
    validate_cloud(cloud);
    const int n = static_cast<int>(cloud.size());
    SearchGrid grid = build_grid(cloud.pos, radius, V3{});
    if (threads <= 0) threads = omp_get_max_threads();
    std::vector<std::vector<int>> nbr(n);
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int i = 0; i < n; ++i) {
        std::vector<int> v = radius_search(grid, cloud.pos[i], radius);
        v.erase(std::remove(v.begin(), v.end(), i), v.end());
        nbr[i] = std::move(v);
    }
    std::vector<std::array<double, 33>> spfh(n);
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int i = 0; i < n; ++i) {
        auto& h = spfh[i];
        h.fill(0.0);
        V3 p = cloud.pos[i], np = cloud.nrm[i];
        if (is_zero(np)) continue;
        int votes = 0;
        for (int j : nbr[i]) {
            V3 nq = cloud.nrm[j];
            if (is_zero(nq)) continue;
            double alpha, phi, theta;
            if (!pair_angles(p, np, cloud.pos[j], nq, alpha, phi, theta)) continue;
            h[bin_index(alpha, -1.0, 1.0)] += 1.0;
            h[11 + bin_index(phi, -1.0, 1.0)] += 1.0;
            h[22 + bin_index(theta, -M_PI, M_PI)] += 1.0;
            votes += 1;
        }
        if (votes > 0)
            for (double& v : h) v *= 100.0 / static_cast<double>(votes);
    }
    std::vector<std::array<float, 33>> out(n);
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int i = 0; i < n; ++i) {
        out[i].fill(0.0f);
        V3 p = cloud.pos[i];
        if (is_zero(cloud.nrm[i])) continue;
        std::array<double, 33> acc{};
        int k_count = 0;
        for (int j : nbr[i]) {
            if (is_zero(cloud.nrm[j])) continue;
            double w = norm(sub(cloud.pos[j], p));
            if (w <= 0.0) continue;
            const auto& hj = spfh[j];
            for (int b = 0; b < 33; ++b) acc[b] += hj[b] / w;
            k_count += 1;
        }
        const auto& hi = spfh[i];
        for (int b = 0; b < 33; ++b) {
            double blended = hi[b];
            if (k_count > 0) blended += acc[b] / static_cast<double>(k_count);
            out[i][b] = static_cast<float>(blended);
        }
    }
    return out;
}

// Feature pre-match: the reference binary's float matcher (grid.cpp:176-213),
// score_j = |q_j|^2 - 2 (Q^T f)_j in FP32, argmin with strict < over ascending j
// (ties -> lowest j). The reference's own test pins it only against the FP64
// exhaustive matcher on random features (test_grid.cpp:113-125); on FPFH
// near-ties the two differ (56 of 5,309 sources on B1), and the drop-in must
// match the binary, so this restates Eigen 3.4's float evaluation order
// (SSE2, no FMA; the same rules as oracle/ref_shim/Eigen/Dense, against which
// tests/test_ref_parity.py checks it bit for bit):
//   |q|^2: colwise().squaredNorm() -- redux over 33 floats: two 4-lane packet
//     accumulators r0 (packets 0,2,4,6) and r1 (packets 1,3,5,7), r0 + r1,
//     predux (l0 + l2) + (l1 + l3), then + q32^2;
//   Q^T f: row-major GEMV -- 4 lane accumulators over the 8 whole packets in
//     order (0 + a b, then + a b), predux, then + a32 b32; times alpha = 2
//     (exact).
static inline float eigen_qnorm33(const float* q) {
    float r0[4], r1[4];
    for (int l = 0; l < 4; ++l) {
        r0[l] = q[l] * q[l];
        r1[l] = q[4 + l] * q[4 + l];
    }
    for (int idx = 8; idx < 32; idx += 8)
        for (int l = 0; l < 4; ++l) {
            r0[l] = r0[l] + q[idx + l] * q[idx + l];
            r1[l] = r1[l] + q[idx + 4 + l] * q[idx + 4 + l];
        }
    for (int l = 0; l < 4; ++l) r0[l] = r0[l] + r1[l];
    float res = (r0[0] + r0[2]) + (r0[1] + r0[3]);
    return res + q[32] * q[32];
}
static inline float eigen_dot33(const float* a, const float* b) {
    float c[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    for (int k = 0; k < 32; k += 4)
        for (int l = 0; l < 4; ++l) c[l] = a[k + l] * b[k + l] + c[l];
    float cc = (c[0] + c[2]) + (c[1] + c[3]);
    cc += a[32] * b[32];
    return 0.0f + 2.0f * cc;
}
static std::vector<int32_t> feature_nn_cache(const float* sf, int64_t ns, const float* tf, int64_t nt, int threads) {
    if (ns <= 0 || nt <= 0) fail(OR_MISSING_DATA, "feature_nn_cache: empty feature set");
    std::vector<float> q2(static_cast<size_t>(nt));
    for (int64_t j = 0; j < nt; ++j) q2[static_cast<size_t>(j)] = eigen_qnorm33(tf + 33 * j);
    std::vector<int32_t> cache(ns, -1);
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int64_t i = 0; i < ns; ++i) {
        const float* f = sf + 33 * i;
        int best = 0;
        float best_s = q2[0] - eigen_dot33(tf, f);
        for (int64_t j = 1; j < nt; ++j) {
            float s = q2[static_cast<size_t>(j)] - eigen_dot33(tf + 33 * j, f);
            if (s < best_s) {
                best_s = s;
                best = static_cast<int>(j);
            }
        }
        cache[i] = best;
    }
    return cache;
}

// ---------------------------------------------------------------- context + run
struct Context {
    Cloud source, target;
    std::vector<std::array<float, 33>> sfeat, tfeat;
    std::vector<int32_t> cache;
    EvalGrid eval;
};

static double now_seconds() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// registration.cpp:223-251
static Context* prepare(const Cloud& src_in, const Cloud& tgt_in, const or_params& p) {
    auto ctx = std::make_unique<Context>();
    ctx->source = voxel_downsample(src_in, p.leaf);
    ctx->target = voxel_downsample(tgt_in, p.leaf);
    if (ctx->source.size() < 4 || ctx->target.size() < 4)
        fail(OR_TOO_FEW_POINTS, "register_global: fewer than 4 points after downsampling");
    if (!ctx->source.has_normals()) ctx->source = estimate_normals(ctx->source, p.normal_radius, V3{}, p.threads);
    if (!ctx->target.has_normals()) ctx->target = estimate_normals(ctx->target, p.normal_radius, V3{}, p.threads);
    auto usable = [](const Cloud& c) {
        size_t k = 0;
        for (const V3& nn : c.nrm) k += is_zero(nn) ? 0u : 1u;
        return k;
    };
    if (usable(ctx->source) < 4 || usable(ctx->target) < 4)
        fail(OR_MISSING_DATA, "register_global: fewer than 4 points with usable normals");
    ctx->sfeat = compute_fpfh(ctx->source, p.feature_radius, p.threads);
    ctx->tfeat = compute_fpfh(ctx->target, p.feature_radius, p.threads);
    ctx->cache = feature_nn_cache(ctx->sfeat.data()->data(), static_cast<int64_t>(ctx->sfeat.size()),
                                  ctx->tfeat.data()->data(), static_cast<int64_t>(ctx->tfeat.size()), p.threads);
    ctx->eval = build_eval_grid(ctx->target, p.d_max);
    return ctx.release();
}

static double resolved_max_fitness(const or_params& p) {
    return p.max_fitness < 0 ? p.d_max * p.d_max / 2.0 : p.max_fitness;
}

struct Best {
    double ratio = -1.0;
    double fitness = std::numeric_limits<double>::infinity();
    int64_t index = std::numeric_limits<int64_t>::max();
    int64_t inliers = 0;
    Rigid transform;
    bool valid = false;
};
// registration.cpp:272-276
static bool better(const Best& a, const Best& b) {
    if (a.ratio != b.ratio) return a.ratio > b.ratio;
    if (a.fitness != b.fitness) return a.fitness < b.fitness;
    return a.index < b.index;
}

// registration.cpp:253-332, over hypothesis indices [begin, end)
static void run_hypotheses(const Context& ctx, const or_params& p, int64_t begin, int64_t end, or_result* res,
                           or_stats* st) {
    const int n_src = static_cast<int>(ctx.source.size());
    const double cos_max = std::cos(p.normal_angle_max);
    const double max_fitness = resolved_max_fitness(p);
    const int64_t miss_budget = static_cast<int64_t>(ctx.source.size()) -
                                static_cast<int64_t>(std::ceil(p.min_inlier_ratio * static_cast<double>(ctx.source.size())));
    if (n_src < 4) fail(OR_TOO_FEW_POINTS, "sample_quadruple: need >= 4 source points");
    if (static_cast<int64_t>(ctx.cache.size()) != n_src) fail(OR_MISSING_DATA, "sample_quadruple: cache size mismatch");
    Best global;
    int64_t prerej = 0, degen = 0, evald = 0, qual = 0, w_ref = 0, near = 0, slots = 0, hits = 0;
    int threads = p.threads > 0 ? p.threads : omp_get_max_threads();
    double t0 = now_seconds();
#pragma omp parallel num_threads(threads) reduction(+ : prerej, degen, evald, qual, w_ref, near, slots, hits)
    {
        Best local;
        WorkCounters wc;
#pragma omp for schedule(dynamic, 256)
        for (int64_t i = begin; i < end; ++i) {
            Rng rng(p.seed, static_cast<uint64_t>(i));
            int s_idx[4], t_idx[4];
            sample_quadruple(n_src, ctx.cache.data(), static_cast<int64_t>(ctx.cache.size()), rng, s_idx, t_idx);
            V3 src[4], dst[4];
            for (int k = 0; k < 4; ++k) {
                src[k] = ctx.source.pos[s_idx[k]];
                dst[k] = ctx.target.pos[t_idx[k]];
            }
            if (prerejected(src, dst, p.similarity_tau)) {
                prerej += 1;
                continue;
            }
            Rigid t;
            try {
                t = kabsch(src, dst, 4);
            } catch (const Error& e) {
                if (e.code != OR_DEGENERATE) throw;
                degen += 1;
                continue;
            }
            evald += 1;
            double ratio = 0, fitness = 0;
            int64_t inl = 0;
            bool scored = evaluate_against_grid(ctx.eval, ctx.source, t, p.d_max, cos_max, miss_budget, ratio,
                                                fitness, inl, &wc);
            if (!scored) continue;
            if (ratio < p.min_inlier_ratio || fitness > max_fitness) continue;
            qual += 1;
            Best cand;
            cand.ratio = ratio;
            cand.fitness = fitness;
            cand.index = i;
            cand.inliers = inl;
            cand.transform = t;
            cand.valid = true;
            if (!local.valid || better(cand, local)) local = cand;
        }
        w_ref += wc.visited;
        near += wc.near;
        slots += wc.slots;
        hits += wc.hits;
#pragma omp critical(or_reg_best)
        {
            if (local.valid && (!global.valid || better(local, global))) global = local;
        }
    }
    double t1 = now_seconds();
    if (st) {
        st->sampled = end - begin;
        st->prerejected = prerej;
        st->degenerate = degen;
        st->evaluated = evald;
        st->qualified = qual;
        st->w_ref = w_ref;
        st->near_occupied = near;
        st->slots_scanned = slots;
        st->nn_hits = hits;
        st->hypothesis_seconds = t1 - t0;
    }
    std::memset(res, 0, sizeof(*res));
    res->hypothesis_index = -1;
    if (global.valid) {
        store_m(res->R, global.transform.R);
        res->t[0] = global.transform.t.x;
        res->t[1] = global.transform.t.y;
        res->t[2] = global.transform.t.z;
        res->inlier_ratio = global.ratio;
        res->fitness = global.fitness;
        res->inliers = global.inliers;
        res->hypothesis_index = global.index;
        res->found = 1;
    }
}

// line_process.cpp:11-33
static void edge_info(const Cloud& ci, const Cloud& cj, const Rigid& ti, const Rigid& tj, double eps, double info[36],
                      int64_t& pair_count) {
    if (ci.pos.empty() || cj.pos.empty()) fail(OR_EMPTY_CLOUD, "edge_info: empty cloud");
    std::vector<V3> posed;
    posed.reserve(cj.size());
    for (const V3& q : cj.pos) posed.push_back(apply(tj, q));
    SearchGrid grid = build_grid(posed, eps, V3{});
    double L[6][6] = {};
    pair_count = 0;
    for (const V3& p : ci.pos) {
        Nn nn;
        if (!nn_within(grid, apply(ti, p), eps, &nn)) continue;
        // a = -skew(p); skew(v) = [0 -z y; z 0 -x; -y x 0]
        double a[3][3] = {{-0.0, p.z, -p.y}, {-p.z, -0.0, p.x}, {p.y, -p.x, -0.0}};
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                double ata = (a[0][r] * a[0][c] + a[1][r] * a[1][c]) + a[2][r] * a[2][c];
                L[r][c] += ata;            // TL += a^T a
                L[r][3 + c] += a[c][r];    // TR += a^T
                L[3 + r][c] += a[r][c];    // BL += a
                L[3 + r][3 + c] += r == c ? 1.0 : 0.0;  // BR += I
            }
        pair_count += 1;
    }
    if (pair_count == 0) fail(OR_NO_CORRESPONDENCES, "edge_info: no points within epsilon");
    for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c) info[6 * r + c] = L[r][c];
}

}  // namespace orc

// ================================================================ C ABI
using namespace orc;


// ---- ICP point-to-plane (north-star item 4; config D) ----------------------
// The reference has no ICP (SPEC.md:332 lists it as a non-goal), so this is
// the builder's own specification, frozen here and in DESIGN.md "ICP", and
// the device implementation (lk_icp.cu) must equal it bit for bit:
//  * correspondences: the EvalGrid of the target at cell = max_dist and the
//    exact NN of evaluate_against_grid (registration.cpp:165-199: +-1 cell
//    window, d2 <= max_dist^2, min (d2, original index)); a zero target
//    normal drops the pair;
//  * per pair (y = T p, q, n): r = (y - q) . n, J = (y x n, n) -- the
//    G_p = [-[p]x | I] convention of line_process.cpp:23-28 applied to the
//    plane normal -- contributing H_uv = J_u J_v (u <= v, row-major), g_u =
//    J_u r, e = r r;
//  * a fixed reduction tree over the point order: 32-point butterflies (xor
//    16, 8, 4, 2, 1), 8 of them summed in order per 256-point chunk, chunk
//    values in 32-chunk butterflies, those summed in order from 0.0;
//  * H delta = -g by LDL^T without pivoting; the update is the Cayley map
//    R_d = I + s (K + K^2), K = [delta_w / 2]x, s = 2 / (1 + |delta_w / 2|^2)
//    (a rotation; rational, so host and device agree bitwise), then
//    T <- (R_d R, R_d t + delta_v) in Eigen's Matrix3d product order;
//  * stop after the update when |delta|^2 < eps^2, or when fewer than 6
//    correspondences / a non-positive pivot leave the system singular.
static bool eval_grid_nn(const EvalGrid& g, V3 y, double d2_max, int32_t& slot_out, double& d2_out) {
    int ix = floor_int((y.x - g.origin.x) / g.cell);
    int iy = floor_int((y.y - g.origin.y) / g.cell);
    int iz = floor_int((y.z - g.origin.z) / g.cell);
    if (ix < 0 || iy < 0 || iz < 0 || ix >= g.nx || iy >= g.ny || iz >= g.nz) return false;
    const size_t plane = static_cast<size_t>(g.ny) * g.nz;
    size_t c = static_cast<size_t>(ix) * plane + static_cast<size_t>(iy) * g.nz + static_cast<size_t>(iz);
    if (!g.near_occupied[c]) return false;
    double best_d2 = std::numeric_limits<double>::infinity();
    int32_t best_slot = -1;
    int best_index = std::numeric_limits<int>::max();
    int x0 = std::max(ix - 1, 0), x1 = std::min(ix + 1, g.nx - 1);
    int y0 = std::max(iy - 1, 0), y1 = std::min(iy + 1, g.ny - 1);
    int z0 = std::max(iz - 1, 0), z1 = std::min(iz + 1, g.nz - 1);
    for (int x = x0; x <= x1; ++x)
        for (int yy = y0; yy <= y1; ++yy) {
            size_t row = static_cast<size_t>(x) * plane + static_cast<size_t>(yy) * g.nz;
            for (int32_t s = g.start[row + z0]; s < g.start[row + z1 + 1]; ++s) {
                double d2 = sqnorm(sub(g.slot_position[s], y));
                if (d2 > d2_max) continue;
                int orig = g.index[s];
                if (d2 < best_d2 || (d2 == best_d2 && orig < best_index)) {
                    best_d2 = d2;
                    best_slot = s;
                    best_index = orig;
                }
            }
        }
    slot_out = best_slot;
    d2_out = best_d2;
    return best_slot >= 0;
}

static constexpr int kIcpVals = 28;  // 21 H (upper, row-major) + 6 g + e

// LDL^T solve of H x = -g (6x6, no pivoting); false on a non-positive pivot.
// Shared verbatim (operation for operation) by lk_icp.cu's device solve.
static bool icp_solve(const double* h21, const double* g6, double* x6) {
    double H[6][6];
    int k = 0;
    for (int u = 0; u < 6; ++u)
        for (int w = u; w < 6; ++w) {
            H[u][w] = h21[k];
            H[w][u] = h21[k];
            ++k;
        }
    double L[6][6] = {}, D[6];
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

// Cayley update of T by the twist x6 = (w, v).
static Rigid icp_update(const Rigid& T, const double* x6) {
    const double wx = x6[0] * 0.5, wy = x6[1] * 0.5, wz = x6[2] * 0.5;
    const double s = 2.0 / (1.0 + ((wx * wx + wy * wy) + wz * wz));
    M3 K;
    K.m[0][0] = 0.0; K.m[0][1] = -wz; K.m[0][2] = wy;
    K.m[1][0] = wz; K.m[1][1] = 0.0; K.m[1][2] = -wx;
    K.m[2][0] = -wy; K.m[2][1] = wx; K.m[2][2] = 0.0;
    M3 K2 = mul(K, K);
    M3 Rd;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) Rd.m[i][j] = (i == j ? 1.0 : 0.0) + s * (K.m[i][j] + K2.m[i][j]);
    Rigid out;
    out.R = mul(Rd, T.R);
    out.t = add(mul(Rd, T.t), v3(x6[3], x6[4], x6[5]));
    return out;
}

static void butterfly32(double* x) {
    for (int o = 16; o > 0; o >>= 1) {
        double y[32];
        for (int l = 0; l < 32; ++l) y[l] = x[l] + x[l ^ o];
        for (int l = 0; l < 32; ++l) x[l] = y[l];
    }
}

// One ICP accumulation at T: the 28 reduced values and the pair count.
static void icp_accumulate(const EvalGrid& g, const std::vector<V3>& tgt_n_orig, const Cloud& source, const Rigid& T,
                           double max_dist, double* out, int64_t& count) {
    const int64_t n = static_cast<int64_t>(source.size());
    const int64_t n_chunks = (n + 255) / 256;
    const double d2_max = max_dist * max_dist;
    std::vector<double> chunk_vals(static_cast<size_t>(n_chunks) * kIcpVals, 0.0);
    int64_t total = 0;
    // chunks are independent (their values land in fixed slots): any thread
    // count gives the same bits
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : total)
    for (int64_t c = 0; c < n_chunks; ++c) {
        std::vector<double> contrib(static_cast<size_t>(256) * kIcpVals);
        for (int l = 0; l < 256; ++l) {
            double* v = &contrib[static_cast<size_t>(l) * kIcpVals];
            for (int q = 0; q < kIcpVals; ++q) v[q] = 0.0;
            const int64_t i = c * 256 + l;
            if (i >= n) continue;
            V3 y = apply(T, source.pos[static_cast<size_t>(i)]);
            int32_t slot;
            double d2;
            if (!eval_grid_nn(g, y, d2_max, slot, d2)) continue;
            const V3 q = g.slot_position[static_cast<size_t>(slot)];
            const V3 nn = g.slot_normal[static_cast<size_t>(slot)];
            if (is_zero(nn)) continue;
            const V3 d = sub(y, q);
            const double r = dot(d, nn);
            const V3 a = v3(y.y * nn.z - y.z * nn.y, y.z * nn.x - y.x * nn.z, y.x * nn.y - y.y * nn.x);
            const double J[6] = {a.x, a.y, a.z, nn.x, nn.y, nn.z};
            int k = 0;
            for (int u = 0; u < 6; ++u)
                for (int w = u; w < 6; ++w) v[k++] = J[u] * J[w];
            for (int u = 0; u < 6; ++u) v[k++] = J[u] * r;
            v[k] = r * r;
            total += 1;
        }
        for (int q = 0; q < kIcpVals; ++q) {
            double acc = 0.0;
            for (int w = 0; w < 8; ++w) {
                double x[32];
                for (int l = 0; l < 32; ++l) x[l] = contrib[static_cast<size_t>(w * 32 + l) * kIcpVals + q];
                butterfly32(x);
                acc = w == 0 ? x[0] : acc + x[0];
            }
            chunk_vals[static_cast<size_t>(c) * kIcpVals + q] = acc;
        }
    }
    (void)tgt_n_orig;
    count = total;
    for (int q = 0; q < kIcpVals; ++q) {
        double acc = 0.0;
        for (int64_t s0 = 0; s0 < n_chunks; s0 += 32) {
            double x[32];
            for (int l = 0; l < 32; ++l) x[l] = s0 + l < n_chunks ? chunk_vals[static_cast<size_t>(s0 + l) * kIcpVals + q] : 0.0;
            butterfly32(x);
            acc = acc + x[0];
        }
        out[q] = acc;
    }
}

static int icp_point_to_plane(const Cloud& source, const Cloud& target, const Rigid& T0, double max_dist,
                              int32_t max_iter, double eps, Rigid& T, or_icp_result& res, double* history) {
    if (source.pos.empty() || target.pos.empty()) fail(OR_EMPTY_CLOUD, "icp: empty cloud");
    if (!target.has_normals()) fail(OR_MISSING_NORMALS, "icp: target normals required");
    if (!(max_dist > 0.0)) fail(OR_INVALID_ARGUMENT, "icp: max_correspondence_distance must be positive");
    EvalGrid g = build_eval_grid(target, max_dist);
    T = T0;
    res = or_icp_result{};
    const double ns = static_cast<double>(source.size());
    for (int32_t it = 0; it < max_iter; ++it) {
        double vals[kIcpVals];
        int64_t cnt = 0;
        icp_accumulate(g, target.nrm, source, T, max_dist, vals, cnt);
        res.correspondences = cnt;
        res.fitness = static_cast<double>(cnt) / ns;
        res.rmse = cnt > 0 ? std::sqrt(vals[27] / static_cast<double>(cnt)) : 0.0;
        double x[6] = {0, 0, 0, 0, 0, 0};
        const bool ok = cnt >= 6 && icp_solve(vals, vals + 21, x);
        double dd = 0.0;
        if (ok) {
            for (int k = 0; k < 6; ++k) dd = dd + x[k] * x[k];
        }
        if (history) {
            history[3 * it] = static_cast<double>(cnt);
            history[3 * it + 1] = res.rmse;
            history[3 * it + 2] = dd;
        }
        if (!ok) {
            if (it == 0 && cnt < 6) fail(OR_NO_CORRESPONDENCES, "icp: fewer than 6 correspondences");
            res.iterations = it;
            return OR_OK;
        }
        T = icp_update(T, x);
        res.iterations = it + 1;
        if (dd < eps * eps) {
            res.converged = 1;
            return OR_OK;
        }
    }
    return OR_OK;
}

template <class F>
static int guarded(F&& f) {
    try {
        f();
        return OR_OK;
    } catch (const orc::Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return OR_ERROR;
    }
}

extern "C" {

const char* or_last_error(void) { return g_last_error.c_str(); }

uint64_t or_splitmix64(uint64_t x) { return splitmix64(x); }

void or_rng_u64(uint64_t seed, uint64_t stream, int64_t n, uint64_t* out) {
    Rng r(seed, stream);
    for (int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}
void or_rng_bounded(uint64_t seed, uint64_t stream, uint32_t bound, int64_t n, uint32_t* out) {
    Rng r(seed, stream);
    for (int64_t i = 0; i < n; ++i) out[i] = r.next_bounded(bound);
}
void or_rng_double(uint64_t seed, uint64_t stream, int64_t n, double* out) {
    Rng r(seed, stream);
    for (int64_t i = 0; i < n; ++i) out[i] = r.next_double();
}

int or_sample_quadruples(int32_t source_size, const int32_t* cache, int64_t cache_len, uint64_t seed, uint64_t stream,
                         int32_t trials, int32_t* out_src, int32_t* out_tgt) {
    return guarded([&] {
        Rng r(seed, stream);
        for (int t = 0; t < trials; ++t) {
            int s[4], d[4];
            sample_quadruple(source_size, cache, cache_len, r, s, d);
            for (int k = 0; k < 4; ++k) {
                out_src[4 * t + k] = s[k];
                out_tgt[4 * t + k] = d[k];
            }
        }
    });
}

int or_prerejected(const double* src12, const double* dst12, double tau) {
    V3 s[4], d[4];
    for (int k = 0; k < 4; ++k) {
        s[k] = load3(src12, k);
        d[k] = load3(dst12, k);
    }
    return prerejected(s, d, tau) ? 1 : 0;
}

int or_kabsch(const double* src, const double* dst, int64_t n, double* R9, double* t3, double* sigma3) {
    return guarded([&] {
        std::vector<V3> s(n), d(n);
        for (int64_t i = 0; i < n; ++i) {
            s[i] = load3(src, i);
            d[i] = load3(dst, i);
        }
        Rigid T = kabsch(s.data(), d.data(), n);
        store_m(R9, T.R);
        t3[0] = T.t.x;
        t3[1] = T.t.y;
        t3[2] = T.t.z;
        if (sigma3) {
            // singular values of the covariance for diagnostics
            V3 cs{}, cd{};
            for (int64_t i = 0; i < n; ++i) cs = add(cs, s[i]);
            for (int64_t i = 0; i < n; ++i) cd = add(cd, d[i]);
            cs = divs(cs, static_cast<double>(n));
            cd = divs(cd, static_cast<double>(n));
            M3 h;
            for (int64_t i = 0; i < n; ++i) {
                V3 a = sub(s[i], cs), b = sub(d[i], cd);
                for (int r = 0; r < 3; ++r)
                    for (int c = 0; c < 3; ++c) h.m[r][c] = h.m[r][c] + a[r] * b[c];
            }
            M3 U, V;
            jacobi_svd3(h, U, sigma3, V);
        }
    });
}

int or_svd3(const double* A9, double* U9, double* S3, double* V9) {
    return guarded([&] {
        M3 U, V;
        jacobi_svd3(load_m(A9), U, S3, V);
        store_m(U9, U);
        store_m(V9, V);
    });
}

void* or_search_grid_build(const double* xyz, int64_t n, double cell, const double* center3, int* status) {
    SearchGrid* out = nullptr;
    *status = guarded([&] {
        std::vector<V3> pts(n);
        for (int64_t i = 0; i < n; ++i) pts[i] = load3(xyz, i);
        V3 c = center3 ? v3(center3[0], center3[1], center3[2]) : V3{};
        out = new SearchGrid(build_grid(pts, cell, c));
    });
    return out;
}
void or_search_grid_free(void* g) { delete static_cast<SearchGrid*>(g); }
int or_nn_within(void* g, const double* q3, double d_max, int32_t* idx, double* dist) {
    Nn nn;
    if (!nn_within(*static_cast<SearchGrid*>(g), load3(q3, 0), d_max, &nn)) return 0;
    *idx = nn.index;
    *dist = nn.distance;
    return 1;
}
int or_nn_nearest(void* g, const double* q3, int32_t* idx, double* dist) {
    return guarded([&] {
        Nn nn = nn_nearest(*static_cast<SearchGrid*>(g), load3(q3, 0));
        *idx = nn.index;
        *dist = nn.distance;
    });
}
int64_t or_radius_search(void* g, const double* q3, double radius, int32_t* out, int64_t cap) {
    std::vector<int> r = radius_search(*static_cast<SearchGrid*>(g), load3(q3, 0), radius);
    for (int64_t i = 0; i < static_cast<int64_t>(r.size()) && i < cap; ++i) out[i] = r[i];
    return static_cast<int64_t>(r.size());
}
// reference.hpp:18-31
int or_bf_nn_within(const double* xyz, int64_t n, const double* q3, double d_max, int32_t* idx, double* dist) {
    double best_d2 = std::numeric_limits<double>::infinity();
    int best = -1;
    double d2_max = d_max * d_max;
    V3 q = load3(q3, 0);
    for (int64_t i = 0; i < n; ++i) {
        double d2 = sqnorm(sub(load3(xyz, i), q));
        if (d2 <= d2_max && d2 < best_d2) {
            best_d2 = d2;
            best = static_cast<int>(i);
        }
    }
    if (best < 0) return 0;
    *idx = best;
    *dist = std::sqrt(best_d2);
    return 1;
}

void* or_eval_grid_build(const double* xyz, const double* nxyz, int64_t n, double d_max, int* status) {
    EvalGrid* out = nullptr;
    *status = guarded([&] { out = new EvalGrid(build_eval_grid(make_cloud(xyz, nxyz, n), d_max)); });
    return out;
}
void or_eval_grid_free(void* g) { delete static_cast<EvalGrid*>(g); }
void or_eval_grid_dims(void* gp, double* origin3, double* cell, int32_t* dims3, int64_t* ncells, int64_t* npts) {
    auto* g = static_cast<EvalGrid*>(gp);
    origin3[0] = g->origin.x;
    origin3[1] = g->origin.y;
    origin3[2] = g->origin.z;
    *cell = g->cell;
    dims3[0] = g->nx;
    dims3[1] = g->ny;
    dims3[2] = g->nz;
    *ncells = static_cast<int64_t>(g->near_occupied.size());
    *npts = static_cast<int64_t>(g->index.size());
}
void or_eval_grid_arrays(void* gp, int32_t* start, int32_t* index, double* slot_pos, double* slot_nrm,
                         uint8_t* near_occupied) {
    auto* g = static_cast<EvalGrid*>(gp);
    if (start) std::memcpy(start, g->start.data(), g->start.size() * sizeof(int32_t));
    if (index) std::memcpy(index, g->index.data(), g->index.size() * sizeof(int32_t));
    for (size_t i = 0; i < g->index.size(); ++i) {
        if (slot_pos) store3(slot_pos, static_cast<int64_t>(i), g->slot_position[i]);
        if (slot_nrm) store3(slot_nrm, static_cast<int64_t>(i), g->slot_normal[i]);
    }
    if (near_occupied) std::memcpy(near_occupied, g->near_occupied.data(), g->near_occupied.size());
}
int or_evaluate_against_grid(void* gp, const double* src_xyz, const double* src_n, int64_t ns, const double* R9,
                             const double* t3, double d_max, double cos_max, int64_t miss_budget, double* ratio,
                             double* fitness, int64_t* inliers, int64_t* visited) {
    Cloud s = make_cloud(src_xyz, src_n, ns);
    WorkCounters wc;
    double r = 0, f = 0;
    int64_t inl = 0;
    bool ok = evaluate_against_grid(*static_cast<EvalGrid*>(gp), s, load_rigid(R9, t3), d_max, cos_max, miss_budget,
                                    r, f, inl, &wc);
    *ratio = r;
    *fitness = f;
    *inliers = inl;
    if (visited) *visited = wc.visited;
    return ok ? 1 : 0;
}

int or_evaluate_hypothesis(const double* R9, const double* t3, const double* src_xyz, const double* src_n,
                           int64_t ns, const double* tgt_xyz, const double* tgt_n, int64_t nt, double grid_cell,
                           const or_params* p, double* ratio, double* fitness, int64_t* inliers) {
    return guarded([&] {
        Cloud s = make_cloud(src_xyz, src_n, ns), t = make_cloud(tgt_xyz, tgt_n, nt);
        if (t.pos.empty() || s.pos.empty()) fail(OR_EMPTY_CLOUD, "evaluate_hypothesis: empty cloud");
        SearchGrid g = build_grid(t.pos, grid_cell, V3{});
        int64_t inl = 0;
        evaluate_hypothesis(load_rigid(R9, t3), s, t, g, p->d_max, p->normal_angle_max, *ratio, *fitness, inl);
        if (inliers) *inliers = inl;
    });
}

int or_score_candidates(const double* src_xyz, const double* src_n, int64_t ns, const double* tgt_xyz,
                        const double* tgt_n, int64_t nt, const double* Rt12, int64_t C, int32_t mode,
                        int32_t early_exit, double grid_cell, const or_params* p, double* out_ratio,
                        double* out_fitness, int64_t* out_inliers, int32_t* out_scored, or_result* best,
                        int64_t* qualified) {
    return guarded([&] {
        Cloud s = make_cloud(src_xyz, src_n, ns), t = make_cloud(tgt_xyz, tgt_n, nt);
        if (s.pos.empty() || t.pos.empty()) fail(OR_EMPTY_CLOUD, "score_candidates: empty cloud");
        if (!s.has_normals() || !t.has_normals()) fail(OR_MISSING_NORMALS, "score_candidates: normals required");
        const double cos_max = std::cos(p->normal_angle_max);
        const double max_fitness = resolved_max_fitness(*p);
        const int64_t budget = early_exit ? static_cast<int64_t>(s.size()) -
                                                static_cast<int64_t>(std::ceil(p->min_inlier_ratio * static_cast<double>(s.size())))
                                          : std::numeric_limits<int64_t>::max();
        EvalGrid eg;
        SearchGrid sg;
        if (mode == 0)
            eg = build_eval_grid(t, p->d_max);
        else
            sg = build_grid(t.pos, grid_cell, V3{});
        int threads = p->threads > 0 ? p->threads : omp_get_max_threads();
        Best global;
        int64_t qual = 0;
#pragma omp parallel num_threads(threads) reduction(+ : qual)
        {
            Best local;
#pragma omp for schedule(dynamic, 16)
            for (int64_t c = 0; c < C; ++c) {
                Rigid T = load_rigid(Rt12 + 12 * c, Rt12 + 12 * c + 9);
                double r = 0, f = 0;
                int64_t inl = 0;
                bool scored = true;
                if (mode == 0)
                    scored = evaluate_against_grid(eg, s, T, p->d_max, cos_max, budget, r, f, inl, nullptr);
                else
                    evaluate_hypothesis(T, s, t, sg, p->d_max, p->normal_angle_max, r, f, inl);
                if (out_ratio) out_ratio[c] = scored ? r : 0.0;
                if (out_fitness) out_fitness[c] = scored ? f : 0.0;
                if (out_inliers) out_inliers[c] = scored ? inl : -1;
                if (out_scored) out_scored[c] = scored ? 1 : 0;
                if (!scored || r < p->min_inlier_ratio || f > max_fitness) continue;
                qual += 1;
                Best cand;
                cand.ratio = r;
                cand.fitness = f;
                cand.index = c;
                cand.inliers = inl;
                cand.transform = T;
                cand.valid = true;
                if (!local.valid || better(cand, local)) local = cand;
            }
#pragma omp critical(or_cand_best)
            {
                if (local.valid && (!global.valid || better(local, global))) global = local;
            }
        }
        if (qualified) *qualified = qual;
        if (best) {
            std::memset(best, 0, sizeof(*best));
            best->hypothesis_index = -1;
            if (global.valid) {
                store_m(best->R, global.transform.R);
                best->t[0] = global.transform.t.x;
                best->t[1] = global.transform.t.y;
                best->t[2] = global.transform.t.z;
                best->inlier_ratio = global.ratio;
                best->fitness = global.fitness;
                best->inliers = global.inliers;
                best->hypothesis_index = global.index;
                best->found = 1;
            }
        }
    });
}

int or_voxel_downsample(const double* xyz, const double* nxyz, int64_t n, double leaf, double* out_xyz,
                        double* out_n, int64_t* out_count) {
    return guarded([&] {
        Cloud d = voxel_downsample(make_cloud(xyz, nxyz, n), leaf);
        for (size_t i = 0; i < d.size(); ++i) {
            store3(out_xyz, static_cast<int64_t>(i), d.pos[i]);
            if (out_n && d.has_normals()) store3(out_n, static_cast<int64_t>(i), d.nrm[i]);
        }
        *out_count = static_cast<int64_t>(d.size());
    });
}

int or_estimate_normals(const double* xyz, int64_t n, double radius, const double* viewpoint, int32_t threads,
                        double* out) {
    return guarded([&] {
        Cloud c = estimate_normals(make_cloud(xyz, nullptr, n), radius, viewpoint ? load3(viewpoint, 0) : V3{},
                                   threads);
        for (size_t i = 0; i < c.nrm.size(); ++i) store3(out, static_cast<int64_t>(i), c.nrm[i]);
    });
}

int or_compute_fpfh(const double* xyz, const double* nxyz, int64_t n, double radius, int32_t threads, float* out) {
    return guarded([&] {
        auto f = compute_fpfh(make_cloud(xyz, nxyz, n), radius, threads);
        for (size_t i = 0; i < f.size(); ++i) std::memcpy(out + 33 * i, f[i].data(), 33 * sizeof(float));
    });
}

int or_feature_nn_cache(const float* sf, int64_t ns, const float* tf, int64_t nt, int32_t threads, int32_t* out) {
    return guarded([&] {
        auto c = feature_nn_cache(sf, ns, tf, nt, threads);
        std::memcpy(out, c.data(), c.size() * sizeof(int32_t));
    });
}

void* or_prepare(const double* sxyz, const double* sn, int64_t ns, const double* txyz, const double* tn, int64_t nt,
                 const or_params* p, int* status) {
    Context* out = nullptr;
    *status = guarded([&] {
        if (ns <= 0 || nt <= 0) fail(OR_EMPTY_CLOUD, "voxel_downsample: empty cloud");
        out = prepare(make_cloud(sxyz, sn, ns), make_cloud(txyz, tn, nt), *p);
    });
    return out;
}

void* or_ctx_from_prepared(const double* sxyz, const double* sn, int64_t ns, const double* txyz, const double* tn,
                           int64_t nt, const int32_t* cache, double d_max, int* status) {
    Context* out = nullptr;
    *status = guarded([&] {
        auto ctx = std::make_unique<Context>();
        ctx->source = make_cloud(sxyz, sn, ns);
        ctx->target = make_cloud(txyz, tn, nt);
        ctx->cache.assign(cache, cache + ns);
        ctx->eval = build_eval_grid(ctx->target, d_max);
        out = ctx.release();
    });
    return out;
}

void or_ctx_sizes(void* cp, int64_t* ns, int64_t* nt) {
    auto* c = static_cast<Context*>(cp);
    *ns = static_cast<int64_t>(c->source.size());
    *nt = static_cast<int64_t>(c->target.size());
}

void or_ctx_get(void* cp, double* sxyz, double* sn, double* txyz, double* tn, int32_t* cache, float* sfeat,
                float* tfeat) {
    auto* c = static_cast<Context*>(cp);
    for (size_t i = 0; i < c->source.size(); ++i) {
        if (sxyz) store3(sxyz, static_cast<int64_t>(i), c->source.pos[i]);
        if (sn) store3(sn, static_cast<int64_t>(i), c->source.nrm[i]);
    }
    for (size_t i = 0; i < c->target.size(); ++i) {
        if (txyz) store3(txyz, static_cast<int64_t>(i), c->target.pos[i]);
        if (tn) store3(tn, static_cast<int64_t>(i), c->target.nrm[i]);
    }
    if (cache) std::memcpy(cache, c->cache.data(), c->cache.size() * sizeof(int32_t));
    if (sfeat && !c->sfeat.empty()) std::memcpy(sfeat, c->sfeat.data(), c->sfeat.size() * 33 * sizeof(float));
    if (tfeat && !c->tfeat.empty()) std::memcpy(tfeat, c->tfeat.data(), c->tfeat.size() * 33 * sizeof(float));
}

void or_ctx_free(void* cp) { delete static_cast<Context*>(cp); }

int or_run_hypotheses(void* cp, const or_params* p, int64_t begin, int64_t end, or_result* res, or_stats* st) {
    return guarded([&] {
        if (st) std::memset(st, 0, sizeof(*st));
        run_hypotheses(*static_cast<Context*>(cp), *p, begin, end, res, st);
    });
}

int or_better(const or_result* a, const or_result* b) {
    Best x, y;
    x.ratio = a->inlier_ratio;
    x.fitness = a->fitness;
    x.index = a->hypothesis_index;
    y.ratio = b->inlier_ratio;
    y.fitness = b->fitness;
    y.index = b->hypothesis_index;
    return better(x, y) ? 1 : 0;
}

int or_edge_info(const double* ci, int64_t ni, const double* cj, int64_t nj, const double* Ri9, const double* ti3,
                 const double* Rj9, const double* tj3, double epsilon, double* info36, int64_t* pair_count) {
    return guarded([&] {
        edge_info(make_cloud(ci, nullptr, ni), make_cloud(cj, nullptr, nj), load_rigid(Ri9, ti3),
                  load_rigid(Rj9, tj3), epsilon, info36, *pair_count);
    });
}

int or_icp_point_to_plane(const double* sxyz, int64_t ns, const double* txyz, const double* tn, int64_t nt,
                          const double* R0, const double* t0, double max_dist, int32_t max_iter, double eps,
                          double* R9, double* t3, or_icp_result* res, double* history) {
    return guarded([&] {
        Rigid T;
        icp_point_to_plane(make_cloud(sxyz, nullptr, ns), make_cloud(txyz, tn, nt), load_rigid(R0, t0), max_dist,
                           max_iter, eps, T, *res, history);
        store_m(R9, T.R);
        t3[0] = T.t.x;
        t3[1] = T.t.y;
        t3[2] = T.t.z;
    });
}

// propose_loops' overlap of one pair (fragments.cpp:67-100): the later cloud
// posed by T_later, hits within r of the earlier cloud posed by T_earlier
// (SearchGrid at cell r, center 0).
int or_overlap_hits(const double* later, int64_t nl, const double* Rl9, const double* tl3, const double* earlier,
                    int64_t ne, const double* Re9, const double* te3, double r, int64_t* hits) {
    return guarded([&] {
        const Rigid Tl = load_rigid(Rl9, tl3), Te = load_rigid(Re9, te3);
        std::vector<V3> pe;
        pe.reserve(static_cast<size_t>(ne));
        for (int64_t i = 0; i < ne; ++i) pe.push_back(apply(Te, load3(earlier, i)));
        SearchGrid grid = build_grid(pe, r, V3{});
        int64_t h = 0;
        for (int64_t i = 0; i < nl; ++i) {
            Nn nn;
            if (nn_within(grid, apply(Tl, load3(later, i)), r, &nn)) h += 1;
        }
        *hits = h;
    });
}

}  // extern "C"
