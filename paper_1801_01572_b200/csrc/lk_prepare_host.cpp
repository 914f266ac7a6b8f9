// lk_prepare_host.cpp -- see lk_prepare_host.hpp.
#include "lk_prepare_host.hpp"

#include <algorithm>
#include <limits>

#include <omp.h>

#include "../../include/loopkit_b200.h"

namespace lk {

Cloud make_cloud(const double* xyz, const double* nxyz, int64_t n) {
    Cloud c;
    c.pos.resize(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) c.pos[i] = load3(xyz, i);
    if (nxyz) {
        c.nrm.resize(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) c.nrm[i] = load3(nxyz, i);
    }
    return c;
}

// proj/src/geometry.cpp:93-103
void validate_cloud(const Cloud& c) {
    if (!c.nrm.empty() && c.nrm.size() != c.pos.size())
        throw Status(LK_MISSING_NORMALS, "normals array must be empty or match positions");
    for (const Vec3& n : c.nrm) {
        double len = norm(n);
        if (len != 0.0 && std::abs(len - 1.0) > 1e-6)
            throw Status(LK_MISSING_NORMALS, "normals must be unit length or exactly zero");
    }
}

static inline uint64_t voxel_key(int x, int y, int z) {
    constexpr int64_t off = 1 << 20;
    return (static_cast<uint64_t>(x + off) << 42) | (static_cast<uint64_t>(y + off) << 21) |
           static_cast<uint64_t>(z + off);
}

// proj/src/preprocess.cpp:14-59: origin-anchored voxels, mean position,
// normalised mean of the non-zero normals, output ordered by the first input
// index that fell in each voxel.
Cloud voxel_downsample(const Cloud& cloud, double leaf) {
    if (cloud.pos.empty()) throw Status(LK_EMPTY_CLOUD, "voxel_downsample: empty cloud");
    if (!(leaf > 0.0)) throw Status(LK_INVALID_ARGUMENT, "voxel_downsample: leaf must be positive");
    validate_cloud(cloud);
    struct Accum {
        Vec3 pos_sum{}, normal_sum{};
        int count = 0;
        int min_index = 0;
    };
    std::unordered_map<uint64_t, int> slot_of;
    slot_of.reserve(cloud.size());
    std::vector<Accum> acc;  // in first-seen order == ascending min_index
    acc.reserve(cloud.size() / 4 + 16);
    const Vec3 zero{};
    for (size_t i = 0; i < cloud.size(); ++i) {
        Vec3 q = (cloud.pos[i] - zero) / leaf;
        uint64_t key = voxel_key(floor_to_int(q.x), floor_to_int(q.y), floor_to_int(q.z));
        auto ins = slot_of.try_emplace(key, static_cast<int>(acc.size()));
        if (ins.second) {
            acc.emplace_back();
            acc.back().min_index = static_cast<int>(i);
        }
        Accum& a = acc[ins.first->second];
        a.pos_sum = a.pos_sum + cloud.pos[i];
        if (cloud.has_normals() && !is_zero(cloud.nrm[i])) a.normal_sum = a.normal_sum + cloud.nrm[i];
        a.count += 1;
    }
    Cloud out;
    out.pos.reserve(acc.size());
    if (cloud.has_normals()) out.nrm.reserve(acc.size());
    for (const Accum& a : acc) {
        out.pos.push_back(a.pos_sum / static_cast<double>(a.count));
        if (cloud.has_normals()) {
            double len = norm(a.normal_sum);
            out.nrm.push_back(len > 1e-12 ? a.normal_sum / len : Vec3{});
        }
    }
    return out;
}

// proj/src/geometry.cpp:105-114
Cloud transformed(const Cloud& c, const Rigid& t) {
    Cloud out;
    out.pos.reserve(c.pos.size());
    for (const Vec3& p : c.pos) out.pos.push_back(apply(t, p));
    out.nrm.reserve(c.nrm.size());
    for (const Vec3& n : c.nrm) out.nrm.push_back(is_zero(n) ? n : t.R * n);
    return out;
}

// proj/src/geometry.cpp:116-121
Vec3 centroid(const Cloud& c) {
    if (c.pos.empty()) throw Status(LK_EMPTY_CLOUD, "centroid: empty cloud");
    Vec3 s{};
    for (const Vec3& p : c.pos) s = s + p;
    return s / static_cast<double>(c.size());
}

static inline void cell_of(const HostGrid& g, Vec3 p, int c[3]) {
    Vec3 q = (p - g.center) / g.cell;
    c[0] = floor_to_int(q.x);
    c[1] = floor_to_int(q.y);
    c[2] = floor_to_int(q.z);
}

void build_host_grid(HostGrid& g, const std::vector<Vec3>& pts, double cell, Vec3 center) {
    if (pts.empty()) throw Status(LK_EMPTY_CLOUD, "build_grid: empty cloud");
    if (!(cell > 0.0)) throw Status(LK_INVALID_ARGUMENT, "build_grid: cell_length must be positive");
    g.cell = cell;
    g.center = center;
    g.points = &pts;
    const int n = static_cast<int>(pts.size());
    std::vector<uint64_t> keys(n);
    for (int a = 0; a < 3; ++a) {
        g.cmin[a] = std::numeric_limits<int>::max();
        g.cmax[a] = std::numeric_limits<int>::min();
    }
    g.cells.clear();
    for (int i = 0; i < n; ++i) {
        int c[3];
        cell_of(g, pts[i], c);
        for (int a = 0; a < 3; ++a) {
            g.cmin[a] = std::min(g.cmin[a], c[a]);
            g.cmax[a] = std::max(g.cmax[a], c[a]);
        }
        keys[i] = voxel_key(c[0], c[1], c[2]);
        g.cells.try_emplace(keys[i], 0, 0).first->second.second += 1;
    }
    int start = 0;
    for (auto& kv : g.cells) {
        kv.second.first = start;
        start += kv.second.second;
        kv.second.second = 0;
    }
    g.cell_points.assign(n, 0);
    for (int i = 0; i < n; ++i) {
        auto& r = g.cells[keys[i]];
        g.cell_points[r.first + r.second] = i;
        r.second += 1;
    }
}

int host_nn_within(const HostGrid& g, Vec3 q, double d_max, double* best_d2_out) {
    int c = static_cast<int>(std::ceil(d_max / g.cell));
    double d2_max = d_max * d_max;
    int qc[3];
    cell_of(g, q, qc);
    double best_d2 = std::numeric_limits<double>::infinity();
    int best = std::numeric_limits<int>::max();
    int lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
        lo[a] = std::max(qc[a] - c, g.cmin[a]);
        hi[a] = std::min(qc[a] + c, g.cmax[a]);
    }
    const std::vector<Vec3>& P = *g.points;
    for (int x = lo[0]; x <= hi[0]; ++x)
        for (int y = lo[1]; y <= hi[1]; ++y)
            for (int z = lo[2]; z <= hi[2]; ++z) {
                auto it = g.cells.find(voxel_key(x, y, z));
                if (it == g.cells.end()) continue;
                const int* ids = g.cell_points.data() + it->second.first;
                for (int k = 0; k < it->second.second; ++k) {
                    int idx = ids[k];
                    double d2 = squared_norm(P[idx] - q);
                    if (d2 > d2_max) continue;
                    if (d2 < best_d2 || (d2 == best_d2 && idx < best)) {
                        best_d2 = d2;
                        best = idx;
                    }
                }
            }
    if (best == std::numeric_limits<int>::max()) return -1;
    if (best_d2_out) *best_d2_out = best_d2;
    return best;
}

std::vector<int> host_radius_search(const HostGrid& g, Vec3 q, double radius) {
    std::vector<int> out;
    int c = static_cast<int>(std::ceil(radius / g.cell));
    double r2 = radius * radius;
    int qc[3];
    cell_of(g, q, qc);
    int lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
        lo[a] = std::max(qc[a] - c, g.cmin[a]);
        hi[a] = std::min(qc[a] + c, g.cmax[a]);
    }
    const std::vector<Vec3>& P = *g.points;
    for (int x = lo[0]; x <= hi[0]; ++x)
        for (int y = lo[1]; y <= hi[1]; ++y)
            for (int z = lo[2]; z <= hi[2]; ++z) {
                auto it = g.cells.find(voxel_key(x, y, z));
                if (it == g.cells.end()) continue;
                const int* ids = g.cell_points.data() + it->second.first;
                for (int k = 0; k < it->second.second; ++k)
                    if (squared_norm(P[ids[k]] - q) <= r2) out.push_back(ids[k]);
            }
    std::sort(out.begin(), out.end());
    return out;
}

// proj/src/fpfh.cpp:17-48
static bool pair_angles(Vec3 p1, Vec3 n1, Vec3 p2, Vec3 n2, double& alpha, double& phi, double& theta) {
    Vec3 d = p2 - p1;
    double dist = norm(d);
    if (dist <= 0.0) return false;
    double angle1 = dot(n1, d) / dist;
    double angle2 = dot(n2, d) / dist;
    Vec3 ns = n1, nt = n2, line = d;
    double cos_line = angle1;
    if (std::acos(std::abs(angle1)) > std::acos(std::abs(angle2))) {
        ns = n2;
        nt = n1;
        line = -d;
        cos_line = -angle2;
    }
    Vec3 u = ns;
    Vec3 v = cross(line, u);
    double v_len = norm(v);
    if (v_len <= 1e-12 * dist) return false;
    v = v / v_len;
    Vec3 w = cross(u, v);
    alpha = dot(v, nt);
    phi = cos_line;
    theta = std::atan2(dot(w, nt), dot(u, nt));
    return true;
}

// proj/src/fpfh.cpp:50-53
static inline int bin_index(double value, double lo, double hi) {
    int b = floor_to_int(11 * (value - lo) / (hi - lo));
    return std::clamp(b, 0, 10);
}

// proj/src/fpfh.cpp:57-141
std::vector<Feature> compute_fpfh(const Cloud& cloud, double radius, int threads) {
    if (cloud.pos.empty()) throw Status(LK_EMPTY_CLOUD, "compute_fpfh: empty cloud");
    if (!cloud.has_normals()) throw Status(LK_MISSING_NORMALS, "compute_fpfh: cloud has no normals");
    validate_cloud(cloud);
    const int n = static_cast<int>(cloud.size());
    HostGrid grid;
    build_host_grid(grid, cloud.pos, radius, Vec3{});
    if (threads <= 0) threads = omp_get_max_threads();
    std::vector<std::vector<int>> nbr(n);
#pragma omp parallel for schedule(dynamic, 64) num_threads(threads)
    for (int i = 0; i < n; ++i) {
        std::vector<int> v = host_radius_search(grid, cloud.pos[i], radius);
        v.erase(std::remove(v.begin(), v.end(), i), v.end());
        nbr[i] = std::move(v);
    }
    std::vector<std::array<double, 33>> spfh(n);
#pragma omp parallel for schedule(dynamic, 64) num_threads(threads)
    for (int i = 0; i < n; ++i) {
        auto& h = spfh[i];
        h.fill(0.0);
        Vec3 p = cloud.pos[i], np = cloud.nrm[i];
        if (is_zero(np)) continue;
        int votes = 0;
        for (int j : nbr[i]) {
            Vec3 nq = cloud.nrm[j];
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
    std::vector<Feature> out(n);
#pragma omp parallel for schedule(dynamic, 64) num_threads(threads)
    for (int i = 0; i < n; ++i) {
        out[i].fill(0.0f);
        if (is_zero(cloud.nrm[i])) continue;
        Vec3 p = cloud.pos[i];
        std::array<double, 33> acc{};
        int k_count = 0;
        for (int j : nbr[i]) {
            if (is_zero(cloud.nrm[j])) continue;
            double w = norm(cloud.pos[j] - p);
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

}  // namespace lk
