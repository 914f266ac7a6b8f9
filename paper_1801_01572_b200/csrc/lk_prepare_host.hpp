// lk_prepare_host.hpp -- host restatements used by the FIXTURE library only
// (libloopkit_synth.so: voxel_downsample, transformed, centroid, a SearchGrid
// for the synth_registration_pair overlap test). The product library never
// links them: prepare_registration runs on the device (lk_prepare.cu).
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "lk_host_math.hpp"

namespace lk {

struct Cloud {
    std::vector<Vec3> pos;
    std::vector<Vec3> nrm;  // empty or parallel to pos
    size_t size() const { return pos.size(); }
    bool has_normals() const { return !nrm.empty(); }
};

Cloud make_cloud(const double* xyz, const double* nxyz, int64_t n);
void validate_cloud(const Cloud& c);
Cloud voxel_downsample(const Cloud& cloud, double leaf);
Cloud transformed(const Cloud& c, const Rigid& t);
Vec3 centroid(const Cloud& c);

// Sparse CSR hash grid (proj/src/grid.cpp:32-66) used by host-side stages.
struct HostGrid {
    double cell = 1.0;
    Vec3 center{};
    const std::vector<Vec3>* points = nullptr;
    std::vector<int> cell_points;
    std::unordered_map<uint64_t, std::pair<int, int>> cells;
    int cmin[3] = {0, 0, 0}, cmax[3] = {0, 0, 0};
};
void build_host_grid(HostGrid& g, const std::vector<Vec3>& pts, double cell, Vec3 center);
// exact NN within d_max, ties -> lowest index (grid.cpp:101-109); returns index or -1
int host_nn_within(const HostGrid& g, Vec3 q, double d_max, double* best_d2);
std::vector<int> host_radius_search(const HostGrid& g, Vec3 q, double radius);

using Feature = std::array<float, 33>;
std::vector<Feature> compute_fpfh(const Cloud& cloud, double radius, int threads);

inline int floor_to_int(double q) {
    double f = std::floor(q);
    if (!(f >= -2147483648.0 && f < 2147483648.0)) return INT32_MIN;
    return static_cast<int>(f);
}

}  // namespace lk
