// Compiles the C++ shim (include/loopkit_b200/registration.hpp) against
// reference-shaped types and exercises its error mapping / results.
// usage: test_shim cpu   -> expects CudaError (no device: no CPU fallback)
//        test_shim gpu   -> registers a planted pair and prints the result
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <optional>
#include <random>
#include <vector>

#include "loopkit_b200/registration.hpp"

struct Vec3 {  // stands in for Eigen::Vector3d: 3 packed doubles
    double x, y, z;
};
struct PointCloud {  // proj/include/loopkit/geometry.hpp:92-99
    std::vector<Vec3> positions;
    std::vector<Vec3> normals;
};
struct Rigid {  // proj/include/loopkit/geometry.hpp:20-38 (rotation(r, c), translation[k])
    struct M {
        double m[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
        double operator()(int r, int c) const { return m[r][c]; }
    } rotation;
    std::array<double, 3> translation{0, 0, 0};
};
struct Fragment {  // proj/include/loopkit/fragments.hpp:18-25
    PointCloud cloud;
};
struct LoopEdge {  // proj/include/loopkit/pose_graph.hpp (i, j)
    int i = 0, j = 0;
};
struct PoseGraph {
    std::vector<Rigid> poses;
    std::vector<LoopEdge> loops;
};
struct LoopParams {  // proj/include/loopkit/fragments.hpp:39-42
    double overlap_radius = 0.1;
    double min_overlap = 0.2;
};
struct RegistrationParams {  // proj/include/loopkit/registration.hpp:17-32
    double leaf = 0.05;
    double normal_radius = 0.1;
    double feature_radius = 0.25;
    std::int64_t hypothesis_count = 4'000'000;
    double similarity_tau = 0.9;
    double d_max = 0.075;
    double min_inlier_ratio = 0.25;
    std::optional<double> max_fitness;
    double normal_angle_max = 30.0 * M_PI / 180.0;
    std::uint64_t seed = 0;
    int threads = 0;
};

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
    PointCloud tiny;
    tiny.positions = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}};
    tiny.normals = {{0, 0, 1}, {0, 0, 1}, {0, 0, 1}};
    RegistrationParams params;
    params.hypothesis_count = 10'000;
    // a box-shaped cloud and a shifted copy
    PointCloud src, tgt;
    std::mt19937 rng(5);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    for (int i = 0; i < 6000; ++i) {
        int face = i % 3;
        Vec3 p{u(rng), u(rng), u(rng)};
        Vec3 n{0, 0, 0};
        if (face == 0) { p.x = -1; n.x = 1; }
        if (face == 1) { p.y = -1; n.y = 1; }
        if (face == 2) { p.z = -1; n.z = 1; }
        src.positions.push_back(p);
        src.normals.push_back(n);
        tgt.positions.push_back({p.x + 0.1, p.y - 0.05, p.z + 0.02});
        tgt.normals.push_back(n);
    }
    if (!gpu) {
        try {
            loopkit_b200::register_global(src, tgt, params);
            std::puts("FAIL: expected CudaError without a device");
            return 1;
        } catch (const loopkit_b200::CudaError& e) {
            std::printf("ok: CudaError (%s)\n", e.what());
        }
        return 0;
    }
    try {
        loopkit_b200::register_global(tiny, tgt, params);
        std::puts("FAIL: expected TooFewPoints");
        return 1;
    } catch (const loopkit_b200::TooFewPoints&) {
        std::puts("ok: TooFewPoints");
    }
    loopkit_b200::HypothesisStats st{};
    auto r = loopkit_b200::register_global(src, tgt, params, &st);
    if (!r) {
        std::puts("FAIL: no alignment");
        return 1;
    }
    std::printf("ok: index %lld inliers %lld ratio %.6f t = %.4f %.4f %.4f sampled %lld\n",
                (long long)r->hypothesis_index, (long long)r->inliers, r->inlier_ratio, r->transform.t[0],
                r->transform.t[1], r->transform.t[2], (long long)st.sampled);
    auto ef = loopkit_b200::evaluate_hypothesis(r->transform, src, tgt, 0.075, params);
    std::printf("ok: evaluate_hypothesis ratio %.6f fitness %.3e\n", ef.first, ef.second);
    loopkit_b200::Transform I{{1, 0, 0, 0, 1, 0, 0, 0, 1}, {0, 0, 0}};
    auto ei = loopkit_b200::edge_info(tgt, src, I, r->transform, 0.05);
    std::printf("ok: edge_info pair_count %lld\n", (long long)ei.pair_count);
    try {
        loopkit_b200::edge_info(tiny, tiny, I, loopkit_b200::Transform{{1, 0, 0, 0, 1, 0, 0, 0, 1}, {9, 9, 9}}, 0.05);
        std::puts("FAIL: expected NoCorrespondences");
        return 1;
    } catch (const loopkit_b200::NoCorrespondences&) {
        std::puts("ok: NoCorrespondences");
    }
    // propose_loops: three copies of src at the identity -> only (2, 0) (test_fragments.cpp:183-200)
    std::vector<Fragment> frags(3);
    PoseGraph graph;
    for (auto& f : frags) {
        f.cloud.positions = src.positions;
        graph.poses.emplace_back();
    }
    LoopParams lp;
    lp.min_overlap = 0.0;
    auto props = loopkit_b200::propose_loops(frags, graph, lp);
    if (props.size() != 1 || props[0].i != 2 || props[0].j != 0 || props[0].overlap != 1.0) {
        std::puts("FAIL: propose_loops");
        return 1;
    }
    graph.loops.push_back({0, 2});
    if (!loopkit_b200::propose_loops(frags, graph, lp).empty()) {
        std::puts("FAIL: propose_loops linked pair");
        return 1;
    }
    std::puts("ok: propose_loops (2, 0)");
    auto icp = loopkit_b200::icp_point_to_plane(src, tgt, r->transform, 0.05);
    std::printf("ok: icp iterations %d converged %d rmse %.3e t = %.4f %.4f %.4f\n", icp.iterations,
                icp.converged ? 1 : 0, icp.rmse, icp.transform.t[0], icp.transform.t[1], icp.transform.t[2]);
    return 0;
}
