// loopkit_b200/registration.hpp -- header-only C++ shim over include/loopkit_b200.h
// that re-exposes the reference registration API
// (/root/reference/proj/include/loopkit/registration.hpp) with the same names,
// argument meaning and error behaviour: lk_status codes are turned back into
// the reference's exception types (proj/include/loopkit/errors.hpp) and
// LK_NO_ALIGNMENT into std::nullopt.
//
// The shim is generic over the caller's cloud / params / result types so the
// reference's own Eigen types plug in unchanged:
//   Cloud   : .positions / .normals, contiguous 3-double elements
//             (std::vector<Eigen::Vector3d> qualifies)
//   Params  : the RegistrationParams fields (registration.hpp:17-32)
//   Errors  : a struct with the exception types as nested typedefs; the default
//             `DefaultErrors` below defines them in namespace loopkit_b200.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <iterator>
#include <optional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "../loopkit_b200.h"

namespace loopkit_b200 {

// errors.hpp:9-74 (subset used by the registration path)
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct EmptyCloud : Error { using Error::Error; };
struct TooFewPoints : Error { using Error::Error; };
struct MissingNormals : Error { using Error::Error; };
struct MissingData : Error { using Error::Error; };
struct NoCorrespondences : Error { using Error::Error; };
struct DegenerateConfiguration : Error { using Error::Error; };
struct CudaError : Error { using Error::Error; };

struct DefaultErrors {
    using Base = Error;
    using EmptyCloudT = EmptyCloud;
    using TooFewPointsT = TooFewPoints;
    using MissingNormalsT = MissingNormals;
    using MissingDataT = MissingData;
    using NoCorrespondencesT = NoCorrespondences;
    using DegenerateT = DegenerateConfiguration;
    using DeviceT = CudaError;
};

template <class E = DefaultErrors>
[[noreturn]] inline void throw_status(lk_status s) {
    const char* m = lk_last_error();
    std::string msg = m && *m ? m : "loopkit_b200 error";
    switch (s) {
        case LK_EMPTY_CLOUD: throw typename E::EmptyCloudT(msg);
        case LK_TOO_FEW_POINTS: throw typename E::TooFewPointsT(msg);
        case LK_MISSING_NORMALS: throw typename E::MissingNormalsT(msg);
        case LK_MISSING_DATA: throw typename E::MissingDataT(msg);
        case LK_NO_CORRESPONDENCES: throw typename E::NoCorrespondencesT(msg);
        case LK_DEGENERATE: throw typename E::DegenerateT(msg);
        case LK_CUDA_ERROR:
        case LK_NCCL_ERROR: throw typename E::DeviceT(msg);
        default: throw typename E::Base(msg);
    }
}

template <class E = DefaultErrors>
inline bool check(lk_status s) {  // true: found; false: no alignment
    if (s == LK_OK) return true;
    if (s == LK_NO_ALIGNMENT) return false;
    throw_status<E>(s);
}

// View of a cloud with contiguous xyz triples (no copy). lk_cloud carries one
// count for both arrays, so a normals array that is neither empty nor
// parallel to the positions throws MissingNormals here, as validate_cloud
// does (geometry.cpp:93-96), instead of letting the library read past it.
template <class E = DefaultErrors, class Cloud>
inline lk_cloud as_lk_cloud(const Cloud& c) {
    if (!c.normals.empty() && c.normals.size() != c.positions.size())
        throw typename E::MissingNormalsT("normals array must be empty or match positions");
    lk_cloud out{};
    out.n = static_cast<int64_t>(c.positions.size());
    out.xyz = out.n ? reinterpret_cast<const double*>(c.positions.data()) : nullptr;
    out.nxyz = (!c.normals.empty()) ? reinterpret_cast<const double*>(c.normals.data()) : nullptr;
    static_assert(sizeof(c.positions[0]) == 3 * sizeof(double), "positions must be packed xyz doubles");
    return out;
}

// GPUs per call: the caller's Params::device_count when it has one, else the
// LK_DEVICE_COUNT environment variable (so the reference's own callers, whose
// RegistrationParams have no such field, can opt in unchanged), else 1.
template <class P, class = void>
struct has_device_count : std::false_type {};
template <class P>
struct has_device_count<P, std::void_t<decltype(std::declval<const P&>().device_count)>> : std::true_type {};
template <class Params>
inline int32_t device_count_of(const Params& p) {
    if constexpr (has_device_count<Params>::value) {
        return static_cast<int32_t>(p.device_count);
    } else {
        const char* v = std::getenv("LK_DEVICE_COUNT");
        return v ? static_cast<int32_t>(std::atoi(v)) : 0;
    }
}

template <class Params>
inline lk_reg_params to_lk_params(const Params& p, int32_t device = -1, int32_t device_count = -2) {
    lk_reg_params o{};
    o.leaf = p.leaf;
    o.normal_radius = p.normal_radius;
    o.feature_radius = p.feature_radius;
    o.hypothesis_count = p.hypothesis_count;
    o.similarity_tau = p.similarity_tau;
    o.d_max = p.d_max;
    o.min_inlier_ratio = p.min_inlier_ratio;
    o.max_fitness = p.max_fitness ? static_cast<double>(*p.max_fitness) : -1.0;  // std::optional<double>
    o.normal_angle_max = p.normal_angle_max;
    o.seed = p.seed;
    o.threads = p.threads;
    o.device = device;
    o.device_count = device_count == -2 ? device_count_of(p) : device_count;  // GPUs of one call
    return o;
}

// Result types of the shim (the reference's RegistrationResult /
// HypothesisStats are filled through `fill` callbacks in INTEGRATION.md).
struct Transform {
    double R[9];  // row-major
    double t[3];
};
struct RegistrationResult {
    Transform transform;
    double inlier_ratio = 0.0;
    double fitness = 0.0;
    std::int64_t hypothesis_index = -1;
    std::int64_t inliers = 0;
};
using HypothesisStats = lk_hyp_stats;

inline RegistrationResult from_lk(const lk_reg_result& r) {
    RegistrationResult o;
    for (int k = 0; k < 9; ++k) o.transform.R[k] = r.R[k];
    for (int k = 0; k < 3; ++k) o.transform.t[k] = r.t[k];
    o.inlier_ratio = r.inlier_ratio;
    o.fitness = r.fitness;
    o.hypothesis_index = r.hypothesis_index;
    o.inliers = r.inliers;
    return o;
}

// RegistrationContext resident on one device (registration.hpp:82-89).
template <class E = DefaultErrors>
class RegistrationContext {
public:
    RegistrationContext() = default;
    explicit RegistrationContext(lk_reg_ctx* h) : h_(h) {}
    RegistrationContext(RegistrationContext&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
    RegistrationContext& operator=(RegistrationContext&& o) noexcept {
        std::swap(h_, o.h_);
        return *this;
    }
    RegistrationContext(const RegistrationContext&) = delete;
    RegistrationContext& operator=(const RegistrationContext&) = delete;
    ~RegistrationContext() { lk_reg_ctx_destroy(h_); }
    lk_reg_ctx* handle() const { return h_; }

private:
    lk_reg_ctx* h_ = nullptr;
};

// prepare_registration (registration.hpp:105-107)
template <class E = DefaultErrors, class Cloud, class Params>
RegistrationContext<E> prepare_registration(const Cloud& source, const Cloud& target, const Params& params) {
    lk_cloud s = as_lk_cloud<E>(source), t = as_lk_cloud<E>(target);
    lk_reg_params p = to_lk_params(params);
    lk_reg_ctx* h = nullptr;
    lk_status st = lk_reg_prepare(&s, &t, &p, &h);
    if (st != LK_OK) throw_status<E>(st);
    return RegistrationContext<E>(h);
}

// run_hypotheses (registration.hpp:116-118)
template <class E = DefaultErrors, class Params>
std::optional<RegistrationResult> run_hypotheses(const RegistrationContext<E>& ctx, const Params& params,
                                                 HypothesisStats* stats = nullptr) {
    lk_reg_params p = to_lk_params(params);
    lk_reg_result r{};
    lk_hyp_stats local{};
    if (!check<E>(lk_reg_run_hypotheses(ctx.handle(), &p, &r, stats ? stats : &local))) return std::nullopt;
    return from_lk(r);
}

// register_global (registration.hpp:121-124)
template <class E = DefaultErrors, class Cloud, class Params>
std::optional<RegistrationResult> register_global(const Cloud& source, const Cloud& target, const Params& params,
                                                  HypothesisStats* stats = nullptr) {
    lk_cloud s = as_lk_cloud<E>(source), t = as_lk_cloud<E>(target);
    lk_reg_params p = to_lk_params(params);
    lk_reg_result r{};
    lk_hyp_stats local{};
    if (!check<E>(lk_register_global(&s, &t, &p, &r, stats ? stats : &local))) return std::nullopt;
    return from_lk(r);
}

// evaluate_hypothesis (registration.hpp:60-63) over a device SearchGrid of
// cell `grid_cell` built from `target` (the reference passes a SearchGrid).
template <class E = DefaultErrors, class Cloud, class Params>
std::pair<double, double> evaluate_hypothesis(const Transform& T, const Cloud& source, const Cloud& target,
                                              double grid_cell, const Params& params) {
    if (source.positions.empty() || target.positions.empty())
        throw typename E::EmptyCloudT("evaluate_hypothesis: empty cloud");
    if (source.normals.empty() || target.normals.empty())
        throw typename E::MissingNormalsT("evaluate_hypothesis: both clouds need normals");
    lk_cloud s = as_lk_cloud<E>(source), t = as_lk_cloud<E>(target);
    lk_reg_params p = to_lk_params(params);
    lk_grid* g = nullptr;
    lk_status st = lk_grid_build(&t, 1, grid_cell, params.d_max, -1, &g);
    if (st != LK_OK) throw_status<E>(st);
    double rt[12];
    for (int k = 0; k < 9; ++k) rt[k] = T.R[k];
    for (int k = 0; k < 3; ++k) rt[9 + k] = T.t[k];
    lk_cand_score sc{};
    st = lk_score_candidates(g, &s, rt, 1, &p, 0, &sc, nullptr, nullptr);
    lk_grid_destroy(g);
    if (st != LK_OK) throw_status<E>(st);
    return {sc.inlier_ratio, sc.fitness};
}

// edge_info (line_process.hpp:15-16 / line_process.cpp:11-33): the 6x6
// information matrix (row-major) and pair count; throws NoCorrespondences.
struct EdgeInfo {
    double info[36];
    std::int64_t pair_count = 0;
};
template <class E = DefaultErrors, class Cloud>
EdgeInfo edge_info(const Cloud& cloud_i, const Cloud& cloud_j, const Transform& t_i, const Transform& t_j,
                   double epsilon) {
    lk_cloud ci = as_lk_cloud<E>(cloud_i), cj = as_lk_cloud<E>(cloud_j);
    double ti[12], tj[12];
    for (int k = 0; k < 9; ++k) {
        ti[k] = t_i.R[k];
        tj[k] = t_j.R[k];
    }
    for (int k = 0; k < 3; ++k) {
        ti[9 + k] = t_i.t[k];
        tj[9 + k] = t_j.t[k];
    }
    EdgeInfo out;
    lk_status st = lk_edge_info_batched(&ci, &cj, ti, tj, 1, epsilon, -1, out.info, &out.pair_count);
    if (st != LK_OK) throw_status<E>(st);
    if (out.pair_count == 0) throw typename E::NoCorrespondencesT("edge_info: no points within epsilon");
    return out;
}

// Line-process weight of a loop edge (line_process.cpp:35-46), host-only:
// f = xi^T Lambda xi with xi = twist(rel * t_j^-1 * t_i) (a residual rotation
// of pi/2 or more maps to E::Base via LK_ROTATION_TOO_LARGE), and the closed
// form weight (mu / (mu + f))^2.
template <class E = DefaultErrors>
inline double edge_residual(const Transform& t_i, const Transform& t_j, const Transform& rel, const EdgeInfo& info) {
    double a[12], b[12], r[12];
    for (int k = 0; k < 9; ++k) {
        a[k] = t_i.R[k];
        b[k] = t_j.R[k];
        r[k] = rel.R[k];
    }
    for (int k = 0; k < 3; ++k) {
        a[9 + k] = t_i.t[k];
        b[9 + k] = t_j.t[k];
        r[9 + k] = rel.t[k];
    }
    double f = 0.0;
    const lk_status st = lk_edge_residual(a, b, r, info.info, &f);
    if (st != LK_OK) throw_status<E>(st);
    return f;
}
inline double update_weight(double f, double mu) { return lk_update_weight(f, mu); }

// propose_loops (fragments.hpp:46-60, fragments.cpp:61-109) on the device.
// Generic over the caller's types: fragments[f].cloud (a Cloud as above),
// graph.poses[f] with rotation(r, c) / translation[k] (the reference's
// RigidTransform) and graph.loops[e].i / .j; params has overlap_radius and
// min_overlap (LoopParams). Throws MissingData when the pose count differs
// (fragments.cpp:64-66) and EmptyCloud for an empty fragment.
struct LoopProposal {
    int i = 0;  // later fragment
    int j = 0;  // earlier fragment
    double overlap = 0.0;
};
template <class E = DefaultErrors, class Fragments, class Graph, class LoopParamsT>
std::vector<LoopProposal> propose_loops(const Fragments& fragments, const Graph& graph, const LoopParamsT& params,
                                        int32_t device = -1) {
    const size_t n = std::size(fragments);
    if (graph.poses.size() != n) throw typename E::MissingDataT("propose_loops: one graph pose per fragment required");
    std::vector<lk_cloud> clouds;
    std::vector<double> poses;
    clouds.reserve(n);
    poses.reserve(12 * n);
    for (size_t f = 0; f < n; ++f) {
        const auto& c = fragments[f].cloud;
        lk_cloud lc{};
        lc.n = static_cast<int64_t>(c.positions.size());
        lc.xyz = lc.n ? reinterpret_cast<const double*>(c.positions.data()) : nullptr;
        clouds.push_back(lc);
        const auto& T = graph.poses[f];
        for (int r = 0; r < 3; ++r)
            for (int k = 0; k < 3; ++k) poses.push_back(T.rotation(r, k));
        for (int k = 0; k < 3; ++k) poses.push_back(T.translation[k]);
    }
    std::vector<int32_t> loops;
    for (const auto& e : graph.loops) {
        loops.push_back(static_cast<int32_t>(e.i));
        loops.push_back(static_cast<int32_t>(e.j));
    }
    lk_loop_params lp{params.overlap_radius, params.min_overlap, device, 0};
    std::vector<lk_loop_proposal> out(n * n > 0 ? n * n : 1);
    int64_t count = 0;
    const lk_status st = lk_propose_loops(clouds.data(), poses.data(), static_cast<int32_t>(n), loops.data(),
                                          static_cast<int32_t>(loops.size() / 2), &lp, out.data(),
                                          static_cast<int64_t>(out.size()), &count);
    if (st != LK_OK) throw_status<E>(st);
    std::vector<LoopProposal> props;
    props.reserve(static_cast<size_t>(count));
    for (int64_t k = 0; k < count; ++k) props.push_back({out[k].i, out[k].j, out[k].overlap});
    return props;
}

// ICP point-to-plane refinement of `init` (source -> target); DESIGN.md "ICP".
struct IcpResult {
    Transform transform;
    int iterations = 0;
    bool converged = false;
    std::int64_t correspondences = 0;
    double rmse = 0.0;
    double fitness = 0.0;
};
template <class E = DefaultErrors, class Cloud>
IcpResult icp_point_to_plane(const Cloud& source, const Cloud& target, const Transform& init,
                             double max_correspondence_distance = 0.05, int max_iterations = 30,
                             double convergence_eps = 1e-10, int32_t device = -1) {
    lk_cloud s = as_lk_cloud<E>(source), t = as_lk_cloud<E>(target);
    double T0[12];
    for (int k = 0; k < 9; ++k) T0[k] = init.R[k];
    for (int k = 0; k < 3; ++k) T0[9 + k] = init.t[k];
    lk_icp_params p{max_correspondence_distance, max_iterations, device, convergence_eps};
    lk_icp_result r{};
    lk_status st = lk_icp_point_to_plane(&s, &t, T0, &p, &r, nullptr);
    if (st != LK_OK) throw_status<E>(st);
    IcpResult o;
    for (int k = 0; k < 9; ++k) o.transform.R[k] = r.R[k];
    for (int k = 0; k < 3; ++k) o.transform.t[k] = r.t[k];
    o.iterations = r.iterations;
    o.converged = r.converged != 0;
    o.correspondences = r.correspondences;
    o.rmse = r.rmse;
    o.fitness = r.fitness;
    return o;
}

}  // namespace loopkit_b200
