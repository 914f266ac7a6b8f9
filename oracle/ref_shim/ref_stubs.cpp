// oracle/ref_shim/ref_stubs.cpp -- TEST INFRASTRUCTURE ONLY.
// Link stubs for reference functions outside the registration path whose
// sources are not compiled into oracle/_ref: the pose-graph solver
// (proj/src/pose_graph.cpp needs Eigen's LDLT over MatrixXd), bundle
// adjustment (proj/src/ba.cpp) and file I/O (proj/src/io.cpp needs
// nlohmann-json). They are referenced by line_process.cpp (the optimizer, not
// edge_info) and synth.cpp (dataset writers and landmark projection), never by
// anything oracle/_ref runs. Each throws if reached.
#include <stdexcept>
#include <string>

#include "loopkit/ba.hpp"
#include "loopkit/io.hpp"
#include "loopkit/pose_graph.hpp"

namespace loopkit {

[[noreturn]] static void out_of_scope(const char* fn) {
    throw std::logic_error(std::string("oracle/_ref: ") + fn + " is outside the compiled registration path");
}

double graph_cost(const PoseGraph&, double) { out_of_scope("graph_cost"); }
namespace detail {
bool pose_step(PoseGraph&, double, double&, double&, double&) { out_of_scope("detail::pose_step"); }
void check_connected(const PoseGraph&) { out_of_scope("detail::check_connected"); }
}  // namespace detail
std::optional<Vec2> project(const CameraIntrinsics&, const RigidTransform&, const Vec3&) { out_of_scope("project"); }
void write_ply(const std::string&, const PointCloud&, bool) { out_of_scope("write_ply"); }
void write_trajectory(const std::string&, std::span<const TimedPose>) { out_of_scope("write_trajectory"); }
void write_surfel_map(const std::string&, const std::string&, const SurfelMap&) { out_of_scope("write_surfel_map"); }
void write_ba_json(const std::string&, const BaProblem&) { out_of_scope("write_ba_json"); }

}  // namespace loopkit
