// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C ABI over the REFERENCE's own code, compiled unmodified from
// /root/reference/proj/src/{geometry,grid,preprocess,fpfh,registration,
// fragments,line_process,synth}.cpp against the committed Eigen/doctest shim
// (oracle/ref_shim/) into oracle/_ref/liblk_ref.so by oracle/Makefile.ref.
// tests/ use it to pin oracle/ (and, through committed golden files, the
// device path) to the reference's own code; bench.py's reference arm times it.
// Nothing in paper_1801_01572_b200/ links or calls it.
//
// Every entry point forwards to the reference function named in its comment;
// exceptions become the status codes of lk_oracle.h (errors.hpp:9-74).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include <omp.h>

#include "loopkit/errors.hpp"
#include "loopkit/fpfh.hpp"
#include "loopkit/fragments.hpp"
#include "loopkit/grid.hpp"
#include "loopkit/line_process.hpp"
#include "loopkit/preprocess.hpp"
#include "loopkit/reference.hpp"
#include "loopkit/registration.hpp"
#include "loopkit/rng.hpp"
#include "loopkit/synth.hpp"
#include "lk_oracle.h"
#include "support/helpers.hpp"

using namespace loopkit;

namespace {

thread_local std::string g_err;

int code_of(const std::exception& e) {
    if (dynamic_cast<const EmptyCloud*>(&e)) return OR_EMPTY_CLOUD;
    if (dynamic_cast<const TooFewPoints*>(&e)) return OR_TOO_FEW_POINTS;
    if (dynamic_cast<const MissingNormals*>(&e)) return OR_MISSING_NORMALS;
    if (dynamic_cast<const MissingData*>(&e)) return OR_MISSING_DATA;
    if (dynamic_cast<const NoCorrespondences*>(&e)) return OR_NO_CORRESPONDENCES;
    if (dynamic_cast<const DegenerateConfiguration*>(&e)) return OR_DEGENERATE;
    return OR_ERROR;
}

template <class F>
int guard(F&& fn) {
    try {
        return fn();
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

Vec3 ld3(const double* p, int64_t i) { return Vec3(p[3 * i], p[3 * i + 1], p[3 * i + 2]); }
void st3(double* p, int64_t i, const Vec3& v) {
    p[3 * i] = v.x();
    p[3 * i + 1] = v.y();
    p[3 * i + 2] = v.z();
}
PointCloud cloud_of(const double* xyz, const double* nxyz, int64_t n) {
    PointCloud c;
    c.positions.reserve(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) c.positions.push_back(ld3(xyz, i));
    if (nxyz) {
        c.normals.reserve(static_cast<std::size_t>(n));
        for (int64_t i = 0; i < n; ++i) c.normals.push_back(ld3(nxyz, i));
    }
    return c;
}
void put_cloud(const PointCloud& c, double* xyz, double* nxyz) {
    for (std::size_t i = 0; i < c.size(); ++i) {
        if (xyz) st3(xyz, static_cast<int64_t>(i), c.positions[i]);
        if (nxyz && c.has_normals()) st3(nxyz, static_cast<int64_t>(i), c.normals[i]);
    }
}
RigidTransform rigid_of(const double* R9, const double* t3) {
    RigidTransform t;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) t.rotation(r, c) = R9[3 * r + c];
    t.translation = Vec3(t3[0], t3[1], t3[2]);
    return t;
}
void put_rigid(const RigidTransform& t, double* R9, double* t3) {
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) R9[3 * r + c] = t.rotation(r, c);
    t3[0] = t.translation.x();
    t3[1] = t.translation.y();
    t3[2] = t.translation.z();
}
RegistrationParams params_of(const or_params* p) {
    RegistrationParams q;
    q.leaf = p->leaf;
    q.normal_radius = p->normal_radius;
    q.feature_radius = p->feature_radius;
    q.hypothesis_count = p->hypothesis_count;
    q.similarity_tau = p->similarity_tau;
    q.d_max = p->d_max;
    q.min_inlier_ratio = p->min_inlier_ratio;
    if (p->max_fitness >= 0.0) q.max_fitness = p->max_fitness;
    q.normal_angle_max = p->normal_angle_max;
    q.seed = p->seed;
    q.threads = p->threads;
    return q;
}
void put_result(const std::optional<RegistrationResult>& r, int64_t ns, or_result* out) {
    std::memset(out, 0, sizeof(*out));
    out->found = r.has_value() ? 1 : 0;
    out->hypothesis_index = -1;
    if (!r) return;
    put_rigid(r->transform, out->R, out->t);
    out->inlier_ratio = r->inlier_ratio;
    out->fitness = r->fitness;
    out->hypothesis_index = r->hypothesis_index;
    // ratio = inliers / Ns exactly rounded (registration.cpp:216): recover the count
    out->inliers = static_cast<int64_t>(std::llround(r->inlier_ratio * static_cast<double>(ns)));
}
void put_stats(const HypothesisStats& s, or_stats* out) {
    std::memset(out, 0, sizeof(*out));
    out->sampled = s.sampled;
    out->prerejected = s.prerejected;
    out->degenerate = s.degenerate;
    out->evaluated = s.evaluated;
    out->qualified = s.qualified;
    out->prepare_seconds = s.prepare_seconds;
    out->hypothesis_seconds = s.hypothesis_seconds;
}

struct Fixture {
    std::vector<PointCloud> clouds;
    RigidTransform truth;
    double scalar = 0.0;
};

void* fixture_guard(int* status, const std::function<Fixture()>& fn) {
    try {
        auto* f = new Fixture(fn());
        *status = OR_OK;
        return f;
    } catch (const std::exception& e) {
        g_err = e.what();
        *status = code_of(e);
        return nullptr;
    }
}

// synth.cpp:315-322 orbit_pose (file-local there; restated with the
// reference's SynthConfig defaults and its public look_at)
RigidTransform orbit_pose(int frames, int frame) {
    SynthConfig c;
    c.frames = frames;
    double theta = 2.0 * M_PI * c.orbits * static_cast<double>(frame) / static_cast<double>(c.frames);
    double radius = c.orbit_radius + 0.08 * std::cos(3.0 * theta);
    Vec3 eye(radius * std::sin(theta), -0.1 + 0.2 * std::sin(2.0 * theta), radius * std::cos(theta));
    return look_at(eye, Vec3(0.0, 0.45, 0.0));
}

// synth.cpp:571-583 random_transform (file-local there)
RigidTransform synth_random_transform(RngStream& rng, double max_angle, double max_trans) {
    Vec3 axis(rng.next_gaussian(), rng.next_gaussian(), rng.next_gaussian());
    if (axis.norm() < 1e-9) axis = Vec3::UnitZ();
    axis.normalize();
    double angle = max_angle * rng.next_double();
    Vec3 dir(rng.next_gaussian(), rng.next_gaussian(), rng.next_gaussian());
    if (dir.norm() < 1e-9) dir = Vec3::UnitX();
    dir.normalize();
    RigidTransform t;
    t.rotation = Eigen::AngleAxisd(angle, axis).toRotationMatrix();
    t.translation = dir * (max_trans * rng.next_double());
    return t;
}

void append(PointCloud& dst, const PointCloud& src) {
    dst.positions.insert(dst.positions.end(), src.positions.begin(), src.positions.end());
    dst.normals.insert(dst.normals.end(), src.normals.begin(), src.normals.end());
}

}  // namespace

extern "C" {

const char* rf_last_error(void) { return g_err.c_str(); }
int rf_max_threads(void) { return omp_get_max_threads(); }

// ---------------------------------------------------------------- fixtures
// synth.cpp:587-623 synth_registration_pair
void* rf_registration_pair(uint64_t seed, double leaf, int* status) {
    return fixture_guard(status, [&] {
        RegistrationPair p = synth_registration_pair(seed, leaf);
        Fixture f;
        f.clouds = {p.source, p.target};
        f.truth = p.truth;
        f.scalar = p.overlap;
        return f;
    });
}
// synth.cpp:625-653 synth_negative_pair
void* rf_negative_pair(uint64_t seed, double leaf, int* status) {
    return fixture_guard(status, [&] {
        RegistrationPair p = synth_negative_pair(seed, leaf);
        Fixture f;
        f.clouds = {p.source, p.target};
        return f;
    });
}
// Config B1/B2: make_room_scene + render_view of two orbit frames
// (frame i rendered with RngStream(seed, 0x3E0 + i), synth.cpp:340-367)
void* rf_frame_pair(uint64_t seed, int boxes, int width, int height, double fx, double fy, double cx, double cy,
                    int stride, double noise, int frames, int frame_a, int frame_b, int* status) {
    return fixture_guard(status, [&] {
        TriangleScene scene = make_room_scene(seed, boxes);
        CameraIntrinsics k{fx, fy, cx, cy, width, height};
        RigidTransform pa = orbit_pose(frames, frame_a), pb = orbit_pose(frames, frame_b);
        RngStream ra(seed, 0x3E0 + static_cast<uint64_t>(frame_a));
        RngStream rb(seed, 0x3E0 + static_cast<uint64_t>(frame_b));
        Fixture f;
        f.clouds.push_back(render_view(scene, pa, k, stride, noise, ra));
        f.clouds.push_back(render_view(scene, pb, k, stride, noise, rb));
        f.truth = compose(inverse(pb), pa);
        return f;
    });
}
// Config D: two submaps, each the union of `views` renders (no downsample)
void* rf_submap_pair(uint64_t seed, int boxes, int views, int width, int height, int stride, double noise,
                     int frames, int a0, int b0, int step, int* status) {
    return fixture_guard(status, [&] {
        TriangleScene scene = make_room_scene(seed, boxes);
        CameraIntrinsics k{525.0, 525.0, 319.5 * width / 640.0, 239.5 * height / 480.0, width, height};
        auto submap = [&](int f0) {
            PointCloud world;
            for (int v = 0; v < views; ++v) {
                const int fr = f0 + step * v;
                RigidTransform pose = orbit_pose(frames, fr);
                RngStream r(seed, 0xD10 + static_cast<uint64_t>(fr));
                append(world, transformed(render_view(scene, pose, k, stride, noise, r), pose));
            }
            return world;
        };
        PointCloud a = submap(a0), b = submap(b0);
        RngStream rng(seed, 0xD00);
        RigidTransform displace = synth_random_transform(rng, M_PI / 3.0, 1.0);
        Fixture f;
        f.clouds.push_back(transformed(a, displace));
        f.clouds.push_back(std::move(b));
        f.truth = inverse(displace);
        return f;
    });
}
// Config A: Q = sample_surface(make_scatter_scene(seed)), P = T^-1 (Q + noise)
void* rf_surface_pair(uint64_t seed, double density, double noise, int* status) {
    return fixture_guard(status, [&] {
        TriangleScene scene = make_scatter_scene(seed);
        PointCloud q = sample_surface(scene, density, seed);
        RngStream trng(seed, 0xA110);
        RigidTransform truth = synth_random_transform(trng, M_PI / 3.0, 1.0);
        RigidTransform inv = inverse(truth);
        RngStream nrng(seed, 0xA11CE);
        PointCloud p;
        for (std::size_t i = 0; i < q.size(); ++i) {
            Vec3 noisy = q.positions[i];
            noisy.x() += noise * nrng.next_gaussian();
            noisy.y() += noise * nrng.next_gaussian();
            noisy.z() += noise * nrng.next_gaussian();
            p.positions.push_back(inv * noisy);
            p.normals.push_back(inv.rotation * q.normals[i]);
        }
        Fixture f;
        f.clouds.push_back(std::move(p));
        f.clouds.push_back(std::move(q));
        f.truth = truth;
        return f;
    });
}
// proj/tests/support/helpers.hpp:16-31 testing::random_cloud
void* rf_random_cloud(uint64_t seed, uint64_t stream, int n, double lo, double hi, int with_normals, int* status) {
    return fixture_guard(status, [&] {
        RngStream rng(seed, stream);
        Fixture f;
        f.clouds.push_back(testing::random_cloud(n, rng, lo, hi, with_normals != 0));
        return f;
    });
}
int64_t rf_count(void* h, int which) {
    auto* f = static_cast<Fixture*>(h);
    return which < static_cast<int>(f->clouds.size()) ? static_cast<int64_t>(f->clouds[which].size()) : -1;
}
int rf_has_normals(void* h, int which) { return static_cast<Fixture*>(h)->clouds[which].has_normals() ? 1 : 0; }
void rf_get(void* h, int which, double* xyz, double* nxyz) { put_cloud(static_cast<Fixture*>(h)->clouds[which], xyz, nxyz); }
void rf_truth(void* h, double* R9, double* t3, double* scalar) {
    auto* f = static_cast<Fixture*>(h);
    put_rigid(f->truth, R9, t3);
    if (scalar) *scalar = f->scalar;
}
void rf_free(void* h) { delete static_cast<Fixture*>(h); }
// helpers.hpp:34-46 testing::random_transform
void rf_random_transform(uint64_t seed, uint64_t stream, int skip_draws, double max_angle, double max_trans,
                         double* R9, double* t3) {
    RngStream rng(seed, stream);
    for (int i = 0; i < skip_draws; ++i) rng.next_u64();
    put_rigid(testing::random_transform(rng, max_angle, max_trans), R9, t3);
}

// ---------------------------------------------------------------- geometry
void rf_transform_from_twist(const double* xi6, double* R9, double* t3) {  // geometry.cpp:42-52
    put_rigid(transform_from_twist(Twist{xi6[0], xi6[1], xi6[2], xi6[3], xi6[4], xi6[5]}), R9, t3);
}
void rf_compose(const double* Ra, const double* ta, const double* Rb, const double* tb, double* R9, double* t3) {
    put_rigid(compose(rigid_of(Ra, ta), rigid_of(Rb, tb)), R9, t3);  // geometry.cpp:8-11
}
void rf_inverse(const double* Ra, const double* ta, double* R9, double* t3) {
    put_rigid(inverse(rigid_of(Ra, ta)), R9, t3);  // geometry.cpp:13-16
}
void rf_apply(const double* R9, const double* t3, const double* xyz, int64_t n, double* out) {
    RigidTransform T = rigid_of(R9, t3);  // geometry.hpp:26
    for (int64_t i = 0; i < n; ++i) st3(out, i, T * ld3(xyz, i));
}
int rf_kabsch(const double* src, const double* dst, int64_t n, double* R9, double* t3) {  // geometry.cpp:62-91
    return guard([&] {
        std::vector<Vec3> s, d;
        for (int64_t i = 0; i < n; ++i) {
            s.push_back(ld3(src, i));
            d.push_back(ld3(dst, i));
        }
        put_rigid(kabsch(s, d), R9, t3);
        return OR_OK;
    });
}
void rf_svd3(const double* A9, double* U9, double* S3, double* V9) {  // Eigen::JacobiSVD (shim)
    Mat3 a;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) a(r, c) = A9[3 * r + c];
    Eigen::JacobiSVD<Mat3> svd(a, Eigen::ComputeFullU | Eigen::ComputeFullV);
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            U9[3 * r + c] = svd.matrixU()(r, c);
            V9[3 * r + c] = svd.matrixV()(r, c);
        }
    for (int i = 0; i < 3; ++i) S3[i] = svd.singularValues()(i);
}

// ---------------------------------------------------------------- prepare pieces
int rf_voxel_downsample(const double* xyz, const double* nxyz, int64_t n, double leaf, double* out_xyz,
                        double* out_n, int64_t* out_count) {  // preprocess.cpp:14-59
    return guard([&] {
        PointCloud d = voxel_downsample(cloud_of(xyz, nxyz, n), leaf);
        *out_count = static_cast<int64_t>(d.size());
        put_cloud(d, out_xyz, out_n);
        return OR_OK;
    });
}
int rf_estimate_normals(const double* xyz, int64_t n, double radius, const double* vp, int32_t threads,
                        double* out) {  // preprocess.cpp:61-96
    return guard([&] {
        PointCloud c = estimate_normals(cloud_of(xyz, nullptr, n), radius, ld3(vp, 0), threads);
        put_cloud(c, nullptr, out);
        return OR_OK;
    });
}
int rf_compute_fpfh(const double* xyz, const double* nxyz, int64_t n, double radius, int32_t threads,
                    float* out) {  // fpfh.cpp:57-141
    return guard([&] {
        auto f = compute_fpfh(cloud_of(xyz, nxyz, n), radius, threads);
        for (std::size_t i = 0; i < f.size(); ++i) std::memcpy(out + i * kFpfhDim, f[i].bins.data(), sizeof(float) * kFpfhDim);
        return OR_OK;
    });
}
static std::vector<FpfhFeature> features_of(const float* f, int64_t n) {
    std::vector<FpfhFeature> v(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) std::memcpy(v[static_cast<std::size_t>(i)].bins.data(), f + i * kFpfhDim, sizeof(float) * kFpfhDim);
    return v;
}
// grid.cpp:176-213 (the binary's float GEMV matcher); exhaustive != 0 selects
// reference.hpp:56-76 (the FP64 exhaustive matcher the tests compare against)
int rf_feature_nn_cache(const float* sf, int64_t ns, const float* tf, int64_t nt, int32_t threads, int32_t exhaustive,
                        int32_t* out) {
    return guard([&] {
        auto s = features_of(sf, ns), t = features_of(tf, nt);
        std::vector<int> c = exhaustive ? reference::feature_nn_cache(s, t) : feature_nn_cache(s, t, threads);
        for (std::size_t i = 0; i < c.size(); ++i) out[i] = c[i];
        return OR_OK;
    });
}

// ---------------------------------------------------------------- registration
// registration.cpp:223-251 prepare_registration
void* rf_prepare(const double* sxyz, const double* sn, int64_t ns, const double* txyz, const double* tn, int64_t nt,
                 const or_params* p, int* status) {
    try {
        auto* ctx = new RegistrationContext(prepare_registration(cloud_of(sxyz, sn, ns), cloud_of(txyz, tn, nt), params_of(p)));
        *status = OR_OK;
        return ctx;
    } catch (const std::exception& e) {
        g_err = e.what();
        *status = code_of(e);
        return nullptr;
    }
}
// a RegistrationContext from already-prepared clouds and cache (the eval grid
// built by the reference's build_eval_grid, registration.cpp:80-148)
void* rf_ctx_from_prepared(const double* sxyz, const double* sn, int64_t ns, const double* txyz, const double* tn,
                           int64_t nt, const int32_t* cache, double d_max, int* status) {
    try {
        auto* ctx = new RegistrationContext();
        ctx->source = cloud_of(sxyz, sn, ns);
        ctx->target = cloud_of(txyz, tn, nt);
        ctx->cache.assign(cache, cache + ns);
        ctx->eval = build_eval_grid(ctx->target, d_max);
        *status = OR_OK;
        return ctx;
    } catch (const std::exception& e) {
        g_err = e.what();
        *status = code_of(e);
        return nullptr;
    }
}
void rf_ctx_sizes(void* h, int64_t* ns, int64_t* nt) {
    auto* c = static_cast<RegistrationContext*>(h);
    *ns = static_cast<int64_t>(c->source.size());
    *nt = static_cast<int64_t>(c->target.size());
}
void rf_ctx_get(void* h, double* sxyz, double* sn, double* txyz, double* tn, int32_t* cache, float* sfeat,
                float* tfeat) {
    auto* c = static_cast<RegistrationContext*>(h);
    put_cloud(c->source, sxyz, sn);
    put_cloud(c->target, txyz, tn);
    if (cache)
        for (std::size_t i = 0; i < c->cache.size(); ++i) cache[i] = c->cache[i];
    if (sfeat)
        for (std::size_t i = 0; i < c->source_features.size(); ++i)
            std::memcpy(sfeat + i * kFpfhDim, c->source_features[i].bins.data(), sizeof(float) * kFpfhDim);
    if (tfeat)
        for (std::size_t i = 0; i < c->target_features.size(); ++i)
            std::memcpy(tfeat + i * kFpfhDim, c->target_features[i].bins.data(), sizeof(float) * kFpfhDim);
}
void rf_ctx_eval_dims(void* h, double* origin3, double* cell, int32_t* dims3, int64_t* ncells) {
    const EvalGrid& g = static_cast<RegistrationContext*>(h)->eval;
    st3(origin3, 0, g.origin);
    *cell = g.cell;
    dims3[0] = g.nx;
    dims3[1] = g.ny;
    dims3[2] = g.nz;
    *ncells = static_cast<int64_t>(g.near_occupied.size());
}
void rf_ctx_eval_arrays(void* h, int32_t* start, int32_t* index, double* slot_pos, double* slot_nrm, uint8_t* near) {
    const EvalGrid& g = static_cast<RegistrationContext*>(h)->eval;
    std::memcpy(start, g.start.data(), g.start.size() * sizeof(int32_t));
    std::memcpy(index, g.index.data(), g.index.size() * sizeof(int32_t));
    for (std::size_t i = 0; i < g.slot_position.size(); ++i) {
        st3(slot_pos, static_cast<int64_t>(i), g.slot_position[i]);
        st3(slot_nrm, static_cast<int64_t>(i), g.slot_normal[i]);
    }
    std::memcpy(near, g.near_occupied.data(), g.near_occupied.size());
}
void rf_ctx_free(void* h) { delete static_cast<RegistrationContext*>(h); }
// registration.cpp:253-332 run_hypotheses
int rf_run_hypotheses(void* h, const or_params* p, or_result* res, or_stats* st) {
    return guard([&] {
        auto* c = static_cast<RegistrationContext*>(h);
        HypothesisStats s;
        auto r = run_hypotheses(*c, params_of(p), &s);
        put_result(r, static_cast<int64_t>(c->source.size()), res);
        if (st) put_stats(s, st);
        return r ? OR_OK : OR_NO_ALIGNMENT;
    });
}
// registration.cpp:336-343 register_global
int rf_register_global(const double* sxyz, const double* sn, int64_t ns, const double* txyz, const double* tn,
                       int64_t nt, const or_params* p, or_result* res, or_stats* st) {
    return guard([&] {
        HypothesisStats s;
        RegistrationParams q = params_of(p);
        // the inlier count needs Ns after downsampling: prepare + run, exactly as register_global does
        double t0 = omp_get_wtime();
        RegistrationContext ctx = prepare_registration(cloud_of(sxyz, sn, ns), cloud_of(txyz, tn, nt), q);
        s.prepare_seconds = omp_get_wtime() - t0;
        auto r = run_hypotheses(ctx, q, &s);
        put_result(r, static_cast<int64_t>(ctx.source.size()), res);
        if (st) put_stats(s, st);
        return r ? OR_OK : OR_NO_ALIGNMENT;
    });
}
// registration.cpp:53-78 evaluate_hypothesis over build_grid(target, grid_cell)
int rf_evaluate_hypothesis(const double* R9, const double* t3, const double* sxyz, const double* sn, int64_t ns,
                           const double* txyz, const double* tn, int64_t nt, double grid_cell, const or_params* p,
                           double* ratio, double* fitness) {
    return guard([&] {
        PointCloud s = cloud_of(sxyz, sn, ns), t = cloud_of(txyz, tn, nt);
        SearchGrid g = build_grid(t, grid_cell);
        auto [r, f] = evaluate_hypothesis(rigid_of(R9, t3), s, t, g, params_of(p));
        *ratio = r;
        *fitness = f;
        return OR_OK;
    });
}
// grid.cpp:116-150 nn_within over build_grid(cloud, cell)
int rf_nn_within_batch(const double* xyz, int64_t n, double cell, const double* q, int64_t nq, double d_max,
                       int32_t* idx, double* dist) {
    return guard([&] {
        SearchGrid g = build_grid(cloud_of(xyz, nullptr, n), cell);
        for (int64_t i = 0; i < nq; ++i) {
            auto r = nn_within(g, ld3(q, i), d_max);
            idx[i] = r ? r->index : -1;
            dist[i] = r ? r->distance : 0.0;
        }
        return OR_OK;
    });
}

// ---------------------------------------------------------------- verification
// line_process.cpp:11-33 edge_info
int rf_edge_info(const double* ci, int64_t ni, const double* cj, int64_t nj, const double* Ri9, const double* ti3,
                 const double* Rj9, const double* tj3, double epsilon, double* info36, int64_t* pair_count) {
    return guard([&] {
        EdgeInfo e = edge_info(cloud_of(ci, nullptr, ni), cloud_of(cj, nullptr, nj), rigid_of(Ri9, ti3),
                               rigid_of(Rj9, tj3), epsilon);
        for (int r = 0; r < 6; ++r)
            for (int c = 0; c < 6; ++c) info36[6 * r + c] = e.info(r, c);
        *pair_count = e.pair_count;
        return OR_OK;
    });
}
// line_process.cpp:35-40 edge_residual and :42-46 update_weight
double rf_edge_residual(const double* Ri, const double* ti, const double* Rj, const double* tj, const double* Rr,
                        const double* tr, const double* info36, int64_t pair_count, int* status) {
    double out = 0.0;
    *status = guard([&] {
        EdgeInfo e;
        for (int r = 0; r < 6; ++r)
            for (int c = 0; c < 6; ++c) e.info(r, c) = info36[6 * r + c];
        e.pair_count = pair_count;
        out = edge_residual(rigid_of(Ri, ti), rigid_of(Rj, tj), rigid_of(Rr, tr), e);
        return OR_OK;
    });
    return out;
}
double rf_update_weight(double f, double mu) { return update_weight(f, mu); }

// fragments.cpp:61-109 propose_loops. clouds: concatenated xyz of n fragments
// (counts[f] points each), poses: n x (R9, t3); loops: n_loops x (i, j).
// Writes up to cap proposals (i, j, overlap); returns the proposal count or < 0.
int64_t rf_propose_loops(const double* xyz, const int64_t* counts, int32_t n, const double* R9s, const double* t3s,
                         const int32_t* loops, int32_t n_loops, double overlap_radius, double min_overlap,
                         int32_t* out_i, int32_t* out_j, double* out_overlap, int64_t cap) {
    int64_t count = -1;
    int st = guard([&] {
        std::vector<Fragment> frags(static_cast<std::size_t>(n));
        PoseGraph graph;
        int64_t off = 0;
        for (int f = 0; f < n; ++f) {
            frags[static_cast<std::size_t>(f)].id = f;
            frags[static_cast<std::size_t>(f)].cloud = cloud_of(xyz + 3 * off, nullptr, counts[f]);
            off += counts[f];
            graph.poses.push_back(rigid_of(R9s + 9 * f, t3s + 3 * f));
        }
        for (int e = 0; e < n_loops; ++e) {
            LoopEdge le;
            le.i = loops[2 * e];
            le.j = loops[2 * e + 1];
            graph.loops.push_back(le);
        }
        LoopParams lp;
        lp.overlap_radius = overlap_radius;
        lp.min_overlap = min_overlap;
        auto props = propose_loops(frags, graph, lp);
        count = static_cast<int64_t>(props.size());
        for (int64_t k = 0; k < count && k < cap; ++k) {
            out_i[k] = props[static_cast<std::size_t>(k)].i;
            out_j[k] = props[static_cast<std::size_t>(k)].j;
            out_overlap[k] = props[static_cast<std::size_t>(k)].overlap;
        }
        return OR_OK;
    });
    return st == OR_OK ? count : -static_cast<int64_t>(st);
}

}  // extern "C"
