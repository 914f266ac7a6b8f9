// lk_synth.cpp -- synthetic fixture generators (host C++), used to build the
// bench and test inputs. Restates the reference's generators so the
// reference's own seeded fixtures can be reproduced:
//   make_room_scene / make_scatter_scene   proj/src/synth.cpp:80-179
//   raycast / look_at / render_view        proj/src/synth.cpp:51-76,185-226
//   sample_surface                         proj/src/synth.cpp:248-268
//   orbit_pose                             proj/src/synth.cpp:315-322
//   synth_registration_pair / negative     proj/src/synth.cpp:548-653
//   testing::random_cloud/random_transform proj/tests/support/helpers.hpp:16-46
// This is input generation, not the measured path.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include <omp.h>

#include "../../include/loopkit_b200.h"
#include "lk_prepare_host.hpp"
#include "lk_acos_cr.hpp"

namespace lk {
namespace {

using Tri = std::array<Vec3, 3>;

// The reference is built with GCC, which evaluates constructor arguments
// right to left: Vec3(f(), g(), h()) calls h, g, f. Fixtures that construct
// a Vec3 from three RNG draws therefore fill z, then y, then x.
template <class F>
Vec3 vec3_rtl(F&& draw) {
    Vec3 v;
    v.z = draw(2);
    v.y = draw(1);
    v.x = draw(0);
    return v;
}
struct Scene {
    std::vector<Tri> tris;
};

Vec3 tri_normal(const Tri& t) {
    Vec3 n = cross(t[1] - t[0], t[2] - t[0]);
    double len = norm(n);
    return len > 1e-15 ? n / len : Vec3{0, 0, 1};
}
void add_quad(Scene& s, Vec3 a, Vec3 b, Vec3 c, Vec3 d) {
    s.tris.push_back({a, b, c});
    s.tris.push_back({a, c, d});
}
void add_box(Scene& s, Vec3 center, Vec3 half, const Mat3& r, bool open_bottom) {
    auto corner = [&](int sx, int sy, int sz) {
        Vec3 local{sx * half.x, sy * half.y, sz * half.z};
        return center + r * local;
    };
    Vec3 c_mmm = corner(-1, -1, -1), c_pmm = corner(1, -1, -1), c_mpm = corner(-1, 1, -1), c_ppm = corner(1, 1, -1),
         c_mmp = corner(-1, -1, 1), c_pmp = corner(1, -1, 1), c_mpp = corner(-1, 1, 1), c_ppp = corner(1, 1, 1);
    add_quad(s, c_mmm, c_pmm, c_ppm, c_mpm);
    add_quad(s, c_mmp, c_pmp, c_ppp, c_mpp);
    add_quad(s, c_mmm, c_mpm, c_mpp, c_mmp);
    add_quad(s, c_pmm, c_ppm, c_ppp, c_pmp);
    add_quad(s, c_mmm, c_pmm, c_pmp, c_mmp);
    if (!open_bottom) add_quad(s, c_mpm, c_ppm, c_ppp, c_mpp);
}

// proj/src/synth.cpp:51-76 (Moller-Trumbore, nearest hit)
std::optional<std::pair<double, size_t>> raycast_hit(const Scene& scene, Vec3 origin, Vec3 dir) {
    double best = std::numeric_limits<double>::infinity();
    size_t best_tri = 0;
    for (size_t i = 0; i < scene.tris.size(); ++i) {
        const Tri& t = scene.tris[i];
        Vec3 e1 = t[1] - t[0], e2 = t[2] - t[0];
        Vec3 p = cross(dir, e2);
        double det = dot(e1, p);
        if (std::abs(det) < 1e-12) continue;
        double inv = 1.0 / det;
        Vec3 s = origin - t[0];
        double u = dot(s, p) * inv;
        if (u < 0.0 || u > 1.0) continue;
        Vec3 q = cross(s, e1);
        double v = dot(dir, q) * inv;
        if (v < 0.0 || u + v > 1.0) continue;
        double dist = dot(e2, q) * inv;
        if (dist > 1e-9 && dist < best) {
            best = dist;
            best_tri = i;
        }
    }
    if (!std::isfinite(best)) return std::nullopt;
    return std::make_pair(best, best_tri);
}

Scene make_room_scene(uint64_t seed, int boxes) {
    RngStream rng(seed, 0x500);
    Scene s;
    const double hx = 2.3, hz = 1.8, y_floor = 1.0, y_top = -1.0;
    add_quad(s, {-hx, y_floor, -hz}, {hx, y_floor, -hz}, {hx, y_floor, hz}, {-hx, y_floor, hz});
    add_quad(s, {-hx, y_top, -hz}, {hx, y_top, -hz}, {hx, y_floor, -hz}, {-hx, y_floor, -hz});
    add_quad(s, {-hx, y_top, hz}, {hx, y_top, hz}, {hx, y_floor, hz}, {-hx, y_floor, hz});
    add_quad(s, {-hx, y_top, -hz}, {-hx, y_top, hz}, {-hx, y_floor, hz}, {-hx, y_floor, -hz});
    add_quad(s, {hx, y_top, -hz}, {hx, y_top, hz}, {hx, y_floor, hz}, {hx, y_floor, -hz});
    add_box(s, {1.9, y_floor - 0.85, 1.4}, {0.28, 0.85, 0.28}, Mat3{}, true);
    add_box(s, {-2.0, y_floor - 0.25, -0.4}, {0.22, 0.25, 0.8}, Mat3{}, true);
    if (boxes <= 0) boxes = 4 + static_cast<int>(rng.next_bounded(4));
    for (int b = 0; b < boxes; ++b) {
        Vec3 half = vec3_rtl([&](int a) { return a == 1 ? 0.15 + 0.3 * rng.next_double() : 0.15 + 0.25 * rng.next_double(); });
        double radius = b % 2 == 0 ? 0.55 * rng.next_double() : 1.55 + 0.25 * rng.next_double();
        double angle = 2.0 * M_PI * rng.next_double();
        Vec3 center{radius * std::sin(angle), y_floor - half.y, radius * std::cos(angle)};
        double reach = std::hypot(half.x, half.z) + 0.02;
        center.x = std::clamp(center.x, -hx + reach, hx - reach);
        center.z = std::clamp(center.z, -hz + reach, hz - reach);
        double yaw = 2.0 * M_PI * rng.next_double();
        Mat3 r = angle_axis(yaw, Vec3{0, 1, 0});
        add_box(s, center, half, r, true);
    }
    return s;
}

void add_icosphere(Scene& s, Vec3 center, double radius) {
    const double g = (1.0 + std::sqrt(5.0)) / 2.0;
    std::array<Vec3, 12> v = {Vec3{-1, g, 0}, Vec3{1, g, 0},   Vec3{-1, -g, 0}, Vec3{1, -g, 0},
                              Vec3{0, -1, g}, Vec3{0, 1, g},   Vec3{0, -1, -g}, Vec3{0, 1, -g},
                              Vec3{g, 0, -1}, Vec3{g, 0, 1},   Vec3{-g, 0, -1}, Vec3{-g, 0, 1}};
    for (Vec3& p : v) p = normalized(p);
    static constexpr int faces[20][3] = {{0, 11, 5}, {0, 5, 1},  {0, 1, 7},   {0, 7, 10}, {0, 10, 11},
                                         {1, 5, 9},  {5, 11, 4}, {11, 10, 2}, {10, 7, 6}, {7, 1, 8},
                                         {3, 9, 4},  {3, 4, 2},  {3, 2, 6},   {3, 6, 8},  {3, 8, 9},
                                         {4, 9, 5},  {2, 4, 11}, {6, 2, 10},  {8, 6, 7},  {9, 8, 1}};
    for (const auto& f : faces) {
        Vec3 a = v[f[0]], b = v[f[1]], c = v[f[2]];
        Vec3 ab = normalized((a + b) * 0.5), bc = normalized((b + c) * 0.5), ca = normalized((c + a) * 0.5);
        for (const Tri& t : {Tri{a, ab, ca}, Tri{ab, b, bc}, Tri{ca, bc, c}, Tri{ab, bc, ca}})
            s.tris.push_back({center + radius * t[0], center + radius * t[1], center + radius * t[2]});
    }
}

Scene make_scatter_scene(uint64_t seed) {
    RngStream rng(seed, 0x5CA);
    Scene s;
    for (int b = 0; b < 36; ++b) {
        Vec3 half = vec3_rtl([&](int) { return 0.10 + 0.30 * rng.next_double(); });
        double hr = 1.45 * std::sqrt(rng.next_double());
        double ha = 2.0 * M_PI * rng.next_double();
        Vec3 center;
        center.x = hr * std::sin(ha);
        center.y = 1.6 * (rng.next_double() - 0.5);
        center.z = hr * std::cos(ha);
        Vec3 axis = vec3_rtl([&](int) { return rng.next_gaussian(); });
        if (norm(axis) < 1e-9) axis = Vec3{0, 0, 1};
        axis = normalized(axis);
        double angle = 2.0 * M_PI * rng.next_double();
        Mat3 shear;
        shear.m[0][1] = 0.9 * (rng.next_double() - 0.5);
        shear.m[0][2] = 0.9 * (rng.next_double() - 0.5);
        shear.m[1][2] = 0.9 * (rng.next_double() - 0.5);
        Mat3 m = angle_axis(angle, axis) * shear;
        add_box(s, center, half, m, false);
    }
    for (int b = 0; b < 12; ++b) {
        double radius = 0.14 + 0.24 * rng.next_double();
        double hr = 1.45 * std::sqrt(rng.next_double());
        double ha = 2.0 * M_PI * rng.next_double();
        Vec3 center;
        center.x = hr * std::sin(ha);
        center.y = 1.6 * (rng.next_double() - 0.5);
        center.z = hr * std::cos(ha);
        add_icosphere(s, center, radius);
    }
    return s;
}

// proj/src/synth.cpp:185-203
Rigid look_at(Vec3 eye, Vec3 target) {
    Vec3 z = target - eye;
    double len = norm(z);
    if (len < 1e-12) throw Status(LK_DEGENERATE, "look_at: eye equals target");
    z = z / len;
    Vec3 down{0, 1, 0};
    Vec3 x = cross(down, z);
    if (norm(x) < 1e-9) x = Vec3{1, 0, 0};
    x = normalized(x);
    Vec3 y = cross(z, x);
    Rigid t;
    for (int r = 0; r < 3; ++r) {
        t.R.m[r][0] = x[r];
        t.R.m[r][1] = y[r];
        t.R.m[r][2] = z[r];
    }
    t.t = eye;
    return t;
}

struct Intrinsics {
    double fx, fy, cx, cy;
    int width, height;
};

// proj/src/synth.cpp:205-226. Rays are cast in parallel; the noise draws are
// then applied in pixel order so the RNG sequence matches the serial loop.
Cloud render_view(const Scene& scene, const Rigid& cam_to_world, const Intrinsics& k, int stride, double noise_sigma,
                  RngStream& rng) {
    std::vector<std::pair<int, int>> pix;
    for (int v = stride / 2; v < k.height; v += stride)
        for (int u = stride / 2; u < k.width; u += stride) pix.emplace_back(u, v);
    const int64_t np = static_cast<int64_t>(pix.size());
    std::vector<double> depth(np, -1.0);
    std::vector<size_t> tri(np, 0);
    std::vector<Vec3> dcam(np);
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < np; ++i) {
        int u = pix[i].first, v = pix[i].second;
        Vec3 dir_cam{(u + 0.5 - k.cx) / k.fx, (v + 0.5 - k.cy) / k.fy, 1.0};
        dir_cam = normalized(dir_cam);
        dcam[i] = dir_cam;
        Vec3 dir_world = cam_to_world.R * dir_cam;
        auto hit = raycast_hit(scene, cam_to_world.t, dir_world);
        if (!hit) continue;
        depth[i] = hit->first;
        tri[i] = hit->second;
    }
    Cloud cloud;
    for (int64_t i = 0; i < np; ++i) {
        if (depth[i] < 0.0) continue;
        double d = depth[i];
        if (noise_sigma > 0.0) d += noise_sigma * rng.next_gaussian();
        if (d <= 1e-6) continue;
        cloud.pos.push_back(dcam[i] * d);
        Vec3 dir_world = cam_to_world.R * dcam[i];
        Vec3 n = tri_normal(scene.tris[tri[i]]);
        if (dot(n, dir_world) > 0.0) n = -n;
        cloud.nrm.push_back(transpose_mul(cam_to_world.R, n));
    }
    return cloud;
}

// proj/src/synth.cpp:248-268
Cloud sample_surface(const Scene& scene, double density, uint64_t seed) {
    RngStream rng(seed, 0x5A9);
    Cloud cloud;
    for (const Tri& t : scene.tris) {
        double area = 0.5 * norm(cross(t[1] - t[0], t[2] - t[0]));
        double want = area * density;
        int count = static_cast<int>(want);
        if (rng.next_double() < want - count) count += 1;
        Vec3 n = tri_normal(t);
        for (int i = 0; i < count; ++i) {
            double a = rng.next_double(), b = rng.next_double();
            if (a + b > 1.0) {
                a = 1.0 - a;
                b = 1.0 - b;
            }
            cloud.pos.push_back(t[0] + a * (t[1] - t[0]) + b * (t[2] - t[0]));
            cloud.nrm.push_back(n);
        }
    }
    return cloud;
}

// proj/src/synth.cpp:315-322 (SynthConfig defaults: orbit_radius 1.2, orbits 1)
Rigid orbit_pose(int frames, int frame, double orbit_radius = 1.2, double orbits = 1.0) {
    double theta = 2.0 * M_PI * orbits * static_cast<double>(frame) / static_cast<double>(frames);
    double radius = orbit_radius + 0.08 * std::cos(3.0 * theta);
    Vec3 eye{radius * std::sin(theta), -0.1 + 0.2 * std::sin(2.0 * theta), radius * std::cos(theta)};
    return look_at(eye, Vec3{0.0, 0.45, 0.0});
}

void append(Cloud& dst, const Cloud& src) {
    dst.pos.insert(dst.pos.end(), src.pos.begin(), src.pos.end());
    dst.nrm.insert(dst.nrm.end(), src.nrm.begin(), src.nrm.end());
}

// proj/src/synth.cpp:548-569
Cloud fragment_union(const Scene& scene, const Intrinsics& k, double theta0, double spacing, double noise,
                     RngStream& rng, double orbit_radius, Vec3 target, double leaf) {
    int stride = leaf < 0.04 ? 3 : 2;
    Cloud world;
    for (int view = 0; view < 3; ++view) {
        double theta = theta0 + spacing * view;
        Vec3 eye{orbit_radius * std::sin(theta), -0.1 + 0.15 * std::sin(2.0 * theta), orbit_radius * std::cos(theta)};
        Rigid pose = look_at(eye, target);
        Cloud local = render_view(scene, pose, k, stride, noise, rng);
        append(world, transformed(local, pose));
    }
    return voxel_downsample(world, leaf);
}

void recenter(Cloud& c, Vec3 ctr) {
    for (Vec3& p : c.pos) p = p - ctr;
}

// proj/src/synth.cpp:575-590 (the synth.cpp variant, not the test helper)
Rigid synth_random_transform(RngStream& rng, double max_angle, double max_trans) {
    Vec3 axis = vec3_rtl([&](int) { return rng.next_gaussian(); });
    if (norm(axis) < 1e-9) axis = Vec3{0, 0, 1};
    axis = normalized(axis);
    double angle = max_angle * rng.next_double();
    Vec3 dir = vec3_rtl([&](int) { return rng.next_gaussian(); });
    if (norm(dir) < 1e-9) dir = Vec3{1, 0, 0};
    dir = normalized(dir);
    Rigid t;
    t.R = angle_axis(angle, axis);
    t.t = dir * (max_trans * rng.next_double());
    return t;
}

// proj/tests/support/helpers.hpp:34-46
Rigid helper_random_transform(RngStream& rng, double max_angle, double max_trans) {
    Vec3 axis = vec3_rtl([&](int) { return rng.next_gaussian(); });
    if (norm(axis) < 1e-12) axis = Vec3{1, 0, 0};
    axis = normalized(axis);
    double angle = rng.next_double(0.0, max_angle);
    Rigid t;
    t.R = angle_axis(angle, axis);
    t.t = vec3_rtl([&](int) { return rng.next_double(-max_trans, max_trans); });
    return t;
}

struct Fixture {
    std::vector<Cloud> clouds;
    std::vector<Rigid> transforms;
    std::vector<double> scalars;
};

const Intrinsics kFragK{130.0, 130.0, 80.0, 60.0, 160, 120};

// proj/src/synth.cpp:592-623
Fixture registration_pair(uint64_t seed, double leaf) {
    for (uint64_t attempt = 0; attempt < 64; ++attempt) {
        RngStream rng(seed, 0xA110 + attempt);
        Scene scene = make_scatter_scene(seed * 64 + attempt);
        double theta0 = 2.0 * M_PI * rng.next_double();
        double delta = 2.0 * M_PI * (0.065 + 0.04 * rng.next_double());
        Cloud a = fragment_union(scene, kFragK, theta0, 0.20, 0.005, rng, 2.6, Vec3{}, leaf);
        Cloud b = fragment_union(scene, kFragK, theta0 + delta, 0.20, 0.005, rng, 2.3, Vec3{}, leaf);
        if (a.size() < 2500 || b.size() < 2500) continue;
        Vec3 c = centroid(b);
        recenter(a, c);
        recenter(b, c);
        HostGrid grid;
        build_host_grid(grid, b.pos, 0.075, Vec3{});
        size_t hits = 0;
        for (const Vec3& p : a.pos)
            if (host_nn_within(grid, p, 0.075, nullptr) >= 0) hits += 1;
        double overlap = static_cast<double>(hits) / static_cast<double>(a.size());
        if (overlap < 0.62) continue;
        Rigid displace = synth_random_transform(rng, M_PI / 3.0, 1.0);
        Fixture f;
        f.clouds.push_back(transformed(a, displace));
        f.clouds.push_back(std::move(b));
        f.transforms.push_back(inverse(displace));
        f.scalars.push_back(overlap);
        return f;
    }
    throw Status(LK_DEGENERATE, "synth_registration_pair: no overlapping view pair found");
}

// proj/src/synth.cpp:625-653
Fixture negative_pair(uint64_t seed, double leaf) {
    RngStream rng(seed, 0xBAD);
    Scene sa = make_scatter_scene(seed * 2 + 1);
    Scene sb = make_scatter_scene(seed * 2 + 2);
    auto views = [&](const Scene& scene) {
        int stride = leaf < 0.04 ? 3 : 2;
        Cloud world;
        double theta0 = 2.0 * M_PI * rng.next_double();
        for (int view = 0; view < 3; ++view) {
            double theta = theta0 + 0.25 * view;
            Vec3 eye{1.8 * std::sin(theta), 0.4 * std::sin(theta * 1.7), 1.8 * std::cos(theta)};
            Rigid pose = look_at(eye, Vec3{});
            append(world, transformed(render_view(scene, pose, kFragK, stride, 0.005, rng), pose));
        }
        Cloud down = voxel_downsample(world, leaf);
        recenter(down, centroid(down));
        return down;
    };
    Fixture f;
    f.clouds.push_back(views(sa));
    f.clouds.push_back(views(sb));
    f.transforms.push_back(Rigid{});
    f.scalars.push_back(0.0);
    return f;
}

// Config B1/B2: two full-resolution depth-frame clouds of the
// room scene from the synth_scene orbit (proj/src/synth.cpp:340-367 renders
// frame i with RngStream(seed, 0x3E0 + i)); truth maps frame a's camera
// coordinates into frame b's.
Fixture frame_pair(uint64_t seed, int boxes, int width, int height, double fx, double fy, double cx, double cy,
                   int stride, double noise, int frames, int frame_a, int frame_b) {
    Scene scene = make_room_scene(seed, boxes);
    Intrinsics k{fx, fy, cx, cy, width, height};
    Rigid pa = orbit_pose(frames, frame_a), pb = orbit_pose(frames, frame_b);
    RngStream ra(seed, 0x3E0 + static_cast<uint64_t>(frame_a));
    RngStream rb(seed, 0x3E0 + static_cast<uint64_t>(frame_b));
    Fixture f;
    f.clouds.push_back(render_view(scene, pa, k, stride, noise, ra));
    f.clouds.push_back(render_view(scene, pb, k, stride, noise, rb));
    f.transforms.push_back(compose(inverse(pb), pa));
    f.scalars.push_back(0.0);
    return f;
}

// Config D: two submaps of make_room_scene(seed), each the
// world-frame union of `views` full renders along an orbit arc (frames
// a0 + step k and b0 + step k of the synth_scene orbit), not downsampled;
// the source is displaced by synth_random_transform(pi/3, 1 m) from
// RngStream(seed, 0xD00); truth maps the source back onto the target.
Fixture submap_pair(uint64_t seed, int boxes, int views, int width, int height, int stride, double noise, int frames,
                    int a0, int b0, int step) {
    Scene scene = make_room_scene(seed, boxes);
    Intrinsics k{525.0, 525.0, 319.5 * width / 640.0, 239.5 * height / 480.0, width, height};
    auto submap = [&](int f0) {
        Cloud world;
        for (int v = 0; v < views; ++v) {
            const int fr = f0 + step * v;
            Rigid pose = orbit_pose(frames, fr);
            RngStream r(seed, 0xD10 + static_cast<uint64_t>(fr));
            append(world, transformed(render_view(scene, pose, k, stride, noise, r), pose));
        }
        return world;
    };
    Cloud a = submap(a0), b = submap(b0);
    RngStream rng(seed, 0xD00);
    Rigid displace = synth_random_transform(rng, M_PI / 3.0, 1.0);
    Fixture f;
    f.clouds.push_back(transformed(a, displace));
    f.clouds.push_back(std::move(b));
    f.transforms.push_back(inverse(displace));
    f.scalars.push_back(0.0);
    return f;
}

// Config A: Q = sample_surface(scatter scene), P = T^-1 (Q + noise).
Fixture surface_pair(uint64_t seed, double density, double noise) {
    Scene scene = make_scatter_scene(seed);
    Cloud q = sample_surface(scene, density, seed);
    RngStream trng(seed, 0xA110);
    Rigid truth = synth_random_transform(trng, M_PI / 3.0, 1.0);
    Rigid inv = inverse(truth);
    RngStream nrng(seed, 0xA11CE);
    Cloud p;
    p.pos.reserve(q.size());
    p.nrm.reserve(q.size());
    for (size_t i = 0; i < q.size(); ++i) {
        Vec3 noisy = q.pos[i];
        noisy.x += noise * nrng.next_gaussian();
        noisy.y += noise * nrng.next_gaussian();
        noisy.z += noise * nrng.next_gaussian();
        p.pos.push_back(apply(inv, noisy));
        p.nrm.push_back(inv.R * q.nrm[i]);
    }
    Fixture f;
    f.clouds.push_back(std::move(p));
    f.clouds.push_back(std::move(q));
    f.transforms.push_back(truth);
    f.scalars.push_back(0.0);
    return f;
}

thread_local std::string g_synth_err;

template <class F>
void* guard(int* status, F&& fn) {
    try {
        Fixture* f = new Fixture(fn());
        *status = LK_OK;
        return f;
    } catch (const Status& e) {
        g_synth_err = e.what();
        *status = e.code;
    } catch (const std::exception& e) {
        g_synth_err = e.what();
        *status = LK_INTERNAL_ERROR;
    }
    return nullptr;
}

}  // namespace
}  // namespace lk

using namespace lk;

extern "C" {

// Test hooks for lk_acos_cr.hpp (tests/test_acos_cr.py): acos_cr against this
// machine's libm acos. check: the given arguments; sweep: n xorshift draws,
// uniform on [0, 1) and cubed (more small arguments) alternately.
void lks_acos_cr_check(const double* xs, int64_t n, int64_t* decided, int64_t* wrong) {
    int64_t d = 0, w = 0;
    for (int64_t k = 0; k < n; ++k) {
        double c;
        if (lkacos::acos_cr(xs[k], &c)) {
            ++d;
            if (c != std::acos(xs[k])) ++w;
        }
    }
    *decided = d;
    *wrong = w;
}

// acos_greater(x1, x2) against libm's acos(x1) > acos(x2) on pairs of
// arguments a few ulps apart (the FPFH ties)
void lks_acos_greater_sweep(uint64_t seed, int64_t n, int64_t* decided, int64_t* wrong) {
    uint64_t s = seed | 1u;
    int64_t d = 0, w = 0;
    for (int64_t k = 0; k < n; ++k) {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        double x1 = static_cast<double>(s >> 11) * 0x1p-53;
        if (k & 1) x1 = x1 * x1 * x1;
        double x2 = x1;
        for (int j = static_cast<int>(s & 7u); j >= 0; --j) x2 = std::nextafter(x2, 2.0);
        if (k & 2) std::swap(x1, x2);
        const int g = lkacos::acos_greater(x1, x2);
        if (g != 2) {
            ++d;
            if (g != (std::acos(x1) > std::acos(x2) ? 1 : 0)) ++w;
        }
    }
    *decided = d;
    *wrong = w;
}

// swap_decision's first rule (csrc/lk_prepare.cu): arguments more than
// 2.5e-16 apart have libm acos values ordered like the exact ones
void lks_acos_threshold_sweep(uint64_t seed, int64_t n, int64_t* checked, int64_t* wrong) {
    uint64_t s = seed | 1u;
    int64_t c = 0, w = 0;
    for (int64_t k = 0; k < n; ++k) {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        double x1 = static_cast<double>(s >> 11) * 0x1p-53;
        if (k % 3 == 1) x1 = x1 * x1 * x1;
        if (k % 3 == 2) x1 = 1.0 - x1 * x1 * x1;
        // the smallest step above 2.5e-16, plus a few ulps
        double x2 = x1 + 2.5e-16;
        for (int j = static_cast<int>(s & 3u); j >= 0; --j) x2 = std::nextafter(x2, 2.0);
        if (!(x2 <= 1.0) || !(x2 - x1 > 2.5e-16)) continue;
        ++c;
        if (!(std::acos(x1) > std::acos(x2))) ++w;
    }
    *checked = c;
    *wrong = w;
}

void lks_acos_cr_sweep(uint64_t seed, int64_t n, int64_t* decided, int64_t* wrong) {
    uint64_t s = seed | 1u;
    int64_t d = 0, w = 0;
    for (int64_t k = 0; k < n; ++k) {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        double x = static_cast<double>(s >> 11) * 0x1p-53;
        if (k & 1) x = x * x * x;
        double c;
        if (lkacos::acos_cr(x, &c)) {
            ++d;
            if (c != std::acos(x)) ++w;
        }
    }
    *decided = d;
    *wrong = w;
}

const char* lks_last_error(void) { return g_synth_err.c_str(); }

void* lks_registration_pair(uint64_t seed, double leaf, int* status) {
    return guard(status, [&] { return registration_pair(seed, leaf); });
}
void* lks_negative_pair(uint64_t seed, double leaf, int* status) {
    return guard(status, [&] { return negative_pair(seed, leaf); });
}
void* lks_frame_pair(uint64_t seed, int boxes, int width, int height, double fx, double fy, double cx, double cy,
                     int stride, double noise, int frames, int frame_a, int frame_b, int* status) {
    return guard(status, [&] {
        return frame_pair(seed, boxes, width, height, fx, fy, cx, cy, stride, noise, frames, frame_a, frame_b);
    });
}
void* lks_submap_pair(uint64_t seed, int boxes, int views, int width, int height, int stride, double noise,
                      int frames, int a0, int b0, int step, int* status) {
    return guard(status,
                 [&] { return submap_pair(seed, boxes, views, width, height, stride, noise, frames, a0, b0, step); });
}
void* lks_surface_pair(uint64_t seed, double density, double noise, int* status) {
    return guard(status, [&] { return surface_pair(seed, density, noise); });
}
// proj/tests/support/helpers.hpp:16-31 (draws from one stream, positions then normals)
void* lks_random_cloud(uint64_t seed, uint64_t stream, int n, double lo, double hi, int with_normals, int* status) {
    return guard(status, [&] {
        RngStream rng(seed, stream);
        Fixture f;
        Cloud c;
        for (int i = 0; i < n; ++i) {
            c.pos.push_back(vec3_rtl([&](int) { return rng.next_double(lo, hi); }));
        }
        if (with_normals) {
            for (int i = 0; i < n; ++i) {
                Vec3 v = vec3_rtl([&](int) { return rng.next_gaussian(); });
                double len = norm(v);
                c.nrm.push_back(len > 1e-12 ? v / len : Vec3{0, 0, 1});
            }
        }
        f.clouds.push_back(std::move(c));
        return f;
    });
}
int64_t lks_count(void* h, int which) {
    auto* f = static_cast<Fixture*>(h);
    return which < static_cast<int>(f->clouds.size()) ? static_cast<int64_t>(f->clouds[which].size()) : -1;
}
int lks_has_normals(void* h, int which) { return static_cast<Fixture*>(h)->clouds[which].has_normals() ? 1 : 0; }
void lks_get(void* h, int which, double* xyz, double* nxyz) {
    const Cloud& c = static_cast<Fixture*>(h)->clouds[which];
    for (size_t i = 0; i < c.size(); ++i) {
        if (xyz) store3(xyz, static_cast<int64_t>(i), c.pos[i]);
        if (nxyz && c.has_normals()) store3(nxyz, static_cast<int64_t>(i), c.nrm[i]);
    }
}
void lks_truth(void* h, double* R9, double* t3, double* scalar) {
    auto* f = static_cast<Fixture*>(h);
    store_mat(R9, f->transforms[0].R);
    store3(t3, 0, f->transforms[0].t);
    if (scalar) *scalar = f->scalars[0];
}
void lks_free(void* h) { delete static_cast<Fixture*>(h); }

// RigidTransform helpers with the reference's evaluation order
void lks_transform_from_twist(const double* xi6, double* R9, double* t3) {
    Rigid t = transform_from_twist(xi6);
    store_mat(R9, t.R);
    store3(t3, 0, t.t);
}
void lks_compose(const double* Ra, const double* ta, const double* Rb, const double* tb, double* R9, double* t3) {
    Rigid a{load_mat(Ra), load3(ta, 0)}, b{load_mat(Rb), load3(tb, 0)};
    Rigid c = compose(a, b);
    store_mat(R9, c.R);
    store3(t3, 0, c.t);
}
void lks_inverse(const double* Ra, const double* ta, double* R9, double* t3) {
    Rigid c = inverse(Rigid{load_mat(Ra), load3(ta, 0)});
    store_mat(R9, c.R);
    store3(t3, 0, c.t);
}
void lks_apply(const double* R9, const double* t3, const double* xyz, int64_t n, double* out) {
    Rigid T{load_mat(R9), load3(t3, 0)};
    for (int64_t i = 0; i < n; ++i) store3(out, i, apply(T, load3(xyz, i)));
}
void lks_rotate(const double* R9, const double* xyz, int64_t n, double* out) {
    Mat3 R = load_mat(R9);
    for (int64_t i = 0; i < n; ++i) store3(out, i, R * load3(xyz, i));
}
void lks_random_transform(uint64_t seed, uint64_t stream, int skip_draws, double max_angle, double max_trans,
                          double* R9, double* t3) {
    RngStream rng(seed, stream);
    for (int i = 0; i < skip_draws; ++i) rng.next_u64();
    Rigid t = helper_random_transform(rng, max_angle, max_trans);
    store_mat(R9, t.R);
    store3(t3, 0, t.t);
}
void lks_angle_axis(double angle, const double* axis3, double* R9) { store_mat(R9, angle_axis(angle, load3(axis3, 0))); }

}  // extern "C"
