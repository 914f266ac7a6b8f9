// lk_host_math.hpp -- host-side FP64 vector/matrix helpers for the product.
//
// Evaluation order follows the reference's Eigen expressions as documented
// in DESIGN.md ("Arithmetic contract"), so host-side results (fixtures,
// prepare stage, merges) agree bit-for-bit with the device code in
// lk_device_math.cuh. Compiled with -ffp-contract=off (no FMA).
#pragma once

#include <stdexcept>
#include <string>

#include <cmath>
#include <cstdint>

namespace lk {

// Error carrying an lk_status code (include/loopkit_b200.h).
struct Status : std::runtime_error {
    int code;
    Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct Vec3 {
    double x = 0, y = 0, z = 0;
    double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
    double& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
};

inline Vec3 operator+(Vec3 a, Vec3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline Vec3 operator-(Vec3 a, Vec3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline Vec3 operator-(Vec3 a) { return {-a.x, -a.y, -a.z}; }
inline Vec3 operator*(double s, Vec3 a) { return {s * a.x, s * a.y, s * a.z}; }
inline Vec3 operator*(Vec3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline Vec3 operator/(Vec3 a, double s) { return {a.x / s, a.y / s, a.z / s}; }
inline double dot(Vec3 a, Vec3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
inline double squared_norm(Vec3 a) { return (a.x * a.x + a.y * a.y) + a.z * a.z; }
inline double norm(Vec3 a) { return std::sqrt(squared_norm(a)); }
inline bool is_zero(Vec3 a) { return a.x == 0.0 && a.y == 0.0 && a.z == 0.0; }
inline Vec3 cross(Vec3 a, Vec3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
// Eigen normalized(): v / sqrt(squaredNorm) when > 0
inline Vec3 normalized(Vec3 a) {
    double z = squared_norm(a);
    return z > 0.0 ? a / std::sqrt(z) : a;
}
inline Vec3 cmin(Vec3 a, Vec3 b) { return {b.x < a.x ? b.x : a.x, b.y < a.y ? b.y : a.y, b.z < a.z ? b.z : a.z}; }
inline Vec3 cmax(Vec3 a, Vec3 b) { return {a.x < b.x ? b.x : a.x, a.y < b.y ? b.y : a.y, a.z < b.z ? b.z : a.z}; }

struct Mat3 {
    double m[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};  // m[row][col]; identity by default
    static Mat3 zero() {
        Mat3 r;
        for (auto& row : r.m)
            for (double& v : row) v = 0.0;
        return r;
    }
};

inline Mat3 transpose(const Mat3& a) {
    Mat3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[j][i];
    return r;
}
// Matrix3d * Vector3d: rows 0-1 ((a0 + a1) + a2), row 2 a0 + (a1 + a2)
inline Vec3 operator*(const Mat3& a, Vec3 v) {
    return {(a.m[0][0] * v.x + a.m[0][1] * v.y) + a.m[0][2] * v.z,
            (a.m[1][0] * v.x + a.m[1][1] * v.y) + a.m[1][2] * v.z,
            a.m[2][0] * v.x + (a.m[2][1] * v.y + a.m[2][2] * v.z)};
}
// R.transpose() * v as an Eigen expression: the transposed (row-major) lhs
// has no packet path, each row is a contiguous dot: ((a0 + a1) + a2).
inline Vec3 transpose_mul(const Mat3& r, Vec3 v) {
    return {(r.m[0][0] * v.x + r.m[1][0] * v.y) + r.m[2][0] * v.z,
            (r.m[0][1] * v.x + r.m[1][1] * v.y) + r.m[2][1] * v.z,
            (r.m[0][2] * v.x + r.m[1][2] * v.y) + r.m[2][2] * v.z};
}
inline Mat3 operator*(const Mat3& a, const Mat3& b) {
    Mat3 r;
    for (int j = 0; j < 3; ++j) {
        for (int i = 0; i < 2; ++i)
            r.m[i][j] = (a.m[i][0] * b.m[0][j] + a.m[i][1] * b.m[1][j]) + a.m[i][2] * b.m[2][j];
        r.m[2][j] = a.m[2][0] * b.m[0][j] + (a.m[2][1] * b.m[1][j] + a.m[2][2] * b.m[2][j]);
    }
    return r;
}

struct Rigid {
    Mat3 R;
    Vec3 t;
};
inline Vec3 apply(const Rigid& T, Vec3 p) { return T.R * p + T.t; }
// compose(a, b): b first, then a (proj/src/geometry.cpp:8-11)
inline Rigid compose(const Rigid& a, const Rigid& b) { return {a.R * b.R, a.R * b.t + a.t}; }
// inverse (proj/src/geometry.cpp:13-16)
inline Rigid inverse(const Rigid& t) {
    Mat3 rt = transpose(t.R);
    return {rt, -(rt * t.t)};
}

// Eigen AngleAxisd::toRotationMatrix
inline Mat3 angle_axis(double angle, Vec3 axis) {
    Mat3 res;
    Vec3 sin_axis = std::sin(angle) * axis;
    double c = std::cos(angle);
    Vec3 cos1_axis = (1.0 - c) * axis;
    double tmp;
    tmp = cos1_axis.x * axis.y;
    res.m[0][1] = tmp - sin_axis.z;
    res.m[1][0] = tmp + sin_axis.z;
    tmp = cos1_axis.x * axis.z;
    res.m[0][2] = tmp + sin_axis.y;
    res.m[2][0] = tmp - sin_axis.y;
    tmp = cos1_axis.y * axis.z;
    res.m[1][2] = tmp - sin_axis.x;
    res.m[2][1] = tmp + sin_axis.x;
    res.m[0][0] = cos1_axis.x * axis.x + c;
    res.m[1][1] = cos1_axis.y * axis.y + c;
    res.m[2][2] = cos1_axis.z * axis.z + c;
    return res;
}

// transform_from_twist: Rx(alpha) Ry(beta) Rz(gamma) (proj/src/geometry.cpp:42-52)
inline Rigid transform_from_twist(const double xi[6]) {
    double ca = std::cos(xi[0]), sa = std::sin(xi[0]);
    double cb = std::cos(xi[1]), sb = std::sin(xi[1]);
    double cg = std::cos(xi[2]), sg = std::sin(xi[2]);
    Mat3 rx, ry, rz;
    rx.m[1][1] = ca; rx.m[1][2] = -sa; rx.m[2][1] = sa; rx.m[2][2] = ca;
    ry.m[0][0] = cb; ry.m[0][2] = sb; ry.m[2][0] = -sb; ry.m[2][2] = cb;
    rz.m[0][0] = cg; rz.m[0][1] = -sg; rz.m[1][0] = sg; rz.m[1][1] = cg;
    return {rx * ry * rz, Vec3{xi[3], xi[4], xi[5]}};
}

inline Vec3 load3(const double* p, int64_t i) { return {p[3 * i], p[3 * i + 1], p[3 * i + 2]}; }
inline void store3(double* p, int64_t i, Vec3 v) {
    p[3 * i] = v.x;
    p[3 * i + 1] = v.y;
    p[3 * i + 2] = v.z;
}
inline Mat3 load_mat(const double* R9) {
    Mat3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[i][j] = R9[3 * i + j];
    return r;
}
inline void store_mat(double* R9, const Mat3& r) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) R9[3 * i + j] = r.m[i][j];
}

// ---- counter-based RNG (proj/include/loopkit/rng.hpp) ----
inline uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

class RngStream {
public:
    RngStream(uint64_t seed, uint64_t stream)
        : state_(splitmix64(splitmix64(seed) ^ (stream * 0xd1342543de82ef95ull))) {}
    uint64_t next_u64() {
        counter_ += 1;
        return splitmix64(state_ ^ (counter_ * 0x2545f4914f6cdd1dull));
    }
    uint32_t next_bounded(uint32_t bound) {
        while (true) {
            uint64_t x = next_u64() >> 32;
            uint64_t m = x * static_cast<uint64_t>(bound);  // x, bound < 2^32: exact in 64 bits
            uint64_t lo = m & 0xffffffffull;
            if (lo >= bound || lo >= (0x100000000ull % bound)) return static_cast<uint32_t>(m >> 32);
        }
    }
    double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double next_double(double lo, double hi) { return lo + (hi - lo) * next_double(); }
    double next_gaussian() {
        if (have_spare_) {
            have_spare_ = false;
            return spare_;
        }
        double u1 = 0.0;
        while (u1 <= 0.0) u1 = next_double();
        double u2 = next_double();
        double r = std::sqrt(-2.0 * std::log(u1));
        double a = 2.0 * M_PI * u2;
        spare_ = r * std::sin(a);
        have_spare_ = true;
        return r * std::cos(a);
    }

private:
    uint64_t state_;
    uint64_t counter_ = 0;
    bool have_spare_ = false;
    double spare_ = 0.0;
};

}  // namespace lk
