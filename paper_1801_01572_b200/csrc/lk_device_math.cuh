// lk_device_math.cuh -- device-side FP64 arithmetic of the registration path.
//
// Every routine reproduces the reference's operation order exactly (DESIGN.md
// "Arithmetic contract"). This translation unit is
// compiled with -fmad=false: no FMA contraction, IEEE-rounded add/mul/div/sqrt,
// so integer outcomes (winner index, inlier counts, stats) are bit-exact
// against the CPU oracle and fitness/transform bits match too.
#pragma once

#include <cstdint>

namespace lkd {

struct V3 {
    double x, y, z;
};

__device__ __forceinline__ V3 mk(double x, double y, double z) { return V3{x, y, z}; }
__device__ __forceinline__ V3 sub(V3 a, V3 b) { return V3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 add(V3 a, V3 b) { return V3{a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ double dot(V3 a, V3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
__device__ __forceinline__ double sqnorm(V3 a) { return (a.x * a.x + a.y * a.y) + a.z * a.z; }
__device__ __forceinline__ bool is_zero(V3 a) { return a.x == 0.0 && a.y == 0.0 && a.z == 0.0; }
__device__ __forceinline__ V3 ld3(const double* __restrict__ p, int64_t i) {
    return V3{__ldg(p + 3 * i), __ldg(p + 3 * i + 1), __ldg(p + 3 * i + 2)};
}

// (x, y, z, 0) records: one 32-byte sector per point, two 16-byte loads
__device__ __forceinline__ V3 ld4(const double4* __restrict__ p, int64_t i) {
    const double2* q = reinterpret_cast<const double2*>(p + i);
    const double2 a = __ldg(q), b = __ldg(q + 1);
    return V3{a.x, a.y, b.x};
}

// Matrix3d * Vector3d: rows 0-1 ((a0 + a1) + a2), row 2 a0 + (a1 + a2).
// R is row-major r[9].
__device__ __forceinline__ V3 rot(const double* r, V3 v) {
    return V3{(r[0] * v.x + r[1] * v.y) + r[2] * v.z, (r[3] * v.x + r[4] * v.y) + r[5] * v.z,
              r[6] * v.x + (r[7] * v.y + r[8] * v.z)};
}
// RigidTransform::operator* (proj/include/loopkit/geometry.hpp:26)
__device__ __forceinline__ V3 xform(const double* r, const double* t, V3 v) {
    V3 a = rot(r, v);
    return V3{a.x + t[0], a.y + t[1], a.z + t[2]};
}

// ---- counter-based RNG (proj/include/loopkit/rng.hpp:14-46) --------------
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
struct Rng {
    uint64_t state, counter;
    __device__ __forceinline__ Rng(uint64_t seed_mix, uint64_t stream)
        : state(splitmix64(seed_mix ^ (stream * 0xd1342543de82ef95ull))), counter(0) {}
    __device__ __forceinline__ uint64_t next_u64() {
        counter += 1;
        return splitmix64(state ^ (counter * 0x2545f4914f6cdd1dull));
    }
    // Lemire; `thresh` = 2^32 mod bound, precomputed on the host
    __device__ __forceinline__ uint32_t next_bounded(uint32_t bound, uint32_t thresh) {
        while (true) {
            uint64_t x = next_u64() >> 32;
            uint64_t m = x * static_cast<uint64_t>(bound);
            uint32_t lo = static_cast<uint32_t>(m);
            if (lo >= bound || lo >= thresh) return static_cast<uint32_t>(m >> 32);
        }
    }
};

// ---- 3x3 Jacobi SVD (Eigen 3.4 JacobiSVD<Matrix3d>, full U/V) ------------
// Matrices are row-major m[3*r + c].
struct Rot {
    double c, s;
};
__device__ __forceinline__ void rot_apply(double& x, double& y, double c, double s) {
    double xi = x, yi = y;
    x = c * xi + s * yi;
    y = -s * xi + c * yi;
}
// applyOnTheLeft(p, q, j): rows p, q
__device__ __forceinline__ void apply_left(double* w, int p, int q, Rot j) {
    if (j.c == 1.0 && j.s == 0.0) return;
#pragma unroll
    for (int i = 0; i < 3; ++i) rot_apply(w[3 * p + i], w[3 * q + i], j.c, j.s);
}
// applyOnTheRight(p, q, j): columns p, q rotated by j^T
__device__ __forceinline__ void apply_right(double* w, int p, int q, Rot j) {
    double c = j.c, s = -j.s;
    if (c == 1.0 && s == 0.0) return;
#pragma unroll
    for (int i = 0; i < 3; ++i) rot_apply(w[3 * i + p], w[3 * i + q], c, s);
}
__device__ __forceinline__ Rot make_jacobi(double x, double y, double z) {
    const double dbl_min = 2.2250738585072014e-308;
    double deno = 2.0 * fabs(y);
    if (deno < dbl_min) return Rot{1.0, 0.0};
    double tau = (x - z) / deno;
    double w = sqrt(tau * tau + 1.0);
    double t = tau > 0.0 ? 1.0 / (tau + w) : 1.0 / (tau - w);
    double sign_t = t > 0.0 ? 1.0 : -1.0;
    double n = 1.0 / sqrt(t * t + 1.0);
    double s = -sign_t * (y / fabs(y)) * fabs(t) * n;
    return Rot{n, s};
}
__device__ __forceinline__ void real_2x2_jacobi_svd(const double* w, int p, int q, Rot* jl, Rot* jr) {
    const double dbl_min = 2.2250738585072014e-308;
    double m00 = w[3 * p + p], m01 = w[3 * p + q], m10 = w[3 * q + p], m11 = w[3 * q + q];
    double t = m00 + m11;
    double d = m10 - m01;
    Rot r1;
    if (fabs(d) < dbl_min) {
        r1 = Rot{1.0, 0.0};
    } else {
        double u = t / d;
        double tmp = sqrt(1.0 + u * u);
        r1 = Rot{u / tmp, 1.0 / tmp};
    }
    if (!(r1.c == 1.0 && r1.s == 0.0)) {
        rot_apply(m00, m10, r1.c, r1.s);
        rot_apply(m01, m11, r1.c, r1.s);
    }
    *jr = make_jacobi(m00, m01, m11);
    // j_left = rot1 * j_right^T
    double c2 = jr->c, s2 = -jr->s;
    *jl = Rot{r1.c * c2 - r1.s * s2, r1.c * s2 + r1.s * c2};
}

__device__ __forceinline__ double amax(double a, double b) { return a < b ? b : a; }  // std::max

// Returns singular values (descending) and U, V with A = U diag(S) V^T.
__device__ inline void jacobi_svd3(const double* A, double* U, double* S, double* V) {
    const double dbl_min = 2.2250738585072014e-308;
    const double precision = 2.0 * 2.220446049250313e-16;
    double scale = fabs(A[0]);
    // maxCoeff over cwiseAbs in column-major order (strict >)
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            double a = fabs(A[3 * i + j]);
            if (a > scale) scale = a;
        }
    if (scale == 0.0) scale = 1.0;
    double w[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) w[k] = A[k] / scale;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        U[k] = (k % 4 == 0) ? 1.0 : 0.0;
        V[k] = (k % 4 == 0) ? 1.0 : 0.0;
    }
    double max_diag = fabs(w[0]);
    if (fabs(w[4]) > max_diag) max_diag = fabs(w[4]);
    if (fabs(w[8]) > max_diag) max_diag = fabs(w[8]);
    bool finished = false;
    int sweeps = 0;
    while (!finished && sweeps < 1000) {
        finished = true;
        ++sweeps;
#pragma unroll
        for (int pq = 0; pq < 3; ++pq) {
            const int p = pq == 0 ? 1 : 2;
            const int q = pq == 0 ? 0 : (pq == 1 ? 0 : 1);
            double threshold = amax(dbl_min, precision * max_diag);
            if (fabs(w[3 * p + q]) > threshold || fabs(w[3 * q + p]) > threshold) {
                finished = false;
                Rot jl, jr;
                real_2x2_jacobi_svd(w, p, q, &jl, &jr);
                apply_left(w, p, q, jl);
                apply_right(U, p, q, Rot{jl.c, -jl.s});
                apply_right(w, p, q, jr);
                apply_right(V, p, q, jr);
                max_diag = amax(max_diag, amax(fabs(w[3 * p + p]), fabs(w[3 * q + q])));
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        double a = w[3 * i + i];
        S[i] = fabs(a);
        if (a < 0.0) {
#pragma unroll
            for (int r = 0; r < 3; ++r) U[3 * r + i] = -U[3 * r + i];
        }
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) S[i] *= scale;
    // descending sort, maxCoeff picks the first maximum
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        int pos = i;
        double mx = S[i];
#pragma unroll
        for (int k = i + 1; k < 3; ++k)
            if (S[k] > mx) {
                mx = S[k];
                pos = k;
            }
        if (mx == 0.0) break;
        if (pos != i) {
            double tmp = S[i];
            S[i] = S[pos];
            S[pos] = tmp;
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                double a = U[3 * r + i];
                U[3 * r + i] = U[3 * r + pos];
                U[3 * r + pos] = a;
                double b = V[3 * r + i];
                V[3 * r + i] = V[3 * r + pos];
                V[3 * r + pos] = b;
            }
        }
    }
}

// Matrix3d * Matrix3d, per result column: rows 0-1 packet order, row 2 scalar.
__device__ __forceinline__ void mat_mul(const double* a, const double* b, double* r) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
#pragma unroll
        for (int i = 0; i < 2; ++i)
            r[3 * i + j] = (a[3 * i + 0] * b[0 + j] + a[3 * i + 1] * b[3 + j]) + a[3 * i + 2] * b[6 + j];
        r[6 + j] = a[6] * b[j] + (a[7] * b[3 + j] + a[8] * b[6 + j]);
    }
}
__device__ __forceinline__ void mat_transpose(const double* a, double* r) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) r[3 * i + j] = a[3 * j + i];
}
// Eigen determinant_impl<3>
__device__ __forceinline__ double det3(const double* m) {
    double h0 = m[0] * (m[4] * m[8] - m[5] * m[7]);
    double h1 = m[1] * (m[3] * m[8] - m[5] * m[6]);
    double h2 = m[2] * (m[3] * m[7] - m[4] * m[6]);
    return h0 - h1 + h2;
}

// kabsch for 4 pairs (proj/src/geometry.cpp:62-91). Returns false when the
// covariance has rank < 2 (DegenerateConfiguration).
__device__ inline bool kabsch4(const V3 (&src)[4], const V3 (&dst)[4], double* R, double* t) {
    V3 cs = mk(0.0, 0.0, 0.0), cd = mk(0.0, 0.0, 0.0);
#pragma unroll
    for (int i = 0; i < 4; ++i) cs = add(cs, src[i]);
#pragma unroll
    for (int i = 0; i < 4; ++i) cd = add(cd, dst[i]);
    cs = mk(cs.x / 4.0, cs.y / 4.0, cs.z / 4.0);
    cd = mk(cd.x / 4.0, cd.y / 4.0, cd.z / 4.0);
    double h[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) h[k] = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        V3 a = sub(src[i], cs), b = sub(dst[i], cd);
        double av[3] = {a.x, a.y, a.z}, bv[3] = {b.x, b.y, b.z};
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) h[3 * r + c] = h[3 * r + c] + av[r] * bv[c];
    }
    double U[9], S[3], V[9];
    jacobi_svd3(h, U, S, V);
    double scale = amax(S[0], 1.0);
    if (S[1] <= 1e-12 * scale) return false;
    double Ut[9], VUt[9];
    mat_transpose(U, Ut);
    mat_mul(V, Ut, VUt);
    double D[9] = {1, 0, 0, 0, 1, 0, 0, 0, det3(VUt) < 0 ? -1.0 : 1.0};
    double VD[9];
    mat_mul(V, D, VD);
    mat_mul(VD, Ut, R);
    V3 rc = rot(R, cs);
    t[0] = cd.x - rc.x;
    t[1] = cd.y - rc.y;
    t[2] = cd.z - rc.z;
    return true;
}

}  // namespace lkd
