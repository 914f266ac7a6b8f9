// lk_eig3.hpp -- Eigen's SelfAdjointEigenSolver<Matrix3d> (eigenvectors on),
// operation for operation, for estimate_normals (proj/src/preprocess.cpp:90-91:
// the eigenvector of the smallest eigenvalue of the 3x3 covariance).
//
// Restated from Eigen 3.4 (the reference vendors no Eigen here, so this order
// is the builder's statement of it):
//   * scale = max |lower-triangle coefficient| (1 if 0); the lower triangle
//     divided by it (SelfAdjointEigenSolver::compute);
//   * tridiagonalization_inplace_selector<3x3> (closed form Householder);
//   * computeFromTridiagonal_impl: deflation |e_i| < min_double or
//     (e_i / eps)^2 <= |d_i| + |d_i+1|, Wilkinson-shifted implicit QR steps
//     (tridiagonal_qr_step with hypot and makeGivens), at most 30 n sweeps;
//   * on success, ascending sort of the eigenvalues (first minimum) with the
//     eigenvector columns swapped along.
// Usable on host (g++ -ffp-contract=off) and device (nvcc -fmad=false).
#pragma once

#include <cfloat>
#include <cmath>

#ifdef __CUDACC__
#define LK_HD __host__ __device__ __forceinline__
#else
#define LK_HD inline
#endif

namespace lkeig {

LK_HD double dabs(double x) { return x < 0.0 ? -x : (x == 0.0 ? 0.0 : x); }

// numext::hypot -> positive_real_hypot(|x|, |y|)
LK_HD double hypot_e(double x, double y) {
    x = dabs(x);
    y = dabs(y);
    if (std::isinf(x) || std::isinf(y)) return HUGE_VAL;
    if (std::isnan(x) || std::isnan(y)) return x + y;  // a quiet NaN
    const double p = x < y ? y : x;  // numext::maxi(x, y)
    if (p == 0.0) return 0.0;
    const double qp = (y < x ? y : x) / p;  // numext::mini(y, x) / p
    return p * sqrt(1.0 + qp * qp);
}

// JacobiRotation<double>::makeGivens(p, q) (real case, no r)
LK_HD void make_givens(double p, double q, double& c, double& s) {
    if (q == 0.0) {
        c = p < 0.0 ? -1.0 : 1.0;
        s = 0.0;
    } else if (p == 0.0) {
        c = 0.0;
        s = q < 0.0 ? 1.0 : -1.0;
    } else if (dabs(p) > dabs(q)) {
        const double t = q / p;
        double u = sqrt(1.0 + t * t);
        if (p < 0.0) u = -u;
        c = 1.0 / u;
        s = -t * c;
    } else {
        const double t = p / q;
        double u = sqrt(1.0 + t * t);
        if (q < 0.0) u = -u;
        s = -1.0 / u;
        c = -t * s;
    }
}

// Q (column-major 3x3, Q[3 * col + row]) .applyOnTheRight(k, k + 1, rot):
// apply_rotation_in_the_plane(col k, col k+1, rot.transpose()), i.e. with
// (c, -s): x = c x - s y, y = s x + c y
LK_HD void rotate_cols(double* Q, int k, double c, double s) {
    for (int i = 0; i < 3; ++i) {
        const double xi = Q[3 * k + i], yi = Q[3 * (k + 1) + i];
        Q[3 * k + i] = c * xi + -s * yi;
        Q[3 * (k + 1) + i] = -(-s) * xi + c * yi;
    }
}

// tridiagonal_qr_step (column-major Q)
LK_HD void qr_step(double* diag, double* subdiag, int start, int end, double* Q) {
    const double td = (diag[end - 1] - diag[end]) * 0.5;
    const double e = subdiag[end - 1];
    double mu = diag[end];
    if (td == 0.0) {
        mu -= dabs(e);
    } else if (e != 0.0) {
        const double e2 = e * e;
        const double h = hypot_e(td, e);
        if (e2 == 0.0) {
            mu -= e / ((td + (td > 0.0 ? h : -h)) / e);
        } else {
            mu -= e2 / (td + (td > 0.0 ? h : -h));
        }
    }
    double x = diag[start] - mu;
    double z = subdiag[start];
    for (int k = start; k < end && z != 0.0; ++k) {
        double c, s;
        make_givens(x, z, c, s);
        const double sdk = s * diag[k] + c * subdiag[k];
        const double dkp1 = s * subdiag[k] + c * diag[k + 1];
        diag[k] = c * (c * diag[k] - s * subdiag[k]) - s * (c * subdiag[k] - s * diag[k + 1]);
        diag[k + 1] = s * sdk + c * dkp1;
        subdiag[k] = c * sdk - s * dkp1;
        if (k > start) subdiag[k - 1] = c * subdiag[k - 1] - s * z;
        x = subdiag[k];
        if (k < end - 1) {
            z = -s * subdiag[k + 1];
            subdiag[k + 1] = c * subdiag[k + 1];
        }
        rotate_cols(Q, k, c, s);
    }
}

// Eigenvector of the smallest eigenvalue of the symmetric 3x3 matrix whose
// lower triangle is a00, a10, a20, a11, a21, a22 (column 0 of the sorted
// eigenvector matrix; unsorted if the iteration did not converge).
LK_HD void smallest_eigenvector(double a00, double a10, double a20, double a11, double a21, double a22, double* v) {
    // scale (compute(): mat = lower triangle, upper part zero)
    double scale = dabs(a00);
    const double lower[5] = {a10, a20, a11, a21, a22};
    for (int k = 0; k < 5; ++k) {
        const double m = dabs(lower[k]);
        if (m > scale) scale = m;
    }
    if (scale == 0.0) scale = 1.0;
    a00 /= scale;
    a10 /= scale;
    a20 /= scale;
    a11 /= scale;
    a21 /= scale;
    a22 /= scale;
    // tridiagonalization_inplace_selector<MatrixType, 3, false>
    double diag[3], sub[2], Q[9];
    diag[0] = a00;
    const double v1norm2 = a20 * a20;
    if (v1norm2 <= DBL_MIN) {
        diag[1] = a11;
        diag[2] = a22;
        sub[0] = a10;
        sub[1] = a21;
        for (int k = 0; k < 9; ++k) Q[k] = (k % 4 == 0) ? 1.0 : 0.0;
    } else {
        const double beta = sqrt(a10 * a10 + v1norm2);
        const double inv_beta = 1.0 / beta;
        const double m01 = a10 * inv_beta;
        const double m02 = a20 * inv_beta;
        const double q = 2.0 * m01 * a21 + m02 * (a22 - a11);
        diag[1] = a11 + m02 * q;
        diag[2] = a22 - m02 * q;
        sub[0] = beta;
        sub[1] = a21 - m01 * q;
        // mat << 1, 0, 0, 0, m01, m02, 0, m02, -m01 (column-major storage)
        Q[0] = 1.0; Q[1] = 0.0; Q[2] = 0.0;
        Q[3] = 0.0; Q[4] = m01; Q[5] = m02;
        Q[6] = 0.0; Q[7] = m02; Q[8] = -m01;
    }
    // computeFromTridiagonal_impl
    const int n = 3;
    int end = n - 1, start = 0, iter = 0;
    const double precision_inv = 1.0 / DBL_EPSILON;
    while (end > 0) {
        for (int i = start; i < end; ++i) {
            if (dabs(sub[i]) < DBL_MIN) {
                sub[i] = 0.0;
            } else {
                const double scaled = precision_inv * sub[i];
                if (scaled * scaled <= (dabs(diag[i]) + dabs(diag[i + 1]))) sub[i] = 0.0;
            }
        }
        while (end > 0 && sub[end - 1] == 0.0) end--;
        if (end <= 0) break;
        iter++;
        if (iter > 30 * n) break;
        start = end - 1;
        while (start > 0 && sub[start - 1] != 0.0) start--;
        qr_step(diag, sub, start, end, Q);
    }
    if (iter <= 30 * n) {
        for (int i = 0; i < n - 1; ++i) {
            int k = 0;  // minCoeff(&k) over diag[i..n-1]: first minimum
            for (int j = 1; j < n - i; ++j)
                if (diag[i + j] < diag[i + k]) k = j;
            if (k > 0) {
                const double t = diag[i];
                diag[i] = diag[i + k];
                diag[i + k] = t;
                for (int r = 0; r < 3; ++r) {
                    const double u = Q[3 * i + r];
                    Q[3 * i + r] = Q[3 * (i + k) + r];
                    Q[3 * (i + k) + r] = u;
                }
            }
        }
    }
    v[0] = Q[0];
    v[1] = Q[1];
    v[2] = Q[2];
}

}  // namespace lkeig

#undef LK_HD
