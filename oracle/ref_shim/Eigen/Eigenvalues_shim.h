// oracle/ref_shim/Eigen/Eigenvalues_shim.h -- TEST INFRASTRUCTURE ONLY.
// SelfAdjointEigenSolver for fixed-size symmetric matrices.
//  * 3x3 (estimate_normals, proj/src/preprocess.cpp:87): Eigen 3.4's
//    iterative path restated -- scale by the max |lower coefficient|,
//    tridiagonalization_inplace_selector<3x3> (closed-form Householder),
//    computeFromTridiagonal_impl (deflation, Wilkinson-shifted
//    tridiagonal_qr_step with makeGivens and positive_real_hypot, at most 30 n
//    iterations), ascending sort (first minimum) with the eigenvector
//    columns swapped along. Written independently of the product's
//    csrc/lk_eig3.hpp so the two statements check each other.
//  * other sizes (only the reference's tolerance checks use them, e.g.
//    proj/tests/test_line_process.cpp:90 on a 6x6): cyclic Jacobi, NOT
//    Eigen's operation order.
#pragma once

namespace Eigen {

template <typename MatrixType>
class SelfAdjointEigenSolver {
public:
    using S = typename MatrixType::Scalar;
    static constexpr int N = MatrixType::RowsAtCompileTime;
    using MatN = Matrix<S, N, N>;
    using VecN = Matrix<S, N, 1>;

    SelfAdjointEigenSolver() = default;
    explicit SelfAdjointEigenSolver(const MatrixType& m, int options = ComputeEigenvectors) { compute(m, options); }

    SelfAdjointEigenSolver& compute(const MatrixType& m, int options = ComputeEigenvectors) {
        const bool vectors = (options & EigenvaluesOnly) == 0;
        if constexpr (N == 3) compute3(m, vectors);
        else compute_jacobi(m);
        return *this;
    }
    const MatN& eigenvectors() const { return vec_; }
    const VecN& eigenvalues() const { return val_; }
    ComputationInfo info() const { return info_; }

private:
    static S hypot_pos(S x, S y) {  // numext::hypot -> positive_real_hypot(|x|, |y|)
        x = std::abs(x);
        y = std::abs(y);
        if (std::isinf(x) || std::isinf(y)) return std::numeric_limits<S>::infinity();
        if (std::isnan(x) || std::isnan(y)) return std::numeric_limits<S>::quiet_NaN();
        S p = std::max(x, y);
        if (p == S(0)) return S(0);
        S qp = std::min(y, x) / p;
        return p * std::sqrt(S(1) + qp * qp);
    }
    // JacobiRotation::makeGivens(p, q), real scalars, no r
    static JacobiRotation<S> make_givens(S p, S q) {
        JacobiRotation<S> r;
        if (q == S(0)) {
            r.c() = p < S(0) ? S(-1) : S(1);
            r.s() = S(0);
        } else if (p == S(0)) {
            r.c() = S(0);
            r.s() = q < S(0) ? S(1) : S(-1);
        } else if (std::abs(p) > std::abs(q)) {
            S t = q / p;
            S u = std::sqrt(S(1) + t * t);
            if (p < S(0)) u = -u;
            r.c() = S(1) / u;
            r.s() = -t * r.c();
        } else {
            S t = p / q;
            S u = std::sqrt(S(1) + t * t);
            if (q < S(0)) u = -u;
            r.s() = -S(1) / u;
            r.c() = -t * r.s();
        }
        return r;
    }
    // internal::tridiagonal_qr_step (column-major Q)
    void qr_step(S* diag, S* sub, Index start, Index end) {
        S td = (diag[end - 1] - diag[end]) * S(0.5);
        S e = sub[end - 1];
        S mu = diag[end];
        if (td == S(0)) {
            mu -= std::abs(e);
        } else if (e != S(0)) {
            const S e2 = e * e;
            const S h = hypot_pos(td, e);
            if (e2 == S(0)) mu -= e / ((td + (td > S(0) ? h : -h)) / e);
            else mu -= e2 / (td + (td > S(0) ? h : -h));
        }
        S x = diag[start] - mu;
        S z = sub[start];
        for (Index k = start; k < end && z != S(0); ++k) {
            JacobiRotation<S> rot = make_givens(x, z);
            S sdk = rot.s() * diag[k] + rot.c() * sub[k];
            S dkp1 = rot.s() * sub[k] + rot.c() * diag[k + 1];
            diag[k] = rot.c() * (rot.c() * diag[k] - rot.s() * sub[k]) - rot.s() * (rot.c() * sub[k] - rot.s() * diag[k + 1]);
            diag[k + 1] = rot.s() * sdk + rot.c() * dkp1;
            sub[k] = rot.c() * sdk - rot.s() * dkp1;
            if (k > start) sub[k - 1] = rot.c() * sub[k - 1] - rot.s() * z;
            x = sub[k];
            if (k < end - 1) {
                z = -rot.s() * sub[k + 1];
                sub[k + 1] = rot.c() * sub[k + 1];
            }
            internal::apply_on_the_right(vec_, k, k + 1, rot);
        }
    }
    void compute3(const MatrixType& m, bool vectors) {
        // mat = lower triangle; scale = mat.cwiseAbs().maxCoeff()
        MatN mat = MatN::Zero();
        for (Index j = 0; j < 3; ++j)
            for (Index i = j; i < 3; ++i) mat.coeffRef(i, j) = m.coeff(i, j);
        S scale = mat.cwiseAbs().maxCoeff();
        if (scale == S(0)) scale = S(1);
        for (Index j = 0; j < 3; ++j)
            for (Index i = j; i < 3; ++i) mat.coeffRef(i, j) = mat.coeff(i, j) / scale;
        // tridiagonalization_inplace_selector<MatrixType, 3, false>
        S diag[3], sub[2];
        diag[0] = mat(0, 0);
        S v1norm2 = mat(2, 0) * mat(2, 0);
        if (v1norm2 <= std::numeric_limits<S>::min()) {
            diag[1] = mat(1, 1);
            diag[2] = mat(2, 2);
            sub[0] = mat(1, 0);
            sub[1] = mat(2, 1);
            vec_ = MatN::Identity();
        } else {
            S beta = std::sqrt(mat(1, 0) * mat(1, 0) + v1norm2);
            S inv_beta = S(1) / beta;
            S m01 = mat(1, 0) * inv_beta;
            S m02 = mat(2, 0) * inv_beta;
            S q = S(2) * m01 * mat(2, 1) + m02 * (mat(2, 2) - mat(1, 1));
            diag[1] = mat(1, 1) + m02 * q;
            diag[2] = mat(2, 2) - m02 * q;
            sub[0] = beta;
            sub[1] = mat(2, 1) - m01 * q;
            vec_ << S(1), S(0), S(0), S(0), m01, m02, S(0), m02, -m01;
        }
        (void)vectors;
        // computeFromTridiagonal_impl
        const Index n = 3;
        Index end = n - 1, start = 0, iter = 0;
        const S precision_inv = S(1) / std::numeric_limits<S>::epsilon();
        while (end > 0) {
            for (Index i = start; i < end; ++i) {
                if (std::abs(sub[i]) < std::numeric_limits<S>::min()) {
                    sub[i] = S(0);
                } else {
                    const S scaled = precision_inv * sub[i];
                    if (scaled * scaled <= (std::abs(diag[i]) + std::abs(diag[i + 1]))) sub[i] = S(0);
                }
            }
            while (end > 0 && sub[end - 1] == S(0)) end--;
            if (end <= 0) break;
            iter++;
            if (iter > 30 * n) break;
            start = end - 1;
            while (start > 0 && sub[start - 1] != S(0)) start--;
            qr_step(diag, sub, start, end);
        }
        info_ = iter <= 30 * n ? Success : NoConvergence;
        if (info_ == Success) {
            for (Index i = 0; i < n - 1; ++i) {
                Index k = 0;  // diag.segment(i, n - i).minCoeff(&k)
                for (Index j = 1; j < n - i; ++j)
                    if (diag[i + j] < diag[i + k]) k = j;
                if (k > 0) {
                    std::swap(diag[i], diag[k + i]);
                    for (Index r = 0; r < 3; ++r) std::swap(vec_.coeffRef(r, i), vec_.coeffRef(r, k + i));
                }
            }
        }
        for (Index i = 0; i < 3; ++i) val_.coeffRef(i) = diag[i] * scale;
    }
    void compute_jacobi(const MatrixType& m) {
        MatN a(m);
        vec_ = MatN::Identity();
        for (int sweep = 0; sweep < 100; ++sweep) {
            S off = 0;
            for (Index p = 0; p < N; ++p)
                for (Index q = p + 1; q < N; ++q) off += a(p, q) * a(p, q);
            if (off < S(1e-300)) break;
            for (Index p = 0; p < N; ++p)
                for (Index q = p + 1; q < N; ++q) {
                    if (a(p, q) == S(0)) continue;
                    S theta = (a(q, q) - a(p, p)) / (S(2) * a(p, q));
                    S t = (theta >= 0 ? S(1) : S(-1)) / (std::abs(theta) + std::sqrt(theta * theta + S(1)));
                    S c = S(1) / std::sqrt(t * t + S(1)), s = t * c;
                    for (Index k = 0; k < N; ++k) {
                        S akp = a(k, p), akq = a(k, q);
                        a(k, p) = c * akp - s * akq;
                        a(k, q) = s * akp + c * akq;
                    }
                    for (Index k = 0; k < N; ++k) {
                        S apk = a(p, k), aqk = a(q, k);
                        a(p, k) = c * apk - s * aqk;
                        a(q, k) = s * apk + c * aqk;
                    }
                    for (Index k = 0; k < N; ++k) {
                        S vkp = vec_(k, p), vkq = vec_(k, q);
                        vec_(k, p) = c * vkp - s * vkq;
                        vec_(k, q) = s * vkp + c * vkq;
                    }
                }
        }
        for (Index i = 0; i < N; ++i) val_.coeffRef(i) = a(i, i);
        for (Index i = 0; i < N - 1; ++i) {
            Index k = i;
            for (Index j = i + 1; j < N; ++j)
                if (val_(j) < val_(k)) k = j;
            if (k != i) {
                std::swap(val_.coeffRef(i), val_.coeffRef(k));
                for (Index r = 0; r < N; ++r) std::swap(vec_.coeffRef(r, i), vec_.coeffRef(r, k));
            }
        }
        info_ = Success;
    }

    MatN vec_ = MatN::Identity();
    VecN val_ = VecN::Zero();
    ComputationInfo info_ = Success;
};

}  // namespace Eigen
