// oracle/ref_shim/Eigen/JacobiSVD_shim.h -- TEST INFRASTRUCTURE ONLY.
// Eigen 3.4 JacobiSVD for a square real fixed-size matrix (no QR
// preconditioning needed when rows == cols), restated from Eigen's
// JacobiSVD::compute / real_2x2_jacobi_svd / JacobiRotation::makeJacobi /
// apply_rotation_in_the_plane. Written independently of oracle/lk_oracle.cpp's
// jacobi_svd3 so that the two statements check each other through the
// reference's kabsch (proj/src/geometry.cpp:77).
#pragma once

namespace Eigen {

template <typename S>
struct JacobiRotation {
    S c_ = S(1), s_ = S(0);
    JacobiRotation() = default;
    JacobiRotation(S c, S s) : c_(c), s_(s) {}
    S& c() { return c_; }
    S& s() { return s_; }
    S c() const { return c_; }
    S s() const { return s_; }
    JacobiRotation transpose() const { return JacobiRotation(c_, -s_); }
    JacobiRotation operator*(const JacobiRotation& o) const {
        return JacobiRotation(c_ * o.c_ - s_ * o.s_, c_ * o.s_ + s_ * o.c_);
    }
    // JacobiRotation::makeJacobi(x, y, z) for real scalars
    bool makeJacobi(S x, S y, S z) {
        S deno = S(2) * std::abs(y);
        if (deno < std::numeric_limits<S>::min()) {
            c_ = S(1);
            s_ = S(0);
            return false;
        }
        S tau = (x - z) / deno;
        S w = std::sqrt(tau * tau + S(1));
        S t = tau > S(0) ? S(1) / (tau + w) : S(1) / (tau - w);
        S sign_t = t > S(0) ? S(1) : S(-1);
        S n = S(1) / std::sqrt(t * t + S(1));
        s_ = -sign_t * (y / std::abs(y)) * std::abs(t) * n;
        c_ = n;
        return true;
    }
};

namespace internal {

// apply_rotation_in_the_plane(x, y, j): x' = c x + s y, y' = -s x + c y;
// an identity rotation returns early.
template <typename GetX, typename GetY, typename S>
void rotate_plane(Index n, GetX xr, GetY yr, const JacobiRotation<S>& j) {
    if (j.c() == S(1) && j.s() == S(0)) return;
    for (Index i = 0; i < n; ++i) {
        S& x = xr(i);
        S& y = yr(i);
        S xi = x, yi = y;
        x = j.c() * xi + j.s() * yi;
        y = -j.s() * xi + j.c() * yi;
    }
}

template <typename M, typename S>
void apply_on_the_left(M& m, Index p, Index q, const JacobiRotation<S>& j) {
    rotate_plane(m.cols(), [&](Index i) -> S& { return m.coeffRef(p, i); }, [&](Index i) -> S& { return m.coeffRef(q, i); }, j);
}
template <typename M, typename S>
void apply_on_the_right(M& m, Index p, Index q, const JacobiRotation<S>& j) {
    JacobiRotation<S> jt = j.transpose();
    rotate_plane(m.rows(), [&](Index i) -> S& { return m.coeffRef(i, p); }, [&](Index i) -> S& { return m.coeffRef(i, q); }, jt);
}

}  // namespace internal

template <typename MatrixType, int QRPreconditioner = 0>
class JacobiSVD {
public:
    using S = typename MatrixType::Scalar;
    static constexpr int N = MatrixType::RowsAtCompileTime;
    static_assert(N == MatrixType::ColsAtCompileTime && N > 0, "shim: square fixed-size JacobiSVD only");
    using MatN = Matrix<S, N, N>;
    using VecN = Matrix<S, N, 1>;

    JacobiSVD(const MatrixType& a, unsigned int options = 0) { compute(a, options); }

    const MatN& matrixU() const { return u_; }
    const MatN& matrixV() const { return v_; }
    const VecN& singularValues() const { return sv_; }
    Index nonzeroSingularValues() const { return nonzero_; }
    ComputationInfo info() const { return info_; }

private:
    void compute(const MatrixType& a, unsigned int options) {
        const bool compute_u = options & (ComputeFullU | ComputeThinU);
        const bool compute_v = options & (ComputeFullV | ComputeThinV);
        const S precision = S(2) * std::numeric_limits<S>::epsilon();
        const S consider_as_zero = std::numeric_limits<S>::min();
        // scale = cwiseAbs().maxCoeff<PropagateNaN>()
        S scale = std::abs(a.coeff(0, 0));
        for (Index j = 0; j < N; ++j)
            for (Index i = 0; i < N; ++i) {
                S v = std::abs(a.coeff(i, j));
                if (std::isnan(v) || v > scale) scale = v;
            }
        if (!std::isfinite(scale)) {
            info_ = InvalidInput;
            nonzero_ = 0;
            return;
        }
        if (scale == S(0)) scale = S(1);
        MatN w = MatN(a) / scale;
        u_ = MatN::Identity();
        v_ = MatN::Identity();
        // maxDiagEntry = cwiseAbs().diagonal().maxCoeff()
        S max_diag = std::abs(w.coeff(0, 0));
        for (Index i = 1; i < N; ++i)
            if (std::abs(w.coeff(i, i)) > max_diag) max_diag = std::abs(w.coeff(i, i));
        bool finished = false;
        while (!finished) {
            finished = true;
            for (Index p = 1; p < N; ++p) {
                for (Index q = 0; q < p; ++q) {
                    S threshold = std::max(consider_as_zero, precision * max_diag);
                    if (std::abs(w.coeff(p, q)) > threshold || std::abs(w.coeff(q, p)) > threshold) {
                        finished = false;
                        JacobiRotation<S> j_left, j_right;
                        real_2x2_jacobi_svd(w, p, q, &j_left, &j_right);
                        internal::apply_on_the_left(w, p, q, j_left);
                        if (compute_u) internal::apply_on_the_right(u_, p, q, j_left.transpose());
                        internal::apply_on_the_right(w, p, q, j_right);
                        if (compute_v) internal::apply_on_the_right(v_, p, q, j_right);
                        max_diag = std::max(max_diag, std::max(std::abs(w.coeff(p, p)), std::abs(w.coeff(q, q))));
                    }
                }
            }
        }
        for (Index i = 0; i < N; ++i) {
            S d = w.coeff(i, i);
            sv_.coeffRef(i) = std::abs(d);
            if (compute_u && d < S(0))
                for (Index r = 0; r < N; ++r) u_.coeffRef(r, i) = -u_.coeff(r, i);
        }
        sv_ *= scale;
        nonzero_ = N;
        for (Index i = 0; i < N; ++i) {
            // tail(N - i).maxCoeff(&pos): first maximum
            Index pos = 0;
            S mx = sv_.coeff(i);
            for (Index k = 1; k < N - i; ++k)
                if (sv_.coeff(i + k) > mx) {
                    mx = sv_.coeff(i + k);
                    pos = k;
                }
            if (mx == S(0)) {
                nonzero_ = i;
                break;
            }
            if (pos) {
                pos += i;
                std::swap(sv_.coeffRef(i), sv_.coeffRef(pos));
                for (Index r = 0; r < N; ++r) {
                    if (compute_u) std::swap(u_.coeffRef(r, pos), u_.coeffRef(r, i));
                    if (compute_v) std::swap(v_.coeffRef(r, pos), v_.coeffRef(r, i));
                }
            }
        }
        info_ = Success;
    }

    // internal::real_2x2_jacobi_svd
    static void real_2x2_jacobi_svd(const MatN& w, Index p, Index q, JacobiRotation<S>* j_left,
                                    JacobiRotation<S>* j_right) {
        Matrix<S, 2, 2> m;
        m << w.coeff(p, p), w.coeff(p, q), w.coeff(q, p), w.coeff(q, q);
        JacobiRotation<S> rot1;
        S t = m.coeff(0, 0) + m.coeff(1, 1);
        S d = m.coeff(1, 0) - m.coeff(0, 1);
        if (std::abs(d) < std::numeric_limits<S>::min()) {
            rot1.s() = S(0);
            rot1.c() = S(1);
        } else {
            S u = t / d;
            S tmp = std::sqrt(S(1) + u * u);
            rot1.s() = S(1) / tmp;
            rot1.c() = u / tmp;
        }
        internal::apply_on_the_left(m, 0, 1, rot1);
        j_right->makeJacobi(m.coeff(0, 0), m.coeff(0, 1), m.coeff(1, 1));
        *j_left = rot1 * j_right->transpose();
    }

    MatN u_ = MatN::Identity(), v_ = MatN::Identity();
    VecN sv_ = VecN::Zero();
    Index nonzero_ = 0;
    ComputationInfo info_ = Success;
};

}  // namespace Eigen
