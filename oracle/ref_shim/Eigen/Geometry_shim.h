// oracle/ref_shim/Eigen/Geometry_shim.h -- TEST INFRASTRUCTURE ONLY.
// Eigen 3.4 AngleAxis<Scalar>::toRotationMatrix (Geometry/AngleAxis.h),
// used by the reference fixtures (proj/src/synth.cpp:110,168,580) and test
// helpers (proj/tests/support/helpers.hpp:41).
#pragma once

namespace Eigen {

template <typename S>
class AngleAxis {
public:
    using Vector3 = Matrix<S, 3, 1>;
    using Matrix3 = Matrix<S, 3, 3>;
    template <EigenExpr E>
    AngleAxis(const S& angle, const E& axis) : angle_(angle), axis_(axis) {}
    S angle() const { return angle_; }
    const Vector3& axis() const { return axis_; }
    Matrix3 toRotationMatrix() const {
        Matrix3 res;
        Vector3 sin_axis = std::sin(angle_) * axis_;
        S c = std::cos(angle_);
        Vector3 cos1_axis = (S(1) - c) * axis_;
        S tmp;
        tmp = cos1_axis.x() * axis_.y();
        res.coeffRef(0, 1) = tmp - sin_axis.z();
        res.coeffRef(1, 0) = tmp + sin_axis.z();
        tmp = cos1_axis.x() * axis_.z();
        res.coeffRef(0, 2) = tmp + sin_axis.y();
        res.coeffRef(2, 0) = tmp - sin_axis.y();
        tmp = cos1_axis.y() * axis_.z();
        res.coeffRef(1, 2) = tmp - sin_axis.x();
        res.coeffRef(2, 1) = tmp + sin_axis.x();
        // res.diagonal() = (cos1_axis.cwiseProduct(m_axis)).array() + c
        for (int i = 0; i < 3; ++i) res.coeffRef(i, i) = cos1_axis.coeff(i) * axis_.coeff(i) + c;
        return res;
    }

private:
    S angle_;
    Vector3 axis_;
};

using AngleAxisd = AngleAxis<double>;
using AngleAxisf = AngleAxis<float>;

}  // namespace Eigen
