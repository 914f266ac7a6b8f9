// lk_acos_cr.hpp -- the correctly rounded acos of a double, when it is safely
// away from a rounding boundary (host and device).
//
// The reference's FPFH frame-source test (proj/src/fpfh.cpp:28) compares
// std::acos(|a1|) > std::acos(|a2|) with the host glibc (2.39 here), whose
// acos is not correctly rounded: measured against libquadmath's acosq on
// 3.2e8 arguments (uniform, cubed, and 1 - cubed), 0.08-0.12 % of its results
// differ from the correctly rounded value, every one of them with the exact
// value within 0.0219 ulp of a rounding midpoint (it returns the other
// neighbour there). So wherever the exact acos lies farther than
// kAcosSafeUlp from every midpoint, glibc returns the correctly rounded value,
// and the device can evaluate the comparison itself; only the rest goes to the
// host's libm. tests/test_acos_cr.py re-checks this premise against the glibc
// of the machine the tests run on.
//
// Method: y0 = acos(x) (device or host libm, a few ulps), one Newton step
// y = y0 + (cos(y0) - x) / sin(y0) with cos(y0) in double-double (Taylor
// series in y0^2, error ~2^-100 absolute), y0 + d split exactly by two-sum
// into the rounded value and its remainder, whose distance to half an ulp is
// the distance to the nearest midpoint. Needs IEEE arithmetic without
// contraction (the product build: -fmad=false / -ffp-contract=off) and a
// correctly rounded fma.
#pragma once

#include <cmath>

#ifdef __CUDACC__
#define LK_ACOS_HD __host__ __device__ __forceinline__
#else
#define LK_ACOS_HD inline
#endif

namespace lkacos {

constexpr double kAcosSafeUlp = 0.05;  // 2.3x the largest deviation measured

struct DD {
    double hi, lo;
};

LK_ACOS_HD DD two_sum(double a, double b) {
    const double s = a + b, bb = s - a;
    return {s, (a - (s - bb)) + (b - bb)};
}
LK_ACOS_HD DD quick_two_sum(double a, double b) {
    const double s = a + b;
    return {s, b - (s - a)};
}
LK_ACOS_HD DD dd_mul(DD a, DD b) {
    const double p = a.hi * b.hi;
    double e = fma(a.hi, b.hi, -p);
    e += a.hi * b.lo + a.lo * b.hi;
    return quick_two_sum(p, e);
}
LK_ACOS_HD DD dd_add(DD a, DD b) {
    DD s = two_sum(a.hi, b.hi);
    const DD t = two_sum(a.lo, b.lo);
    s.lo += t.hi;
    s = quick_two_sum(s.hi, s.lo);
    s.lo += t.lo;
    return quick_two_sum(s.hi, s.lo);
}

// cos(y) in double-double for 0 <= y <= 1.6: sum_k (-1)^k y^2k / (2k)!
LK_ACOS_HD DD cos_dd(double y) {
    // (-1)^k / (2k)! as double-doubles, k = 0..18 (the k = 19 term is < 2^-110)
    const double c[19][2] = {
        {1.0, 0.0},
        {-0.5, 0.0},
        {0.041666666666666664, 2.3129646346357427e-18},
        {-0.001388888888888889, 5.300543954373577e-20},
        {2.48015873015873e-05, 2.1511947866775882e-23},
        {-2.755731922398589e-07, -2.3767714622250297e-23},
        {2.08767569878681e-09, -1.20734505911326e-25},
        {-1.1470745597729725e-11, -2.0655512752830745e-28},
        {4.779477332387385e-14, 4.399205485834081e-31},
        {-1.5619206968586225e-16, -1.1910679660273754e-32},
        {4.110317623312165e-19, 1.4412973378659527e-36},
        {-8.896791392450574e-22, 7.911402614872376e-38},
        {1.6117375710961184e-24, -3.6846573564509766e-41},
        {-2.4795962632247976e-27, 1.2953730964765229e-43},
        {3.279889237069838e-30, 1.5117542744029879e-46},
        {-3.7699876288159054e-33, -2.5870347832750324e-49},
        {3.8003907548547434e-36, 1.7457158024652518e-52},
        {-3.387157535521162e-39, -5.09056148151085e-56},
        {2.6882202662866363e-42, 5.355061165943334e-59},
    };
    const double t = y * y;
    const DD t2{t, fma(y, y, -t)};
    DD p{c[18][0], c[18][1]};
    for (int k = 17; k >= 0; --k) p = dd_add(dd_mul(p, t2), DD{c[k][0], c[k][1]});
    return p;
}

// What glibc's acos(x) can return, for 0 <= x <= 1: 1 with *lo = *hi = the
// correctly rounded value when the exact value is at least kAcosSafeUlp from
// a rounding midpoint; 2 with *lo < *hi the two neighbours of the midpoint it
// is close to; 0 when unknown (x outside [0, 1], NaN, x within ~5e-7 of 1 --
// left to the caller's libm).
LK_ACOS_HD int acos_bracket(double x, double* lo, double* hi) {
    if (x == 1.0) {
        *lo = *hi = 0.0;
        return 1;
    }
    if (!(x >= 0.0 && x < 1.0)) return 0;
    const double y0 = acos(x);
    if (!(y0 >= 1e-3 && y0 <= 1.6)) return 0;
    const DD cy = cos_dd(y0);
    // cos(y0) - x, then the Newton correction d = y - y0
    const DD r = dd_add(cy, DD{-x, 0.0});
    const double d = r.hi / sin(y0);
    const DD s = two_sum(y0, d);
    const double up = nextafter(s.hi, 2.0), dn = nextafter(s.hi, 0.0);
    if (!(fabs(d) <= 8.0 * (up - s.hi))) return 0;  // y0 farther off than libm promises
    const double ulp = s.lo >= 0.0 ? up - s.hi : s.hi - dn;
    if (0.5 - fabs(s.lo) / ulp >= kAcosSafeUlp) {
        *lo = *hi = s.hi;
        return 1;
    }
    *lo = s.lo >= 0.0 ? s.hi : dn;
    *hi = s.lo >= 0.0 ? up : s.hi;
    return 2;
}

// The correctly rounded acos(x) when glibc certainly returns it.
LK_ACOS_HD bool acos_cr(double x, double* out) {
    double lo, hi;
    if (acos_bracket(x, &lo, &hi) != 1) return false;
    *out = lo;
    return true;
}

// glibc's acos(x1) > acos(x2): 1 / 0 when certain, 2 when it depends on how
// glibc rounds near a midpoint (or is unknown).
LK_ACOS_HD int acos_greater(double x1, double x2) {
    double l1, h1, l2, h2;
    if (!acos_bracket(x1, &l1, &h1) || !acos_bracket(x2, &l2, &h2)) return 2;
    if (l1 > h2) return 1;
    if (h1 <= l2) return 0;
    return 2;
}

}  // namespace lkacos
