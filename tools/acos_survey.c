// tools/acos_survey.c -- how far glibc's acos is from correctly rounded
// (the premise of paper_1801_01572_b200/csrc/lk_acos_cr.hpp): N arguments
// (uniform on [0, 1), cubed, and 1 - cubed, a third each), glibc acos against
// libquadmath's acosq rounded to double; prints the mismatch count and the
// largest distance of a mismatching exact value from its rounding midpoint.
//
//   gcc -O2 -o /tmp/acos_survey tools/acos_survey.c -lquadmath -lm
//   /tmp/acos_survey 300000000   # here: 0.12 %, max 0.02183 ulp (glibc 2.39)
#include <math.h>
#include <quadmath.h>
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
static uint64_t s = 0x9e3779b97f4a7c15ull;
static uint64_t nx(void){ s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
int main(int argc, char** argv) {
    long N = argc > 1 ? atol(argv[1]) : 10000000;
    long mism = 0;
    double maxd = 0;
    for (long k = 0; k < N; ++k) {
        double x = (double)(nx() >> 11) * 0x1p-53;  // [0,1)
        if (k % 3 == 1) x = x * x * x; else if (k % 3 == 2) x = 1.0 - x * x * x;                    // more small values
        double g = acos(x);
        __float128 y = acosq((__float128)x);
        double c = (double)y;                        // RN
        // distance of y to nearest midpoint, in ulps of c
        double up = nextafter(c, 2.0), dn = nextafter(c, 0.0);
        __float128 m1 = ((__float128)c + (__float128)up) / 2, m0 = ((__float128)c + (__float128)dn) / 2;
        __float128 d1 = m1 - y, d0 = y - m0;
        __float128 dm = d1 < d0 ? d1 : d0;
        double ulp = up - c;
        double dist = (double)(dm / ulp);
        if (g != c) { ++mism; if (dist > maxd) maxd = dist; }
    }
    printf("N %ld mismatches %ld (%.4g%%) max midpoint distance of a mismatch %.5f ulp\n", N, mism, 100.0 * mism / N, maxd);
    return 0;
}
