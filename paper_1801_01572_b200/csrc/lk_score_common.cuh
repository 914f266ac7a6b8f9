// lk_score_common.cuh -- device helpers shared by the scoring kernels
// (lk_hypotheses.cu) and ICP (lk_icp.cu): the FP32 image of a rigid transform
// in fine-cell units with its guard bands, and the FP32 top-3 scan step.
#pragma once

#include <cstdint>

#include "lk_device_math.cuh"
#include "lk_kernels.cuh"

namespace lkk {

struct FastRT {
    float r[9];    // R / cell
    float t[3];    // (t - o) / cell - off
    float eps;     // guard on cell-coordinate fractions (cells)
    float band;    // guard on d2 (squared cells)
    float ok;      // 1: fast path usable for this candidate
    float pad;
};
static_assert(sizeof(FastRT) == 64, "FastRT layout");

// ---- FP32 image in fine-cell units ------------------------------------------
// FP32 image of (R, t) in fine-cell units (cell / 2, offset 2 off) with the
// same guard-band construction as make_fast.
__device__ __forceinline__ FastRT make_fast_fine(const double* R, const double* t, const GridView& g,
                                                 const ScoreParams& sp) {
    FastRT f;
#pragma unroll
    for (int k = 0; k < 9; ++k) f.r[k] = static_cast<float>(R[k] / g.fcell);
    f.t[0] = static_cast<float>((t[0] - g.ox) / g.fcell - 2 * g.offx);
    f.t[1] = static_cast<float>((t[1] - g.oy) / g.fcell - 2 * g.offy);
    f.t[2] = static_cast<float>((t[2] - g.oz) / g.fcell - 2 * g.offz);
    const float u = 5.9604645e-8f;
    const float tn = sqrtf(f.t[0] * f.t[0] + f.t[1] * f.t[1] + f.t[2] * f.t[2]);
    const float dq = u * (5.0f * 2.0f * sp.pmax_cells + 4.0f * tn + 4.0f);
    const float de = u * (2.0f * sp.nmax_cells + 2.0f);
    const float delta = dq + de;
    const float thr = static_cast<float>((sp.d_max / g.fcell) * (sp.d_max / g.fcell));
    f.eps = 4.0f * dq + 1e-6f;
    // d2 within sqrt(thr) + 1 fine cells: error <= 2 sqrt3 (sqrt(thr) + 1) delta + 3 delta^2 (+ FP32 rounding)
    f.band = 4.0f * (3.5f * (sqrtf(thr) + 1.0f) * delta + 3.0f * delta * delta + 16.0f * u * (thr + 1.0f)) + 1e-7f;
    f.ok = (sp.fast && g.fine_info && sp.d_max <= g.fine_dmax && f.eps < 0.02f && f.band < 0.05f) ? 1.0f : 0.0f;
    f.pad = thr;  // d2_max in squared fine-cell units
    return f;
}

__device__ __forceinline__ void top3(float d2, int32_t o, float& f1, float& f2, float& f3, int32_t& o1, int32_t& o2) {
    if (d2 < f1) {
        f3 = f2;
        f2 = f1;
        o2 = o1;
        f1 = d2;
        o1 = o;
    } else if (d2 < f2) {
        f3 = f2;
        f2 = d2;
        o2 = o;
    } else if (d2 < f3) {
        f3 = d2;
    }
}

// Guard of the FP32 normal gate, relative to |ns|_1 |nt|_1: the FP32 value of
// (R ns) . nt is within ~14 u |ns|_1 |nt|_1 (u = 2^-24) of the exact one.
constexpr float kGateGuard = 1e-5f;

}  // namespace lkk
