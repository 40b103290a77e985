// lab_variants.cuh — MRG32k3a step formulations timed by tools/lab/step2_lab.cu
// and not used by the product. All give the same sequence as the integer step
// (step2_lab checks). Built on the public device header.
#pragma once
#include "../../include/shv_device.cuh"

namespace shv {
namespace dev {

// Floor-reduction FP64 component whose output word comes from the integer
// pipe instead of a DADD: r = p - k*m is exact, so r mod 2^32 =
// (a*ub - b*uc - klo*m) mod 2^32 with ub, uc the previous outputs of the
// component (their residues mod 2^32) and klo = k mod 2^32 = low word of the
// magic-rounded k' (1.5*2^52 has a zero low word). 5 FP64 + 3 IMAD.
// Component 1: p = a12*x1 - a13n*x0, w = a12*u1 - a13n*u0 + 209*klo.
__device__ __forceinline__ uint32_t c1_floor_w(double x0, double x1, uint32_t u0, uint32_t u1, double& r_out,
                                               const MrgFpK& K)
{
    const double t = __dmul_rn((double)kA13n, x0);
    const double p = __fma_rn((double)kA12, x1, -t);
    const double kk = __fma_rd(p, K.inv1, K.magic);
    r_out = __fma_rn(-__dadd_rn(kk, -K.magic), K.m1, p);
    const uint32_t klo = (uint32_t)__double2loint(kk);
    return u1 * K.a12 - u0 * K.a13n + klo * 209u;
}

// Component 2: p = a21*y2 + a23n*(m2 - y0), w = a21*v2 - a23n*v0 + 22853*(klo - a23n).
__device__ __forceinline__ uint32_t c2_floor_w(double y0, double y2, uint32_t v0, uint32_t v2, double& r_out,
                                               const MrgFpK& K)
{
    const double t = __fma_rn(-(double)kA23n, y0, K.a23n_m2);
    const double p = __fma_rn((double)kA21, y2, t);
    const double kk = __fma_rd(p, K.inv2, K.magic);
    r_out = __fma_rn(-__dadd_rn(kk, -K.magic), K.m2, p);
    const uint32_t klo = (uint32_t)__double2loint(kk);
    return v2 * kA21 - v0 * kA23n + (klo - kA23n) * 22853u;
}

// MODE bit 0: component 1 output via IMAD; bit 1: component 2 output via IMAD.
template <int MODE>
struct MrgFW {
    double x0, x1, x2, y0, y1, y2;
    uint32_t u0, u1, u2, v0, v1, v2;
};

template <int MODE>
__device__ __forceinline__ MrgFW<MODE> to_mrg_fw(const Mrg& s)
{
    return MrgFW<MODE>{__uint2double_rn(s.x0), __uint2double_rn(s.x1), __uint2double_rn(s.x2),
                       __uint2double_rn(s.y0), __uint2double_rn(s.y1), __uint2double_rn(s.y2),
                       s.x0, s.x1, s.x2, s.y0, s.y1, s.y2};
}

template <int MODE>
__device__ __forceinline__ uint32_t mrg_next(MrgFW<MODE>& s, const MrgFpK& K)
{
    double r1, r2;
    uint32_t p1, p2;
    if (MODE & 1) p1 = c1_floor_w(s.x0, s.x1, s.u0, s.u1, r1, K);
    else p1 = mrg_c1_floor(s.x0, s.x1, r1, K);
    s.x0 = s.x1; s.x1 = s.x2; s.x2 = r1;
    s.u0 = s.u1; s.u1 = s.u2; s.u2 = p1;
    if (MODE & 2) p2 = c2_floor_w(s.y0, s.y2, s.v0, s.v2, r2, K);
    else p2 = mrg_c2_floor(s.y0, s.y2, r2, K);
    s.y0 = s.y1; s.y1 = s.y2; s.y2 = r2;
    s.v0 = s.v1; s.v1 = s.v2; s.v2 = p2;
    return mrg_combine(p1, p2);
}

}  // namespace dev
}  // namespace shv
