// lab_variants.cuh — MRG32k3a step formulations measured by tools/lab/step_lab.cu
// and not used by the product (DESIGN.md §11 records their rates). Built on the
// public device header.
#pragma once
#include "../../include/shv_device.cuh"

namespace shv {
namespace dev {

// Hybrid state: component 2 held as exact binary64 integers.
struct MrgH {
    uint32_t x0, x1, x2;
    double y0, y1, y2;
};

__device__ __forceinline__ MrgH to_hybrid(const Mrg& s)
{
    return MrgH{s.x0, s.x1, s.x2, __uint2double_rn(s.y0), __uint2double_rn(s.y1), __uint2double_rn(s.y2)};
}

// Same result with a shorter dependency chain on the recurrence input yb:
// q = fma(RN(a/m), yb, RN(-b*yc/m)) approximates p/m to within 2^-31, so
// k = rint(q) (one FRND) keeps |p/m - k| <= 1/2 + 2^-31; the chain from yb to
// r is fma -> rint -> fma instead of fma -> fma -> add -> fma.
template <uint32_t M, uint32_t A, uint32_t B>
__device__ __forceinline__ uint32_t mrg_fp64_short(double yb, double yc, double& r_out)
{
    const double kMagic = 6755399441055744.0;  // 1.5 * 2^52
    const double t = __dmul_rn((double)B, yc);
    const double c0 = __dmul_rn(t, -1.0 / (double)M);
    const double p = __fma_rn((double)A, yb, -t);
    const double q = __fma_rn((double)A / (double)M, yb, c0);
    double k;
    asm("cvt.rni.f64.f64 %0, %1;" : "=d"(k) : "d"(q));
    const double r = __fma_rn(-k, (double)M, p);
    r_out = r;
    uint32_t w = (uint32_t)__double2loint(__dadd_rn(r, kMagic));  // r mod 2^32
    asm("{\n\t.reg .pred n;\n\tsetp.lt.s32 n, %0, 0;\n\t@n add.u32 %0, %0, %1;\n\t}" : "+r"(w) : "n"(M));
    return w;
}

__device__ __forceinline__ uint32_t mrg_next(MrgH& s)
{
    const uint32_t p1 = mrg_c1(s.x0, s.x1);
    s.x0 = s.x1;
    s.x1 = s.x2;
    s.x2 = p1;
    double r;
    const uint32_t p2 = mrg_c2_fp64(s.y0, s.y2, r);
    s.y0 = s.y1;
    s.y1 = s.y2;
    s.y2 = r;
    return mrg_combine(p1, p2);
}

// Both components on the FP64 pipe, short-chain form (lab variant).
struct MrgS {
    double x0, x1, x2;
    double y0, y1, y2;
    int pad;
};

__device__ __forceinline__ MrgS to_fp64s(const Mrg& s)
{
    return MrgS{__uint2double_rn(s.x0), __uint2double_rn(s.x1), __uint2double_rn(s.x2),
                __uint2double_rn(s.y0), __uint2double_rn(s.y1), __uint2double_rn(s.y2), 0};
}

__device__ __forceinline__ uint32_t mrg_next(MrgS& s)
{
    double r1, r2;
    const uint32_t p1 = mrg_fp64_short<kM1, kA12, kA13n>(s.x1, s.x0, r1);
    s.x0 = s.x1;
    s.x1 = s.x2;
    s.x2 = r1;
    const uint32_t p2 = mrg_fp64_short<kM2, kA21, kA23n>(s.y2, s.y0, r2);
    s.y0 = s.y1;
    s.y1 = s.y2;
    s.y2 = r2;
    return mrg_combine(p1, p2);
}

// Both components on the FP64 pipe with the output word computed on the
// integer pipe (lab variant "W"): r mod 2^32 = a*wb - b*wc - k*m (mod 2^32),
// where wb, wc are the previous outputs' residues mod 2^32 and k's low word is
// read off the magic-rounded k' (k' = 1.5*2^52 + k, ulp 1). 5 FP64 ops and
// 3 IMAD per component instead of 6 FP64 ops.
template <uint32_t M, uint32_t A, uint32_t B>
__device__ __forceinline__ uint32_t mrg_fp64w(double yb, double yc, uint32_t wb, uint32_t wc, double& r_out,
                                              uint32_t& w_out)
{
    const double kMagic = 6755399441055744.0;  // 1.5 * 2^52
    const double t = __dmul_rn((double)B, yc);
    const double p = __fma_rn((double)A, yb, -t);
    const double kk = __fma_rn(p, 1.0 / (double)M, kMagic);
    const double r = __fma_rn(-__dadd_rn(kk, -kMagic), (double)M, p);
    r_out = r;
    const uint32_t klo = (uint32_t)__double2loint(kk);
    uint32_t w = wb * A - wc * B - klo * M;
    w_out = w;
    asm("{\n\t.reg .pred n;\n\tsetp.lt.s32 n, %0, 0;\n\t@n add.u32 %0, %0, %1;\n\t}" : "+r"(w) : "n"(M));
    return w;
}

struct MrgW {
    double x0, x1, x2;
    double y0, y1, y2;
    uint32_t u0, u1, u2, v0, v1, v2;  // the same residues mod 2^32
};

__device__ __forceinline__ MrgW to_fp64w(const Mrg& s)
{
    return MrgW{__uint2double_rn(s.x0), __uint2double_rn(s.x1), __uint2double_rn(s.x2),
                __uint2double_rn(s.y0), __uint2double_rn(s.y1), __uint2double_rn(s.y2),
                s.x0, s.x1, s.x2, s.y0, s.y1, s.y2};
}

__device__ __forceinline__ uint32_t mrg_next(MrgW& s)
{
    double r1, r2;
    uint32_t w1, w2;
    const uint32_t p1 = mrg_fp64w<kM1, kA12, kA13n>(s.x1, s.x0, s.u1, s.u0, r1, w1);
    s.x0 = s.x1; s.x1 = s.x2; s.x2 = r1;
    s.u0 = s.u1; s.u1 = s.u2; s.u2 = w1;
    const uint32_t p2 = mrg_fp64w<kM2, kA21, kA23n>(s.y2, s.y0, s.v2, s.v0, r2, w2);
    s.y0 = s.y1; s.y1 = s.y2; s.y2 = r2;
    s.v0 = s.v1; s.v1 = s.v2; s.v2 = w2;
    return mrg_combine(p1, p2);
}

// Lab variants of the all-FP64 step: V=2 mask-add decode, V=3 mask-add decode
// with cvt.rni.s32.f64 instead of the magic-add conversion, V=4 decode via
// IMAD ((w >> 31) * -m + w).
template <uint32_t M, uint32_t A, uint32_t B, int V>
__device__ __forceinline__ uint32_t mrg_fp64v(double yb, double yc, double& r_out)
{
    const double kMagic = 6755399441055744.0;  // 1.5 * 2^52
    const double t = __dmul_rn((double)B, yc);
    const double p = __fma_rn((double)A, yb, -t);
    const double k = __dadd_rn(__fma_rn(p, 1.0 / (double)M, kMagic), -kMagic);
    const double r = __fma_rn(-k, (double)M, p);
    r_out = r;
    uint32_t w;
    if (V == 3) {
        int32_t i;
        asm("cvt.rni.s32.f64 %0, %1;" : "=r"(i) : "d"(r));
        w = (uint32_t)i;
    } else {
        w = (uint32_t)__double2loint(__dadd_rn(r, kMagic));
    }
    if (V == 4) return (uint32_t)((int32_t)w >> 31) * (0u - M) + w;
    return w + ((uint32_t)((int32_t)w >> 31) & M);
}

template <int V>
struct MrgDV {
    double x0, x1, x2;
    double y0, y1, y2;
    char pad[8 * V];
};

template <int V>
__device__ __forceinline__ MrgDV<V> to_fp64v(const Mrg& s)
{
    MrgDV<V> d;
    d.x0 = __uint2double_rn(s.x0); d.x1 = __uint2double_rn(s.x1); d.x2 = __uint2double_rn(s.x2);
    d.y0 = __uint2double_rn(s.y0); d.y1 = __uint2double_rn(s.y1); d.y2 = __uint2double_rn(s.y2);
    return d;
}

template <int V>
__device__ __forceinline__ uint32_t mrg_next(MrgDV<V>& s)
{
    double r1, r2;
    const uint32_t p1 = mrg_fp64v<kM1, kA12, kA13n, V>(s.x1, s.x0, r1);
    s.x0 = s.x1; s.x1 = s.x2; s.x2 = r1;
    const uint32_t p2 = mrg_fp64v<kM2, kA21, kA23n, V>(s.y2, s.y0, r2);
    s.y0 = s.y1; s.y1 = s.y2; s.y2 = r2;
    return mrg_combine(p1, p2);
}

}  // namespace dev
}  // namespace shv
