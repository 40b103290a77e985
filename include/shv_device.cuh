// shv_device.cuh — device-side generator primitives of the ShoveRand hot path
// (arXiv 1412.8266) for sm_100a. Included by the kernels_*.cu files (and by the
// kernel labs under tools/lab/, which time variants of the same functions).
//
// MRG32k3a steps, all exact and bit-identical:
//  - MrgMF: the state as FP64 pairs {x, 0} in the subnormal range (the double
//    x * 2^-1074, whose bit pattern is x and whose ulp is 2^-1074): per
//    component the exact product sum, one round-down multiply that IS the pair
//    D(floor(p/m)), and one FMA that IS the next state pair D(p - k m): 4 FP64
//    instructions, no integer or move instructions. The product step of the
//    row-tile, stream-per-lane and vector fills, the fused Monte Carlo kernel
//    and the device API (1.91 T values/s compute-only, lab65).
//  - MrgSN: the same representation with magic-number quotients and integer
//    residues (3 DFMA + 1 IMAD + a zero move per component; 1.71 T/s, lab47).
//  - MrgIF: component 1 in 32-bit integer arithmetic (two IMAD.WIDE + one IMAD,
//    compare/select on the ALU), component 2 in exact binary64 arithmetic on
//    the FP64 pipe (products < 2^53, floor reduction), as in L'Ecuyer's
//    floating-point formulation [LEcuyer1999]. The transposed Leap Frog fill.
//  - MrgFF: both components on the FP64 pipe (12 FP64 operations per number);
//    the scalar (ragged-shape) fill.
// Measured on B200 (tools/lab, profiles/r02_labs): IMAD.WIDE issues at ~21-24
// per SM per clock (about 6 issue cycles per warp instruction) and slows the
// other kinds it shares the SM with, so MrgIF costs about the sum of its two
// halves (1.44 T values/s compute-only vs 1.33 for MrgFF).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace shv {
namespace dev {

// [LEcuyer1999] MRG32k3a parameters (PAPER.md L255 cites them; not restated there).
constexpr uint32_t kM1 = 4294967087u;  // 2^32 - 209
constexpr uint32_t kM2 = 4294944443u;  // 2^32 - 22853
constexpr uint32_t kC1 = 209u;
constexpr uint32_t kC2 = 22853u;
constexpr uint32_t kA12 = 1403580u;
constexpr uint32_t kA13n = 810728u;
constexpr uint32_t kA21 = 527612u;
constexpr uint32_t kA23n = 1370589u;
// [Salmon.etal.2011] Philox4x32 multipliers and Weyl key increments.
constexpr uint32_t kPM0 = 0xD2511F53u;
constexpr uint32_t kPM1 = 0xCD9E8D57u;
constexpr uint32_t kPW0 = 0x9E3779B9u;
constexpr uint32_t kPW1 = 0xBB67AE85u;

// ------------------------------------------------------------------ integer helpers

// 64-bit + 32-bit on the ALU pipe (add.cc/addc -> IADD3 with carry), keeping
// index arithmetic off the FMA-heavy pipe that the generators saturate.
__device__ __forceinline__ uint64_t add64(uint64_t a, uint32_t b)
{
    uint32_t lo, hi;
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, 0;"
        : "=r"(lo), "=r"(hi)
        : "r"((uint32_t)a), "r"(b), "r"((uint32_t)(a >> 32)));
    return ((uint64_t)hi << 32) | lo;
}

// x mod (2^32 - c) for any 64-bit x (c < 2^15): two folds + one subtraction.
template <uint32_t C>
__device__ __forceinline__ uint32_t red64(uint64_t x)
{
    x = (x >> 32) * C + (uint32_t)x;  // < 2^47.1
    x = (x >> 32) * C + (uint32_t)x;  // < 2^32 + 2^30
    const uint64_t m = (1ull << 32) - C;
    return (uint32_t)(x >= m ? x - m : x);
}

// r = M v (mod m = 2^32 - C), M row-major 3x3 with entries < m, v canonical.
// Each product t = M_kj v_j < m^2 folds once to hi(t)*C + lo(t) < 2^46.5
// (C <= 22853 < 2^14.48); the three folded terms sum to < 2^48.1, whose high
// word h < 2^16.1 folds into V = lo + h*C < 2^32 + 2^30.6 < 2m: u = V mod 2^32
// (one 32-bit IMAD), V >= 2^32 exactly when u < lo, and V mod m = u + C (mod
// 2^32) when V >= 2^32 or u >= m, else u. 7 IMAD.WIDE + ~5 other per row.
template <uint32_t C>
__device__ __forceinline__ void matvec(const uint32_t* M, uint32_t& v0, uint32_t& v1, uint32_t& v2)
{
    uint32_t r[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        uint64_t f = 0;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const uint64_t t = (uint64_t)M[3 * k + j] * (j == 0 ? v0 : j == 1 ? v1 : v2);
            f += (t >> 32) * C + (uint32_t)t;
        }
        const uint32_t lo = (uint32_t)f, hi = (uint32_t)(f >> 32);
        const uint32_t u = hi * C + lo;
        r[k] = ((u < lo) | (u >= 0u - C)) ? u + C : u;
    }
    v0 = r[0];
    v1 = r[1];
    v2 = r[2];
}

// ------------------------------------------------------------------ MRG32k3a

// Integer state (used for jumps, seeding and the reference step).
struct Mrg {
    uint32_t x0, x1, x2;  // component 1, oldest -> newest (R1)
    uint32_t y0, y1, y2;  // component 2
};

__device__ __forceinline__ void apply(const uint32_t* a, const uint32_t* b, Mrg& s)
{
    matvec<kC1>(a, s.x0, s.x1, s.x2);
    matvec<kC2>(b, s.y0, s.y1, s.y2);
}

// Constants of the step. The kernels pass a copy read from their launch
// parameters (or constant memory), so ptxas cannot constant-fold them: the
// integer multipliers then stay plain IMAD.WIDE operands (with immediates
// ptxas strength-reduces a13n*(m1 - x0) into IMAD/IMAD.HI/IADD3.X chains, 26
// instead of 16 issue slots per number), and the non-immediate doubles stay
// in (uniform) registers instead of being re-materialised inside the loop.
// The device API (shv_rng.cuh) uses mrg_fpk() (immediates: same values).
struct MrgFpK {
    double magic;   // 1.5 * 2^52: ulp 1 on [2^52, 2^53)
    double inv1;    // RN(1/m1) = 1/m1 + delta1, 0 < delta1 < 0.34 ulp
    double inv2;    // RU(1/m2) = 1/m2 + delta2, 0 < delta2 < 0.54 ulp
    double m1, m2;
    double a23n_m2; // a23n * m2 = 5886603609186927, exact
    uint32_t a12, a13n;  // component-1 multipliers for the integer half-step
    // Subnormal-state steps (MrgSN; MrgMF uses sn_c2p): constants in units of 2^-1074 and the
    // scaled inverses; the kernels overwrite them from their launch parameters.
    double sn_c1q = 0x0.317b9fd79a126p-1022;  // D(202682 * m1)
    double sn_c2p = 0x1.4e9d5b50f226fp-1022;  // D(a23n * m2)
    double sn_c1s = 0x1.000000d10000bp+980;   // 4 * RN(1/m1) * 2^1010
    double sn_c2s = 0x1.000059451f212p+978;   // RU(1/m2) * 2^1010
    double sn_M = 0x1.8p-12;                  // 1.5 * 2^-12: ulp 2^-64
};
__host__ __device__ __forceinline__ constexpr MrgFpK mrg_fpk()
{
    return MrgFpK{6755399441055744.0, 1.0 / (double)kM1, 0x1.000059451f212p-32,
                  (double)kM1, (double)kM2, (double)kA23n * (double)kM2, kA12, kA13n};
}

// Component 1, integer: x_{1,n} = (a12 x_{1,n-2} - a13n x_{1,n-3}) mod m1 for
// canonical x0 = x_{1,n-3}, x1 = x_{1,n-2} < m1:
//   P = a12*x1 + a13n*(m1 - x0) <= 2214308*m1 < 2^53.1 (two IMAD.WIDE.U32),
//   P = H*2^32 + L with H <= 2214307, so 209*H < 2^28.8;
//   V = L + 209*H == P (mod m1, 2^32 = 209), V < 2^32 + 2^28.8;
//   u = V mod 2^32 (one 32-bit IMAD); V >= 2^32 exactly when u < L;
//   if V >= 2^32: V - m1 = u + 209 (< m1); else if u >= m1: u - m1 = u + 209
//   (mod 2^32); else u. So p1 = (u < L or u >= m1) ? u + 209 : u.
// Bounds pinned in tests/test_fp64_step_bounds.py. a12, a13n arrive in
// registers (MrgFpK): 7 instructions, 2 IMAD.WIDE + IMAD + 4 ALU-class.
__device__ __forceinline__ uint32_t mrg_c1_int(uint32_t x0, uint32_t x1, uint32_t a12, uint32_t a13n)
{
    uint32_t r;
    asm("{\n\t"
        ".reg .u64 q;\n\t"
        ".reg .u32 t, l, h;\n\t"
        ".reg .pred c;\n\t"
        "sub.u32 t, 4294967087, %1;\n\t"          // m1 - x0
        "mul.wide.u32 q, %2, %3;\n\t"             // a12*x1
        "mad.wide.u32 q, t, %4, q;\n\t"           // P = (H, L)
        "mov.b64 {l, h}, q;\n\t"
        "mad.lo.u32 %0, h, 209, l;\n\t"           // u = L + 209*H mod 2^32
        "setp.lt.u32 c, %0, l;\n\t"               // V >= 2^32
        "setp.ge.or.u32 c, %0, 4294967087, c;\n\t"
        "@c add.u32 %0, %0, 209;\n\t"
        "}"
        : "=r"(r)
        : "r"(x0), "r"(x1), "r"(a12), "r"(a13n));
    return r;
}

// Component 2, integer (reference / seeding path): Q = a21*y2 + a23n*(m2-y0)
// < 2^52.9 folded twice with 2^32 = 22853 (mod m2).
__device__ __forceinline__ uint32_t mrg_c2_int(uint32_t y0, uint32_t y2)
{
    const uint64_t q = (uint64_t)kA21 * y2 + (uint64_t)kA23n * (kM2 - y0);
    const uint64_t t = (uint64_t)(uint32_t)(q >> 32) * kC2 + (uint32_t)q;
    const uint32_t tlo = (uint32_t)t;
    const uint32_t r2 = tlo + (uint32_t)(t >> 32) * kC2;
    return r2 + ((r2 < tlo) | (r2 >= kM2) ? kC2 : 0u);
}

// Combination (R2): (p1 - p2) mod m1 with 0 -> m1, exact in wrap-around.
__device__ __forceinline__ uint32_t mrg_combine(uint32_t p1, uint32_t p2)
{
    uint32_t z;
    asm("{\n\t.reg .pred le;\n\t"
        "sub.u32 %0, %1, %2;\n\t"
        "setp.le.u32 le, %1, %2;\n\t"
        "@le add.u32 %0, %0, 4294967087;\n\t}"
        : "=r"(z)
        : "r"(p1), "r"(p2));
    return z;
}

// All-integer step (reference; the lab's variant 0).
__device__ __forceinline__ uint32_t mrg_next(Mrg& s, const MrgFpK& K = mrg_fpk())
{
    const uint32_t p1 = mrg_c1_int(s.x0, s.x1, K.a12, K.a13n);
    s.x0 = s.x1;
    s.x1 = s.x2;
    s.x2 = p1;
    const uint32_t p2 = mrg_c2_int(s.y0, s.y2);
    s.y0 = s.y1;
    s.y1 = s.y2;
    s.y2 = p2;
    return mrg_combine(p1, p2);
}

// Component 2 on the FP64 pipe with a floor reduction, no decode. For a
// canonical state (y < m2) the positive form p = a21*y2 + a23n*(m2 - y0) lies
// in [0, 2^52.86), exact in binary64 (t = fma(-a23n, y0, a23n*m2) and
// p = fma(a21, y2, t) are exact integers). With inv2 = RU(1/m2) =
// 1/m2 + delta, 0 < delta < 0.54 ulp, p*delta*m2 < 0.97 for every such p, so
// floor(p*inv2) = floor(p/m2) exactly; fma.rm(p, inv2, 1.5*2^52) returns
// 1.5*2^52 + floor(p/m2) (ulp 1 there). r = p - k*m2 is then the canonical
// residue in [0, m2): it is both the next state word (canonical again, so the
// bound holds at every step) and, as the low word of r + 1.5*2^52, the
// component's output, with no sign fix-up. 6 FP64 operations, 0 integer.
__device__ __forceinline__ uint32_t mrg_c2_floor(double y0, double y2, double& r_out, const MrgFpK& K)
{
    const double t = __fma_rn(-(double)kA23n, y0, K.a23n_m2);  // a23n*(m2 - y0)
    const double p = __fma_rn((double)kA21, y2, t);
    const double k = __dadd_rn(__fma_rd(p, K.inv2, K.magic), -K.magic);
    const double r = __fma_rn(-k, K.m2, p);
    r_out = r;
    return (uint32_t)__double2loint(__dadd_rn(r, K.magic));
}

// Component 1 on the FP64 pipe with a floor reduction. The signed form
// p = a12*x1 - a13n*x0 satisfies |p| < 2^52.42 for states in [0, m1]. With
// kInv = RN(1/m1) = 1/m1 + delta, 0 < delta < 0.34 ulp, |p|*delta*m1 < 0.45,
// so floor(p*kInv) = floor(p/m1) except when p = k*m1 exactly with p < 0,
// where it is k - 1 and r = m1 (= 0 mod m1). r is therefore in [0, m1], a
// valid state word, and the output r (low word of r + 1.5*2^52) equals p1 or,
// only when p1 = 0, m1 — which mrg_combine maps to the same z (p1 - p2 + m1 if
// p1 <= p2 gives m1 - p2 for p1 = 0; m1 - p2 > 0 for p1 = m1). 6 FP64 ops.
__device__ __forceinline__ uint32_t mrg_c1_floor(double x0, double x1, double& r_out, const MrgFpK& K)
{
    const double t = __dmul_rn((double)kA13n, x0);
    const double p = __fma_rn((double)kA12, x1, -t);
    const double k = __dadd_rn(__fma_rd(p, K.inv1, K.magic), -K.magic);
    const double r = __fma_rn(-k, K.m1, p);
    r_out = r;
    return (uint32_t)__double2loint(__dadd_rn(r, K.magic));
}

// Both components on the FP64 pipe with floor reductions: 12 FP64 ops and the
// 3-instruction combine per number (round-1 product step; FP64-bound at
// 24 pipe cycles per warp and number).
struct MrgFF {
    double x0, x1, x2;
    double y0, y1, y2;
};

__device__ __forceinline__ MrgFF to_mrg_ff(const Mrg& s)
{
    return MrgFF{__uint2double_rn(s.x0), __uint2double_rn(s.x1), __uint2double_rn(s.x2),
                 __uint2double_rn(s.y0), __uint2double_rn(s.y1), __uint2double_rn(s.y2)};
}

__device__ __forceinline__ uint32_t mrg_next(MrgFF& s, const MrgFpK& K = mrg_fpk())
{
    double r1, r2;
    const uint32_t p1 = mrg_c1_floor(s.x0, s.x1, r1, K);
    s.x0 = s.x1;
    s.x1 = s.x2;
    s.x2 = r1;
    const uint32_t p2 = mrg_c2_floor(s.y0, s.y2, r2, K);
    s.y0 = s.y1;
    s.y1 = s.y2;
    s.y2 = r2;
    return mrg_combine(p1, p2);
}

// The product's MRG32k3a step: component 1 in integer arithmetic (mrg_c1_int:
// 2 IMAD.WIDE + IMAD on the FMA-heavy pipe, compare/select on the ALU),
// component 2 on the FP64 pipe (mrg_c2_floor: 6 ops), combine on the ALU (3):
// 16 issue slots per number with the FMA-heavy, ALU and FP64 pipes each at
// ~12 cycles per warp, instead of 24 FP64 cycles for MrgFF.
struct MrgIF {
    uint32_t x0, x1, x2;
    double y0, y1, y2;
};

__device__ __forceinline__ MrgIF to_mrg_if(const Mrg& s)
{
    return MrgIF{s.x0, s.x1, s.x2, __uint2double_rn(s.y0), __uint2double_rn(s.y1), __uint2double_rn(s.y2)};
}

__device__ __forceinline__ uint32_t mrg_next(MrgIF& s, const MrgFpK& K = mrg_fpk())
{
    const uint32_t p1 = mrg_c1_int(s.x0, s.x1, K.a12, K.a13n);
    s.x0 = s.x1;
    s.x1 = s.x2;
    s.x2 = p1;
    double r;
    const uint32_t p2 = mrg_c2_floor(s.y0, s.y2, r, K);
    s.y0 = s.y1;
    s.y1 = s.y2;
    s.y2 = r;
    return mrg_combine(p1, p2);
}

// The product's MRG32k3a step since round 2b: the state as the FP64 pairs
// D(x) = {x, 0}, i.e. x * 2^-1074 in the SUBNORMAL range.
// For an integer v in [0, 2^53) the bit pattern of D(v) is v itself (the
// subnormal/normal boundary at 2^52 is seamless: exponent field 1 = bit 52),
// so a product sum p formed exactly on the FP64 pipe hands p mod 2^32 to the
// integer pipes as its low word, and the floor quotient
// Q = fma.rm(p, inv * 2^1010, 1.5 * 2^-12) = 1.5 * 2^-12 + floor(p / m) * 2^-64
// hands k = floor(p / m) < 2^22 as its low word. The canonical residue is then
// r = p - k m = lo(p) + c k (mod 2^32), m = 2^32 - c: one IMAD, no bias, no
// conversion, no fix-up. Per component 3 DFMA + 1-2 integer instructions:
//  - component 2: p = a21 y2 + a23n (m2 - y0) in [0, 2^52.86) (exact), the
//    floor by inv2 = RU(1/m2) exactly as in mrg_c2_floor;
//  - component 1: the signed form has negative values (sign-magnitude bits)
//    and the positive form a12 x1 + a13n (m1 - x0) reaches 2^53.08, so the
//    common factor 4 comes out: q = 350895 x1 + 202682 (m1 - x0) < 2^51.08 is
//    exact, p = 4q, floor(4q / m1) = floor(q * 4 inv1) because
//    4q * delta1 * m1 < 0.72 (inv1 = RN(1/m1) = 1/m1 + delta1, delta1 > 0),
//    and r = 4 lo(q) + 209 k (mod 2^32).
// Bounds pinned in tests/test_fp64_step_bounds.py. Compute-only on B200
// (tools/lab/step4_lab.cu, lab47): 1.71 T numbers/s against 1.42 for MrgIF
// and 1.34 for MrgFF: 6 DFMA, 3 IMAD, 1 shift, 2 zero moves (the pairs' high
// words) and the 3-instruction combine per number.
struct MrgSN {
    uint32_t x0, x1, x2;  // component 1, oldest -> newest (canonical, < m1)
    uint32_t y0, y1, y2;  // component 2 (< m2)
};

__device__ __forceinline__ double mrg_sn(uint32_t x) { return __hiloint2double(0, (int)x); }

__device__ __forceinline__ uint32_t mrg_c1_sn(uint32_t x0, uint32_t x1, const MrgFpK& K)
{
    const double t = __fma_rn(-202682.0, mrg_sn(x0), K.sn_c1q);  // 202682 (m1 - x0)
    const double q = __fma_rn(350895.0, mrg_sn(x1), t);
    const double Q = __fma_rd(q, K.sn_c1s, K.sn_M);
    return 4u * (uint32_t)__double2loint(q) + 209u * (uint32_t)__double2loint(Q);
}

__device__ __forceinline__ uint32_t mrg_c2_sn(uint32_t y0, uint32_t y2, const MrgFpK& K)
{
    const double t = __fma_rn(-(double)kA23n, mrg_sn(y0), K.sn_c2p);  // a23n (m2 - y0)
    const double p = __fma_rn((double)kA21, mrg_sn(y2), t);
    const double Q = __fma_rd(p, K.sn_c2s, K.sn_M);
    return (uint32_t)__double2loint(p) + kC2 * (uint32_t)__double2loint(Q);
}

__device__ __forceinline__ uint32_t mrg_next(MrgSN& s, const MrgFpK& K = mrg_fpk())
{
    const uint32_t p1 = mrg_c1_sn(s.x0, s.x1, K);
    s.x0 = s.x1;
    s.x1 = s.x2;
    s.x2 = p1;
    const uint32_t p2 = mrg_c2_sn(s.y0, s.y2, K);
    s.y0 = s.y1;
    s.y1 = s.y2;
    s.y2 = p2;
    return mrg_combine(p1, p2);
}

__device__ __forceinline__ MrgSN to_mrg_sn(const Mrg& s) { return MrgSN{s.x0, s.x1, s.x2, s.y0, s.y1, s.y2}; }

// MrgMF: the same subnormal representation with magic-free quotients. In the
// subnormal range every double has ulp 2^-1074, so for p_sub = D(p)
//   k_sub = mul.rm(p_sub, inv) = floor(p * inv) * 2^-1074 = D(k)
// exactly (the product is rounded once, toward -inf, onto the 2^-1074 grid;
// floor(p * inv) = floor(p / m) by the floor step's inverse bounds), and
//   r_sub = fma(-k_sub, m, p_sub) = D(p - k m)
// is the next state pair itself (bits {r, 0}) with the output in its low word.
// 4 FP64 instructions per component and no integer or move instructions:
// component 1 takes the signed form (|p| < 2^52.42; r in [0, m1], m1 only at
// p = k m1 < 0, as in mrg_c1_floor), component 2 the positive form.
struct MrgMF {
    double x0, x1, x2;  // D(x), component 1
    double y0, y1, y2;  // D(y), component 2
};

__device__ __forceinline__ uint32_t mrg_next(MrgMF& s, const MrgFpK& K = mrg_fpk())
{
    const double t1 = __dmul_rn((double)kA13n, s.x0);
    const double p1 = __fma_rn((double)kA12, s.x1, -t1);
    const double r1 = __fma_rn(-__dmul_rd(p1, K.inv1), K.m1, p1);
    s.x0 = s.x1;
    s.x1 = s.x2;
    s.x2 = r1;
    const double t2 = __fma_rn(-(double)kA23n, s.y0, K.sn_c2p);
    const double p2 = __fma_rn((double)kA21, s.y2, t2);
    const double r2 = __fma_rn(-__dmul_rd(p2, K.inv2), K.m2, p2);
    s.y0 = s.y1;
    s.y1 = s.y2;
    s.y2 = r2;
    return mrg_combine((uint32_t)__double2loint(r1), (uint32_t)__double2loint(r2));
}

__device__ __forceinline__ MrgMF to_mrg_mf(const Mrg& s)
{
    return MrgMF{mrg_sn(s.x0), mrg_sn(s.x1), mrg_sn(s.x2), mrg_sn(s.y0), mrg_sn(s.y1), mrg_sn(s.y2)};
}


// ------------------------------------------------------------------ Philox4x32-10

struct W4 {
    uint32_t x, y, z, w;
};

__device__ __forceinline__ W4 philox10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                       uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)kPM0 * c0;
        const uint64_t p1 = (uint64_t)kPM1 * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
        k0 += kPW0;
        k1 += kPW1;
    }
    return W4{c0, c1, c2, c3};
}

// Rounds 2..10 of a block whose round-1 products are given (lets callers
// hoist the multiplications that only depend on the stream index).
__device__ __forceinline__ W4 philox10_from_r1(uint32_t hi0, uint32_t lo0, uint32_t hi1, uint32_t lo1,
                                               uint32_t c1, uint32_t c3, uint32_t k0, uint32_t k1)
{
    uint32_t c0 = hi1 ^ c1 ^ k0, c2 = hi0 ^ c3 ^ k1;
    c1 = lo1;
    c3 = lo0;
    k0 += kPW0;
    k1 += kPW1;
#pragma unroll
    for (int r = 1; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)kPM0 * c0;
        const uint64_t p1 = (uint64_t)kPM1 * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
        k0 += kPW0;
        k1 += kPW1;
    }
    return W4{c0, c1, c2, c3};
}

// Block from its round-1 outputs' varying half: for a fixed stream g and a
// fixed high counter word, round 1 gives c0' = hi(M1*g_lo) ^ blk_hi ^ k0 and
// c1' = lo(M1*g_lo) (both fixed), so round 2's M0*c0' (q) is fixed too; only
// pa = M0*blk_lo varies. Rounds 3..10 as usual. 17 IMAD.WIDE per block.
// HILO: round 10 with separate low (IMAD) and high (IMAD.HI) products, for
// callers that store the block as an STG.256 octet (the bulk fill: 2.51 vs
// 2.53 ms alone, 2.91 vs 2.94 back to back, lab68); the others keep IMAD.WIDE.
template <bool HILO = false>
__device__ __forceinline__ W4 philox10_from_r2(uint64_t pa, uint64_t q, uint32_t c1r1, uint32_t g_hi,
                                               uint32_t k0, uint32_t k1)
{
    // round 1 (key k0, k1): c2' = hi(pa) ^ g_hi ^ k1, c3' = lo(pa)
    const uint32_t c2 = (uint32_t)(pa >> 32) ^ g_hi ^ k1;
    const uint32_t c3 = (uint32_t)pa;
    k0 += kPW0;
    k1 += kPW1;
    // round 2: p0 = q (= M0*c0'), p1 = M1*c2'
    const uint64_t p1 = (uint64_t)kPM1 * c2;
    uint32_t d0 = (uint32_t)(p1 >> 32) ^ c1r1 ^ k0;
    uint32_t d1 = (uint32_t)p1;
    uint32_t d2 = (uint32_t)(q >> 32) ^ c3 ^ k1;
    uint32_t d3 = (uint32_t)q;
    k0 += kPW0;
    k1 += kPW1;
#pragma unroll
    for (int r = 2; r < (HILO ? 9 : 10); ++r) {
        const uint64_t e0 = (uint64_t)kPM0 * d0;
        const uint64_t e1 = (uint64_t)kPM1 * d2;
        const uint32_t n0 = (uint32_t)(e1 >> 32) ^ d1 ^ k0;
        const uint32_t n2 = (uint32_t)(e0 >> 32) ^ d3 ^ k1;
        d1 = (uint32_t)e1;
        d3 = (uint32_t)e0;
        d0 = n0;
        d2 = n2;
        k0 += kPW0;
        k1 += kPW1;
    }
    if (HILO) {
        // round 10: output words 1 and 3 need not come from the even half of
        // an IMAD.WIDE pair, which an STG.256 octet cannot take without moves
        const uint32_t n0 = __umulhi(kPM1, d2) ^ d1 ^ k0;
        const uint32_t n2 = __umulhi(kPM0, d0) ^ d3 ^ k1;
        d1 = kPM1 * d2;
        d3 = kPM0 * d0;
        d0 = n0;
        d2 = n2;
    }
    return W4{d0, d1, d2, d3};
}

// 64-bit + 64-bit on the ALU pipe.
__device__ __forceinline__ uint64_t add64w(uint64_t a, uint64_t b)
{
    uint32_t lo, hi;
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, %5;"
        : "=r"(lo), "=r"(hi)
        : "r"((uint32_t)a), "r"((uint32_t)b), "r"((uint32_t)(a >> 32)), "r"((uint32_t)(b >> 32)));
    return ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ W4 philox_blk(uint64_t blk, uint64_t g, uint32_t k0, uint32_t k1)
{
    return philox10((uint32_t)blk, (uint32_t)(blk >> 32), (uint32_t)g, (uint32_t)(g >> 32), k0, k1);
}

__device__ __forceinline__ uint32_t lane_of(const W4& v, uint32_t l)
{
    return l == 0 ? v.x : l == 1 ? v.y : l == 2 ? v.z : v.w;
}

// Generic per-draw access with a one-block cache (arbitrary offsets).
struct PhiloxCursor {
    uint64_t g;
    uint32_t k0, k1;
    uint64_t blk;
    bool valid;
    W4 v;
    __device__ __forceinline__ uint32_t word(uint64_t b, uint32_t lane)
    {
        if (!valid || b != blk) {
            v = philox_blk(b, g, k0, k1);
            blk = b;
            valid = true;
        }
        return lane_of(v, lane);
    }
};

// ------------------------------------------------------------------ Threefry4x64-20

// Threefry4x64-20 [Salmon.etal.2011] (P L322-336): Threefish-256 ARX rounds
// (64-bit add, rotate, xor: ALU pipe only, no multiplies), key injection every
// 4 rounds from ks = (k0..k3, parity), here with k2 = k3 = 0 (R16).
struct Q4 {
    uint64_t x, y, z, w;
};

// 64-bit rotate as two 32-bit funnel shifts (SHF.L.W on the ALU pipe; R = 32
// is a register swap). ptxas lowers the shift-or form to 4-5 instructions.
template <int R>
__device__ __forceinline__ uint64_t rotl64(uint64_t v)
{
    const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
    constexpr uint32_t S = R >= 32 ? (uint32_t)(R - 32) : (uint32_t)R;
    uint32_t nh, nl;
    if (R == 32) {
        nh = lo;
        nl = hi;
    } else if (R < 32) {
        nh = __funnelshift_l(lo, hi, S);
        nl = __funnelshift_l(hi, lo, S);
    } else {
        nh = __funnelshift_l(hi, lo, S);
        nl = __funnelshift_l(lo, hi, S);
    }
    return ((uint64_t)nh << 32) | nl;
}

template <int A, int B, bool ODD>
__device__ __forceinline__ void tf_mix(Q4& v)
{
    if (!ODD) {
        v.x += v.y; v.y = rotl64<A>(v.y) ^ v.x;
        v.z += v.w; v.w = rotl64<B>(v.w) ^ v.z;
    } else {
        v.x += v.w; v.w = rotl64<A>(v.w) ^ v.x;
        v.z += v.y; v.y = rotl64<B>(v.y) ^ v.z;
    }
}

__device__ __forceinline__ void tf_inject(Q4& v, const uint64_t* ks, int s)
{
    v.x += ks[s % 5];
    v.y += ks[(s + 1) % 5];
    v.z += ks[(s + 2) % 5];
    v.w += ks[(s + 3) % 5] + (uint64_t)s;
}

// Block (blk, g, 0, 0) under key (k0, k1, 0, 0).
__device__ __forceinline__ Q4 threefry20(uint64_t blk, uint64_t g, uint64_t k0, uint64_t k1)
{
    const uint64_t ks[5] = {k0, k1, 0, 0, 0x1BD11BDAA9FC1A22ull ^ k0 ^ k1};
    Q4 v{blk + k0, g + k1, 0, 0};
#pragma unroll
    for (int q = 0; q < 5; ++q) {  // rounds 4q..4q+3 use R[(4q..4q+3) % 8]
        if ((q & 1) == 0) {
            tf_mix<14, 16, false>(v);
            tf_mix<52, 57, true>(v);
            tf_mix<23, 40, false>(v);
            tf_mix<5, 37, true>(v);
        } else {
            tf_mix<25, 33, false>(v);
            tf_mix<46, 12, true>(v);
            tf_mix<58, 22, false>(v);
            tf_mix<32, 32, true>(v);
        }
        tf_inject(v, ks, q + 1);
    }
    return v;
}

// ------------------------------------------------------------------ TinyMT32

// TinyMT32 [Saito2011] (P L287-317 §4.2): 127-bit F2-linear state in four
// words plus the parameter set (mat1, mat2, tmat) from Dynamic Creator.
struct TinyMT {
    uint32_t s0, s1, s2, s3;
    uint32_t mat1, mat2, tmat;
};

// The step is ALU-bound (LOP3, shifts); the conditional masks (y & 1 ? mat : 0)
// are formed as (y & 1) * mat on the FMA-heavy pipe (IMAD), which the
// generator otherwise leaves idle. SHV_TINYMT_IMAD = 0 keeps the mask form.
#ifndef SHV_TINYMT_IMAD
#define SHV_TINYMT_IMAD 1
#endif
__device__ __forceinline__ uint32_t bit_times(uint32_t b, uint32_t mat)
{
    if (SHV_TINYMT_IMAD) {
        uint32_t r;
        asm("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(b), "r"(mat));
        return r;
    }
    return (0u - b) & mat;
}

__device__ __forceinline__ void tinymt_next_state(TinyMT& t)
{
    uint32_t y = t.s3;
    uint32_t x = (t.s0 & 0x7fffffffu) ^ t.s1 ^ t.s2;
    x ^= x << 1;
    y ^= (y >> 1) ^ x;
    const uint32_t b = y & 1u;
    t.s0 = t.s1;
    t.s1 = t.s2 ^ bit_times(b, t.mat1);
    t.s2 = x ^ (y << 10) ^ bit_times(b, t.mat2);
    t.s3 = y;
}

__device__ __forceinline__ uint32_t tinymt_temper(const TinyMT& t)
{
    const uint32_t t1 = t.s0 + (t.s2 >> 8);
    return t.s3 ^ t1 ^ bit_times(t1 & 1u, t.tmat);
}

__device__ __forceinline__ uint32_t tinymt_next(TinyMT& t)
{
    tinymt_next_state(t);
    return tinymt_temper(t);
}

// The authors' seeding: 7 rounds of the 1812433253 scramble, period
// certification ("TINY" if the 127 significant bits are zero), 8 pre-steps.
__device__ __forceinline__ void tinymt_init(TinyMT& t, uint32_t mat1, uint32_t mat2, uint32_t tmat, uint32_t seed)
{
    uint32_t st[4] = {seed, mat1, mat2, tmat};
#pragma unroll
    for (int i = 1; i < 8; ++i)
        st[i & 3] ^= (uint32_t)i + 1812433253u * (st[(i - 1) & 3] ^ (st[(i - 1) & 3] >> 30));
    if ((st[0] & 0x7fffffffu) == 0 && st[1] == 0 && st[2] == 0 && st[3] == 0) {
        st[0] = 'T';
        st[1] = 'I';
        st[2] = 'N';
        st[3] = 'Y';
    }
    t = TinyMT{st[0], st[1], st[2], st[3], mat1, mat2, tmat};
#pragma unroll 1
    for (int i = 0; i < 8; ++i) tinymt_next_state(t);
}

// y = M x over GF(2) for a 128x128 matrix stored as 128 columns of 4 words
// (column c = image of unit vector e_c): XOR of the columns x selects.
__device__ __forceinline__ void gf2_apply(const uint32_t* __restrict__ M, TinyMT& t)
{
    const uint32_t x[4] = {t.s0, t.s1, t.s2, t.s3};
    uint32_t y0 = 0, y1 = 0, y2 = 0, y3 = 0;
#pragma unroll 4
    for (int c = 0; c < 128; ++c) {
        if ((x[c >> 5] >> (c & 31)) & 1u) {
            const uint4 col = *reinterpret_cast<const uint4*>(M + 4 * c);
            y0 ^= col.x;
            y1 ^= col.y;
            y2 ^= col.z;
            y3 ^= col.w;
        }
    }
    t.s0 = y0;
    t.s1 = y1;
    t.s2 = y2;
    t.s3 = y3;
}

// ------------------------------------------------------------------ conversions (R7)

__device__ __forceinline__ float to_f32(uint32_t w)
{
    return __fmul_rn(__uint2float_rn(w >> 8), 0x1p-24f);
}

__device__ __forceinline__ double mrg_f64(uint32_t z)
{
    return __dmul_rn(__uint2double_rn(z), 0x1.000000d00000bp-32);
}

__device__ __forceinline__ double philox_f64(uint32_t lo, uint32_t hi)
{
    const uint64_t b = (((uint64_t)hi << 32) | lo) >> 11;
    return __dmul_rn(__ull2double_rn(b), 0x1p-53);
}

// ------------------------------------------------------------------ stores

// One full 32-byte sector per thread: STG.E.ENL2.256 on sm_100a.
__device__ __forceinline__ void st_v8(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                      uint32_t e, uint32_t f, uint32_t g, uint32_t h)
{
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(a),
                 "r"(b), "r"(c), "r"(d), "r"(e), "r"(f), "r"(g), "r"(h)
                 : "memory");
}

__device__ __forceinline__ void st_v8(void* p, uint4 a, uint4 b)
{
    st_v8(p, a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w);
}

__device__ __forceinline__ void st_v8f(void* p, float a, float b, float c, float d, float e,
                                       float f, float g, float h)
{
    st_v8(p, __float_as_uint(a), __float_as_uint(b), __float_as_uint(c), __float_as_uint(d),
          __float_as_uint(e), __float_as_uint(f), __float_as_uint(g), __float_as_uint(h));
}

__device__ __forceinline__ void st_v4d(void* p, double a, double b, double c, double d)
{
    st_v8(p, __double2loint(a), __double2hiint(a), __double2loint(b), __double2hiint(b),
          __double2loint(c), __double2hiint(c), __double2loint(d), __double2hiint(d));
}

// ------------------------------------------------------------------ reduction

__device__ __forceinline__ void block_reduce_add(uint64_t v, unsigned long long* dst)
{
    __shared__ unsigned long long part[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) part[warp] = v;
    __syncthreads();
    if (warp == 0) {
        const unsigned nw = (blockDim.x + 31) >> 5;
        v = lane < nw ? part[lane] : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && v) atomicAdd(dst, (unsigned long long)v);
    }
}

// Dartboard hit (R9): X = w0>>8, Y = w1>>8, X^2 + Y^2 < 2^48.
__device__ __forceinline__ uint32_t hit(uint32_t w0, uint32_t w1)
{
    const uint32_t X = w0 >> 8, Y = w1 >> 8;
    const uint64_t r2 = (uint64_t)X * X + (uint64_t)Y * Y;  // < 2^49
    return (uint32_t)(r2 >> 48) == 0u;
}

// The same test on the FP64 pipe (for kernels whose FMA-heavy pipe is the
// bottleneck): X, Y < 2^24 become exact doubles via the 2^52 bit pattern,
// X^2 + Y^2 < 2^49 is exact in binary64, and the comparison is exact.
__device__ __forceinline__ uint32_t hit_fp64(uint32_t w0, uint32_t w1)
{
    const double two52 = 4503599627370496.0;
    const double x = __dadd_rn(__hiloint2double(0x43300000, (int)(w0 >> 8)), -two52);
    const double y = __dadd_rn(__hiloint2double(0x43300000, (int)(w1 >> 8)), -two52);
    return __fma_rn(x, x, __dmul_rn(y, y)) < 281474976710656.0 ? 1u : 0u;  // 2^48
}

// The same test with the conversions on the XU pipe (I2F.F64.U32) instead of
// the 2^52 bit pattern, whose pair formation costs a MOV (often IMAD.MOV, on
// the FMA-heavy pipe that the Philox rounds saturate) and a DADD per coordinate.
__device__ __forceinline__ uint32_t hit_fp64_cvt(uint32_t w0, uint32_t w1)
{
    const double x = __uint2double_rn(w0 >> 8), y = __uint2double_rn(w1 >> 8);
    return __fma_rn(x, x, __dmul_rn(y, y)) < 281474976710656.0 ? 1u : 0u;  // 2^48
}

}  // namespace dev
}  // namespace shv
