// step4_lab.cu — MRG32k3a steps with the state in the FP64 SUBNORMAL range.
// D(x) = the register pair {x, 0} = x * 2^-1074 exactly, and for an integer
// v in [0, 2^53) the bit pattern of D(v) IS v (the subnormal/normal boundary
// at 2^52 is seamless: exponent field 1 = bit 52). So a product sum p formed
// exactly on the FP64 pipe hands its low word (p mod 2^32) to the integer
// pipes for free, and the floor quotient k = floor(p / m), taken by one
// fma.rm(p, inv * 2^1010, 1.5 * 2^-12) (ulp 2^-64 there), hands k as its low
// word. The residue r = p - k m is then either
//   (int)  lo(p) + c k  (mod 2^32, m = 2^32 - c): one IMAD, r canonical, or
//   (fp64) fma(-(Q - M), m * 2^-1010, p): two FP64 ops, r = D(r) directly.
// No magic-number bias and no conversion in either direction.
//   c2 (S2): p = a21 y2 + a23n (m2 - y0) in [0, 2^52.86): 2 DFMA + 1 DFMA.RM.
//   c1 (S1P): p = 4 q, q = 350895 x1 + 202682 (m1 - x0) < 2^51.08 (the
//       factor 4 of a12 and a13n pulled out keeps the positive form exact);
//       floor(4q / m1) = floor(q * (4 inv1)) since 4q inv1-err m1 < 0.72;
//       r = 4 lo(q) + 209 k (mod 2^32).
//   c1 (F):  signed p = a12 x1 - a13n x0, |p| < 2^52.42, fp64 residue in [0, m1].
// Variants (compute-only, 8 values per iteration, one stream per thread):
//   if  : MrgIF (product)       ff : MrgFF
//   sA  : c1 S1P int  + c2 S2 int      sB : c1 F fp64 + c2 S2 int
//   sC  : c1 F fp64   + c2 fp64        sD : c1 S1P int + c2 fp64
// Each is checked against the integer step (mismatch counts must be 0).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "shv_device.cuh"
using namespace shv::dev;

struct KP {
    double v[6];
    uint32_t a12, a13n;
    double c1q, c2p, c1s, c1f, c2s, m1s, m2s, M;
};
__device__ __forceinline__ MrgFpK kp(const KP& p) { return MrgFpK{p.v[0], p.v[1], p.v[2], p.v[3], p.v[4], p.v[5], p.a12, p.a13n}; }
__device__ __forceinline__ Mrg seed_of(uint32_t t) { return Mrg{12345u + t, 12345u, 12345u ^ t, 12345u, 777u + t, 12345u}; }

__device__ __forceinline__ double D(uint32_t x) { return __hiloint2double(0, (int)x); }
__device__ __forceinline__ uint32_t lo(double d) { return (uint32_t)__double2loint(d); }

struct SK { double c1q, c2p, c1s, c1f, c2s, m1s, m2s, M; };

__device__ __forceinline__ uint32_t c1_int(uint32_t x0, uint32_t x1, const SK& K)
{
    const double t = __fma_rn(-202682.0, D(x0), K.c1q);
    const double q = __fma_rn(350895.0, D(x1), t);
    const double Q = __fma_rd(q, K.c1s, K.M);
    return 4u * lo(q) + 209u * lo(Q);
}
__device__ __forceinline__ uint32_t c2_int(uint32_t y0, uint32_t y2, const SK& K)
{
    const double t = __fma_rn(-1370589.0, D(y0), K.c2p);
    const double p = __fma_rn(527612.0, D(y2), t);
    const double Q = __fma_rd(p, K.c2s, K.M);
    return lo(p) + 22853u * lo(Q);
}
__device__ __forceinline__ double c1_fp(double x0, double x1, const SK& K)
{
    const double t = __dmul_rn(810728.0, x0);
    const double p = __fma_rn(1403580.0, x1, -t);
    const double Q = __fma_rd(p, K.c1f, K.M);
    return __fma_rn(-__dadd_rn(Q, -K.M), K.m1s, p);
}
__device__ __forceinline__ double c2_fp(double y0, double y2, const SK& K)
{
    const double t = __fma_rn(-1370589.0, y0, K.c2p);
    const double p = __fma_rn(527612.0, y2, t);
    const double Q = __fma_rd(p, K.c2s, K.M);
    return __fma_rn(-__dadd_rn(Q, -K.M), K.m2s, p);
}

// Magic-free quotients: in the subnormal range every double has ulp 2^-1074,
// so k_sub = mul.rm(p_sub, inv) = floor(p inv) 2^-1074 = D(k) exactly (no
// magic constant), and r_sub = fma(-k_sub, m, p_sub) = D(p - k m) is the next
// state pair itself (bits {r, 0}) and its low word the output. 4 FP64 ops per
// component, no integer instructions, no zero moves.
__device__ __forceinline__ double c1_mf(double x0, double x1, double inv1, double m1)
{
    const double t = __dmul_rn(810728.0, x0);
    const double p = __fma_rn(1403580.0, x1, -t);            // signed, |p| < 2^52.42
    const double k = __dmul_rd(p, inv1);                      // D(floor(p / m1)) (negative allowed)
    return __fma_rn(-k, m1, p);                               // D(r), r in [0, m1]
}
__device__ __forceinline__ double c2_mf(double y0, double y2, double inv2, double m2, double c2p)
{
    const double t = __fma_rn(-1370589.0, y0, c2p);
    const double p = __fma_rn(527612.0, y2, t);
    const double k = __dmul_rd(p, inv2);
    return __fma_rn(-k, m2, p);
}
struct SE { double x0, x1, x2, y0, y1, y2; };
struct SF { uint32_t x0, x1, x2; double y0, y1, y2; };
struct SG { double x0, x1, x2; uint32_t y0, y1, y2; };

struct SA { uint32_t x0, x1, x2, y0, y1, y2; };
struct SB { double x0, x1, x2; uint32_t y0, y1, y2; };
struct SC { double x0, x1, x2, y0, y1, y2; };
struct SDs { uint32_t x0, x1, x2; double y0, y1, y2; };

__device__ __forceinline__ uint32_t nxt(SA& s, const SK& K)
{
    const uint32_t p1 = c1_int(s.x0, s.x1, K);
    s.x0 = s.x1; s.x1 = s.x2; s.x2 = p1;
    const uint32_t p2 = c2_int(s.y0, s.y2, K);
    s.y0 = s.y1; s.y1 = s.y2; s.y2 = p2;
    return mrg_combine(p1, p2);
}
__device__ __forceinline__ uint32_t nxt(SB& s, const SK& K)
{
    const double r1 = c1_fp(s.x0, s.x1, K);
    s.x0 = s.x1; s.x1 = s.x2; s.x2 = r1;
    const uint32_t p2 = c2_int(s.y0, s.y2, K);
    s.y0 = s.y1; s.y1 = s.y2; s.y2 = p2;
    return mrg_combine(lo(r1), p2);
}
__device__ __forceinline__ uint32_t nxt(SC& s, const SK& K)
{
    const double r1 = c1_fp(s.x0, s.x1, K);
    s.x0 = s.x1; s.x1 = s.x2; s.x2 = r1;
    const double r2 = c2_fp(s.y0, s.y2, K);
    s.y0 = s.y1; s.y1 = s.y2; s.y2 = r2;
    return mrg_combine(lo(r1), lo(r2));
}
__device__ __forceinline__ uint32_t nxt(SDs& s, const SK& K)
{
    const uint32_t p1 = c1_int(s.x0, s.x1, K);
    s.x0 = s.x1; s.x1 = s.x2; s.x2 = p1;
    const double r2 = c2_fp(s.y0, s.y2, K);
    s.y0 = s.y1; s.y1 = s.y2; s.y2 = r2;
    return mrg_combine(p1, lo(r2));
}

struct MK { double inv1, inv2, m1, m2; };
__device__ __forceinline__ uint32_t nxt(SE& s, const SK& K, const MK& Q)
{
    const double r1 = c1_mf(s.x0, s.x1, Q.inv1, Q.m1);
    s.x0 = s.x1; s.x1 = s.x2; s.x2 = r1;
    const double r2 = c2_mf(s.y0, s.y2, Q.inv2, Q.m2, K.c2p);
    s.y0 = s.y1; s.y1 = s.y2; s.y2 = r2;
    return mrg_combine(lo(r1), lo(r2));
}
__device__ __forceinline__ uint32_t nxt(SF& s, const SK& K, const MK& Q)
{
    const uint32_t p1 = c1_int(s.x0, s.x1, K);
    s.x0 = s.x1; s.x1 = s.x2; s.x2 = p1;
    const double r2 = c2_mf(s.y0, s.y2, Q.inv2, Q.m2, K.c2p);
    s.y0 = s.y1; s.y1 = s.y2; s.y2 = r2;
    return mrg_combine(p1, lo(r2));
}
__device__ __forceinline__ uint32_t nxt(SG& s, const SK& K, const MK& Q)
{
    const double r1 = c1_mf(s.x0, s.x1, Q.inv1, Q.m1);
    s.x0 = s.x1; s.x1 = s.x2; s.x2 = r1;
    const uint32_t p2 = c2_int(s.y0, s.y2, K);
    s.y0 = s.y1; s.y1 = s.y2; s.y2 = p2;
    return mrg_combine(lo(r1), p2);
}

// combine without ISETP: w = r2 - r1 with borrow b = (r1 > r2) as a mask;
// r1 <= r2: z = -w + m1 (r1 == r2 -> m1), else z = -w.
__device__ __forceinline__ uint32_t combine_cc(uint32_t p1, uint32_t p2)
{
    uint32_t w, b;
    asm("{\n\t"
        "sub.cc.u32 %0, %2, %3;\n\t"
        "subc.u32 %1, 0, 0;\n\t"
        "}"
        : "=r"(w), "=r"(b) : "r"(p2), "r"(p1));
    return (0u - w) + (~b & 4294967087u);
}
struct SAc : SA {};
__device__ __forceinline__ uint32_t nxt(SAc& s, const SK& K)
{
    const uint32_t p1 = c1_int(s.x0, s.x1, K);
    s.x0 = s.x1; s.x1 = s.x2; s.x2 = p1;
    const uint32_t p2 = c2_int(s.y0, s.y2, K);
    s.y0 = s.y1; s.y1 = s.y2; s.y2 = p2;
    return combine_cc(p1, p2);
}

template <int V>
__global__ void __launch_bounds__(256) k(uint32_t* out, const __grid_constant__ KP p, int iters)
{
    const MrgFpK K = kp(p);
    const SK S{p.c1q, p.c2p, p.c1s, p.c1f, p.c2s, p.m1s, p.m2s, p.M};
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const Mrg s0 = seed_of(t);
    MrgIF s = to_mrg_if(s0);
    MrgFF f = to_mrg_ff(s0);
    SA a{s0.x0, s0.x1, s0.x2, s0.y0, s0.y1, s0.y2};
    SAc ac; ac.x0 = s0.x0; ac.x1 = s0.x1; ac.x2 = s0.x2; ac.y0 = s0.y0; ac.y1 = s0.y1; ac.y2 = s0.y2;
    SB b{D(s0.x0), D(s0.x1), D(s0.x2), s0.y0, s0.y1, s0.y2};
    SC c{D(s0.x0), D(s0.x1), D(s0.x2), D(s0.y0), D(s0.y1), D(s0.y2)};
    SDs d{s0.x0, s0.x1, s0.x2, D(s0.y0), D(s0.y1), D(s0.y2)};
    SE e{D(s0.x0), D(s0.x1), D(s0.x2), D(s0.y0), D(s0.y1), D(s0.y2)};
    SF ff{s0.x0, s0.x1, s0.x2, D(s0.y0), D(s0.y1), D(s0.y2)};
    SG gg{D(s0.x0), D(s0.x1), D(s0.x2), s0.y0, s0.y1, s0.y2};
    const MK Q{p.v[1], p.v[2], p.v[3], p.v[4]};
    Mrg ri = s0;
    uint32_t acc = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 12; ++u) {
            uint32_t z;
            if (V == 0) z = mrg_next(s, K);
            else if (V == 1) z = mrg_next(f, K);
            else if (V == 2) z = nxt(a, S);
            else if (V == 3) z = nxt(b, S);
            else if (V == 4) z = nxt(c, S);
            else if (V == 5) z = nxt(d, S);
            else if (V == 7) z = nxt(ac, S);
            else if (V == 8) z = nxt(e, S, Q);
            else if (V == 9) z = nxt(ff, S, Q);
            else if (V == 10) z = nxt(gg, S, Q);
            else z = mrg_next(ri, K);
            acc += z;
        }
    }
    out[t] = acc;
}

template <class F>
float tms(F f)
{
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    f(); cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
    return best;
}

int main()
{
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    KP p{{6755399441055744.0, 1.0 / 4294967087.0, 0x1.000059451f212p-32, 4294967087.0, 4294944443.0, 5886603609186927.0},
         1403580u, 810728u, 0, 0, 0x1.000000d10000bp+980, 0x1.000000d10000bp+978, 0x1.000059451f212p+978,
         0x1.fffffe5e00000p-979, 0x1.ffff4d7600000p-979, 0x1.8p-12};
    const uint64_t c1q = 202682ull * 4294967087ull, c2p = 1370589ull * 4294944443ull;
    memcpy(&p.c1q, &c1q, 8);
    memcpy(&p.c2p, &c2p, 8);
    uint32_t* o; cudaMalloc(&o, (size_t)sms * 16 * 256 * 4);
    const int iters = 768;
    const char* names[] = {"if", "ff", "sA", "sB", "sC", "sD", "int", "sAc", "sE", "sF", "sG"};
    printf("{");
    auto run = [&](int v, auto kern) {
        for (int bps : {4, 8}) {
            const size_t n = (size_t)sms * bps * 256;
            float ms = tms([&] { kern<<<sms * bps, 256>>>(o, p, iters); });
            printf("\"%s_b%d\": %.4f, ", names[v], bps, (double)n * iters * 12 / (ms * 1e-3) / 1e12);
        }
    };
    for (int rep = 0; rep < 2; ++rep) {
        run(0, k<0>); run(2, k<2>); run(4, k<4>); run(8, k<8>); run(9, k<9>); run(10, k<10>);
    }
    const size_t n = (size_t)sms * 8 * 256;
    uint32_t* h = new uint32_t[n]; uint32_t* ref = new uint32_t[n];
    k<6><<<sms * 8, 256>>>(o, p, 64); cudaMemcpy(ref, o, n * 4, cudaMemcpyDeviceToHost);
    auto chk = [&](int v, auto kern) {
        kern<<<sms * 8, 256>>>(o, p, 64);
        cudaMemcpy(h, o, n * 4, cudaMemcpyDeviceToHost);
        size_t bad = 0; for (size_t i = 0; i < n; ++i) bad += h[i] != ref[i];
        printf("\"%s_mismatch\": %zu, ", names[v], bad);
    };
    chk(0, k<0>); chk(2, k<2>); chk(4, k<4>); chk(8, k<8>); chk(9, k<9>); chk(10, k<10>);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("\"sms\": %d, \"clock_khz\": %d, \"err\": \"%s\"}\n", sms, clk, cudaGetErrorString(cudaGetLastError()));
}
