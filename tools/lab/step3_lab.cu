// step3_lab.cu — where does the hybrid MRG32k3a step (MrgIF: component 1 in
// 32-bit integer arithmetic, component 2 on the FP64 pipe) lose issue slots?
// Compute-only kernels (no stores), 8 values per iteration, one stream per
// thread, 8 blocks x 256 threads per SM. Each variant prints T values/s and its
// static instruction count per value (from the SASS, counted on the host side
// by tools/lab/sass_count.py) lets one derive the issue rate.
//   c2  : component 2 only (6 FP64 ops)        c1 : component 1 only (7 int ops)
//   if  : the product step (MrgIF)              ff : both components on FP64 (MrgFF)
//   if_nocmb : MrgIF without the combine (p1 ^ p2)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "shv_device.cuh"
using namespace shv::dev;

struct KP { double v[6]; uint32_t a12, a13n; uint32_t k1lo, k1hi; };
__device__ __forceinline__ MrgFpK kp(const KP& p) { return MrgFpK{p.v[0], p.v[1], p.v[2], p.v[3], p.v[4], p.v[5], p.a12, p.a13n}; }
__device__ __forceinline__ Mrg seed_of(uint32_t t) { return Mrg{12345u + t, 12345u, 12345u ^ t, 12345u, 777u + t, 12345u}; }

// DI: component 1's products on the FP64 pipe with the factor 4 of a12 and
// a13n pulled out (q = 350895 x1 + 202682 (m1 - x0) < 2^51.1, so Q = 2^52 + q
// is exact and its low 52 bits are q), the fold 4q mod m1 in 32-bit ALU
// arithmetic (no IMAD.WIDE), the state word back to a double by the 2^52 trick.
struct MrgDI { double x0, x1, x2, y0, y1, y2; };
__device__ __forceinline__ uint32_t c1_di(double x0, double x1, double& xn)
{
    const double t = __fma_rn(-202682.0, x0, 5374112146497830.0);  // 2^52 + 202682 m1 - 202682 x0
    const double Q = __fma_rn(350895.0, x1, t);                      // 2^52 + q
    const uint32_t lo = (uint32_t)__double2loint(Q), hi = (uint32_t)__double2hiint(Q);
    const uint32_t H4 = __funnelshift_l(lo, hi, 2) & 0x3FFFFFu;      // floor(4q / 2^32)
    const uint32_t L4 = lo << 2;                                       // 4q mod 2^32
    uint32_t u = H4 * 209u + L4;
    if ((u < L4) | (u >= 4294967087u)) u += 209u;
    xn = __hiloint2double(0x43300000, (int)u) - 4503599627370496.0;
    return u;
}
__device__ __forceinline__ uint32_t next_di(MrgDI& s, const MrgFpK& K)
{
    double xn, r;
    const uint32_t p1 = c1_di(s.x0, s.x1, xn);
    s.x0 = s.x1; s.x1 = s.x2; s.x2 = xn;
    const uint32_t p2 = mrg_c2_floor(s.y0, s.y2, r, K);
    s.y0 = s.y1; s.y1 = s.y2; s.y2 = r;
    return mrg_combine(p1, p2);
}

// SD: component 1's products on the FP64 pipe in the SUBNORMAL range: the
// register pair {x, 0} is the double x * 2^-1074 (exact), and
// Q = fma(350895, X1, fma(-202682, X0, K)) with K = 202682 m1 * 2^-1074 is
// q * 2^-1074, q = 350895 x1 + 202682 (m1 - x0) < 2^51.1, whose bit pattern IS
// the integer q (no exponent bits to mask). The fold 4q mod m1 on the ALU.
struct MrgSD { uint32_t x0, x1, x2; double y0, y1, y2; };
__device__ __forceinline__ double sub_of(uint32_t x) { return __hiloint2double(0, (int)x); }
__device__ __forceinline__ uint32_t c1_sd(uint32_t x0, uint32_t x1, double K1)
{
    const double t = __fma_rn(-202682.0, sub_of(x0), K1);
    const double Q = __fma_rn(350895.0, sub_of(x1), t);
    const uint32_t lo = (uint32_t)__double2loint(Q), hi = (uint32_t)__double2hiint(Q);
    const uint32_t H4 = __funnelshift_l(lo, hi, 2);   // floor(4q / 2^32) < 2^21.1
    const uint32_t L4 = lo << 2;                        // 4q mod 2^32
    uint32_t u = H4 * 209u + L4;
    if ((u < L4) | (u >= 4294967087u)) u += 209u;
    return u;
}
__device__ __forceinline__ uint32_t next_sd(MrgSD& s, const MrgFpK& K, double K1)
{
    const uint32_t p1 = c1_sd(s.x0, s.x1, K1);
    s.x0 = s.x1; s.x1 = s.x2; s.x2 = p1;
    double r;
    const uint32_t p2 = mrg_c2_floor(s.y0, s.y2, r, K);
    s.y0 = s.y1; s.y1 = s.y2; s.y2 = r;
    return mrg_combine(p1, p2);
}

template <int V>
__global__ void __launch_bounds__(256) k(uint32_t* out, const __grid_constant__ KP p, int iters)
{
    const MrgFpK K = kp(p);
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const Mrg s0 = seed_of(t);
    MrgIF s = to_mrg_if(s0);
    MrgFF f = to_mrg_ff(s0);
    MrgDI g{f.x0, f.x1, f.x2, f.y0, f.y1, f.y2};
    MrgSD sd{s0.x0, s0.x1, s0.x2, f.y0, f.y1, f.y2};
    const double K1 = __hiloint2double(p.k1hi, (int)p.k1lo);  // 202682 m1 * 2^-1074 (subnormal)
    Mrg ri = s0;
    uint32_t acc = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            uint32_t z;
            if (V == 0) {  // c2
                double r;
                z = mrg_c2_floor(s.y0, s.y2, r, K);
                s.y0 = s.y1; s.y1 = s.y2; s.y2 = r;
            } else if (V == 1) {  // c1
                z = mrg_c1_int(s.x0, s.x1, K.a12, K.a13n);
                s.x0 = s.x1; s.x1 = s.x2; s.x2 = z;
            } else if (V == 2) {
                z = mrg_next(s, K);
            } else if (V == 3) {
                z = mrg_next(f, K);
            } else if (V == 5) {
                z = next_di(g, K);
            } else if (V == 6) {
                z = mrg_next(ri, K);
            } else if (V == 10) {
                z = next_sd(sd, K, K1);
            } else if (V >= 7) {  // mixed warps: warp w runs FF if w % (V - 5) == 0, else IF
                if (((t >> 5) % (V - 5)) == 0) z = mrg_next(f, K);
                else z = mrg_next(s, K);
            } else {  // if_nocmb
                const uint32_t p1 = mrg_c1_int(s.x0, s.x1, K.a12, K.a13n);
                s.x0 = s.x1; s.x1 = s.x2; s.x2 = p1;
                double r;
                const uint32_t p2 = mrg_c2_floor(s.y0, s.y2, r, K);
                s.y0 = s.y1; s.y1 = s.y2; s.y2 = r;
                z = p1 ^ p2;
            }
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
    const uint64_t k1 = 202682ull * 4294967087ull;
    KP p{{6755399441055744.0, 1.0 / 4294967087.0, 0x1.000059451f212p-32, 4294967087.0, 4294944443.0, 5886603609186927.0}, 1403580u, 810728u,
         (uint32_t)k1, (uint32_t)(k1 >> 32)};
    uint32_t* o; cudaMalloc(&o, (size_t)sms * 16 * 256 * 4);
    const int iters = 1024;
    const char* names[] = {"c2", "c1", "if", "ff", "if_nocmb", "di", "int", "mix2", "mix3", "mix4", "sd"};
    printf("{");
    auto run = [&](int v, auto kern) {
        for (int bps : {4, 8}) {
            const size_t n = (size_t)sms * bps * 256;
            float ms = tms([&] { kern<<<sms * bps, 256>>>(o, p, iters); });
            printf("\"%s_b%d\": %.4f, ", names[v], bps, (double)n * iters * 8 / (ms * 1e-3) / 1e12);
        }
    };
    run(0, k<0>); run(1, k<1>); run(2, k<2>); run(3, k<3>); run(4, k<4>); run(5, k<5>); run(6, k<6>); run(10, k<10>);
    // full-step variants must give the integer step's sequence
    const size_t n = (size_t)sms * 8 * 256;
    uint32_t* h = new uint32_t[n]; uint32_t* ref = new uint32_t[n];
    k<6><<<sms * 8, 256>>>(o, p, 64); cudaMemcpy(ref, o, n * 4, cudaMemcpyDeviceToHost);
    for (int v : {2, 3, 5, 10}) {
        if (v == 2) k<2><<<sms * 8, 256>>>(o, p, 64);
        if (v == 3) k<3><<<sms * 8, 256>>>(o, p, 64);
        if (v == 5) k<5><<<sms * 8, 256>>>(o, p, 64);
        if (v == 10) k<10><<<sms * 8, 256>>>(o, p, 64);
        cudaMemcpy(h, o, n * 4, cudaMemcpyDeviceToHost);
        size_t bad = 0; for (size_t i = 0; i < n; ++i) bad += h[i] != ref[i];
        printf("\"%s_mismatch\": %zu, ", names[v], bad);
    }
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
}
