// pipe_mix2_lab.cu — per-instruction throughput on a B200 SM, alone and in
// pairs, for the instruction kinds an exact MRG32k3a step can use (extends
// pipe_mix_lab.cu). 8 independent chains per kind per thread, 8 x 256 threads
// per SM; prints each kind's warp-lane ops per SM per clock (64 = a 16-lane
// pipe per SMSP at one warp instruction every 2 clocks).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_mix2_lab tools/lab/pipe_mix2_lab.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int IT = 1024;
constexpr int CH = 8;

// kinds
enum { NONE, DFMA, IMAD, IMADW, LOP3, I2FD, IMADHI, SHF, ISETP, VIADD, IADD3, DADD, FFMA, IMADSHL, SEL, LEA, NK };
static const char* nm[] = {"none", "dfma", "imad", "imad_wide", "lop3", "i2f_f64", "imad_hi", "shf",
                           "isetp", "viadd", "iadd3", "dadd", "ffma", "imad_shl", "sel", "lea"};

template <int K>
__device__ __forceinline__ void op(int c, double* d, uint32_t* a, uint64_t* w, float* f, uint32_t s)
{
    if (K == DFMA) asm volatile("fma.rn.f64 %0, %0, 0d3FEFFFFFFFFFFFEF, %1;" : "+d"(d[c]) : "d"(d[(c + 1) % CH]));
    if (K == DADD) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(d[c]) : "d"(d[(c + 1) % CH]));
    if (K == IMAD) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(s | 1u), "r"(a[(c + 1) % CH]));
    if (K == IMADW) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[c]) : "r"((uint32_t)w[(c + 1) % CH]), "r"(s | 3u));
    if (K == IMADHI) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(a[c]) : "r"(s | 3u));
    if (K == LOP3) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[c]) : "r"(a[(c + 3) % CH]), "r"(s));
    if (K == I2FD) {
        double t;
        asm volatile("cvt.rn.f64.u32 %0, %1;" : "=d"(t) : "r"(a[c]));
        asm volatile("mov.b64 {%0, %1}, %2;" : "=r"(a[c]), "=r"(a[(c + 4) % CH]) : "d"(t));
    }
    if (K == SHF) asm volatile("shf.l.wrap.b32 %0, %0, %1, 7;" : "+r"(a[c]) : "r"(a[(c + 1) % CH]));
    if (K == ISETP) {
        asm volatile("{.reg .pred p; setp.lt.u32 p, %0, %1; selp.u32 %0, %0, %2, p;}" : "+r"(a[c]) : "r"(a[(c + 1) % CH]), "r"(s));
    }
    if (K == VIADD) asm volatile("add.u32 %0, %0, 209;" : "+r"(a[c]));
    if (K == IADD3) asm volatile("add.u32 %0, %0, %1;" : "+r"(a[c]) : "r"(a[(c + 2) % CH]));
    if (K == FFMA) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFF0, %1;" : "+f"(f[c]) : "f"(f[(c + 1) % CH]));
    if (K == IMADSHL) asm volatile("shl.b32 %0, %0, 2;" : "+r"(a[c]));
    if (K == SEL) asm volatile("{.reg .pred p; setp.ne.u32 p, %1, 0; selp.u32 %0, %0, %2, p;}" : "+r"(a[c]) : "r"(s), "r"(a[(c + 1) % CH]));
    if (K == LEA) asm volatile("{.reg .u32 t; shl.b32 t, %0, 2; add.u32 %0, t, %1;}" : "+r"(a[c]) : "r"(a[(c + 5) % CH]));
}

template <int KA, int KB>
__global__ void __launch_bounds__(256) k_mix(uint32_t* out, uint32_t s)
{
    double d[CH];
    uint32_t a[CH];
    uint64_t w[CH];
    float f[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        d[c] = threadIdx.x + c * 0.5;
        a[c] = threadIdx.x * 7u + c + s;
        w[c] = ((uint64_t)(threadIdx.x + c) << 32) | (s + c);
        f[c] = threadIdx.x + c * 0.25f;
    }
    for (int i = 0; i < IT; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            op<KA>(c, d, a, w, f, s);
            op<KB>(c, d, a, w, f, s);
        }
    }
    uint64_t r = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) r ^= (uint64_t)__double_as_longlong(d[c]) ^ a[c] ^ w[c] ^ __float_as_uint(f[c]);
    if (r == 0x12345678ull) out[0] = (uint32_t)r;
}

template <class F>
float tms(F f)
{
    cudaEvent_t x, y; cudaEventCreate(&x); cudaEventCreate(&y);
    f(); cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(x); f(); cudaEventRecord(y); cudaEventSynchronize(y);
        float ms; cudaEventElapsedTime(&ms, x, y); if (ms < best) best = ms; }
    return best;
}

int main()
{
    int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    uint32_t* o; cudaMalloc(&o, 4);
    const int blocks = sms * 8, thr = 256;
    const double per = (double)blocks * thr * IT * CH;
    auto run = [&](auto kern, int ka, int kb) {
        float ms = tms([&] { kern<<<blocks, thr>>>(o, 12345u); });
        const double rate = per / (ms * 1e-3) / sms / (clk * 1e3);
        printf("{\"a\": \"%s\", \"b\": \"%s\", \"per_kind_per_sm_clk\": %.2f}\n", nm[ka], nm[kb], rate);
    };
#define A(x) run(k_mix<x, NONE>, x, NONE);
    A(DFMA) A(DADD) A(IMAD) A(IMADW) A(IMADHI) A(LOP3) A(I2FD) A(SHF) A(ISETP) A(VIADD) A(IADD3) A(FFMA) A(IMADSHL) A(SEL) A(LEA)
#define P(x, y) run(k_mix<x, y>, x, y);
    P(DFMA, LOP3) P(DFMA, IADD3) P(DFMA, ISETP) P(DFMA, SHF) P(DFMA, I2FD) P(DFMA, IMAD) P(DFMA, VIADD) P(DFMA, IMADSHL)
    P(DFMA, LEA) P(DFMA, SEL) P(IMAD, IADD3) P(IMAD, ISETP) P(VIADD, LOP3) P(VIADD, IMAD) P(I2FD, LOP3) P(IMADHI, LOP3)
    P(IMADW, DFMA) P(FFMA, DFMA) P(FFMA, LOP3) P(IADD3, LOP3)
    return 0;
}
