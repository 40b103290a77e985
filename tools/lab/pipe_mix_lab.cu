// pipe_mix_lab.cu — do the FP64, FMA-heavy (IMAD / IMAD.WIDE) and ALU pipes of
// a B200 SM issue side by side? Each kernel runs independent chains of one or
// two instruction kinds (8 chains per kind per thread, full occupancy) and
// reports per-kind instructions per SM per clock. If two kinds share a pipe,
// their rates add up to one pipe's rate instead of each reaching its own.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_mix_lab tools/lab/pipe_mix_lab.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int IT = 2048;
constexpr int CH = 8;

// kinds: 0 none, 1 DFMA (imm form), 2 IMAD, 3 IMAD.WIDE (C = dest), 4 LOP3 (ALU), 5 DFMA (3 reg pairs)
template <int KA, int KB>
__global__ void __launch_bounds__(256) k_mix(uint32_t* out, uint32_t s, double ds, double dm)
{
    double d[CH], e[CH];
    uint32_t a[CH];
    uint64_t w[CH];
    uint32_t b[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        d[c] = threadIdx.x + c * 0.5 + ds;
        e[c] = threadIdx.x * 0.25 + c + ds;
        a[c] = threadIdx.x * 7u + c + s;
        w[c] = ((uint64_t)(threadIdx.x + c) << 32) | (s + c);
        b[c] = threadIdx.x ^ (c * 977u) ^ s;
    }
    for (int i = 0; i < IT; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
#define SHV_OP(K)                                                                                                    \
    if (K == 1) asm volatile("fma.rn.f64 %0, %0, 0d3FEFFFFFFFFFFFEF, %1;" : "+d"(d[c]) : "d"(ds));                     \
    if (K == 5) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(e[c]) : "d"(dm), "d"(d[(c + 1) % CH]));              \
    if (K == 2) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(s | 1u), "r"(s));                          \
    if (K == 3) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[c]) : "r"((uint32_t)w[(c + 1) % CH]), "r"(s | 3u)); \
    if (K == 4) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(b[c]) : "r"(b[(c + 3) % CH]), "r"(s));
            SHV_OP(KA)
            SHV_OP(KB)
#undef SHV_OP
        }
    }
    uint64_t r = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) r ^= (uint64_t)__double_as_longlong(d[c]) ^ (uint64_t)__double_as_longlong(e[c]) ^ a[c] ^ w[c] ^ b[c];
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
    const double per = (double)blocks * thr * IT * CH;  // ops per kind
    const char* nm[] = {"none", "dfma_imm", "imad", "imad_wide", "lop3", "dfma_3reg"};
    auto run = [&](auto kern, int ka, int kb) {
        float ms = tms([&] { kern<<<blocks, thr>>>(o, 12345u, 0.5, 0.999999); });
        // ops per SM per clock at the nominal (max) clock
        const double rate = per / (ms * 1e-3) / sms / (clk * 1e3);
        printf("{\"a\": \"%s\", \"b\": \"%s\", \"ms\": %.3f, \"per_kind_per_sm_clk\": %.2f}\n", nm[ka], nm[kb], ms, rate);
    };
    run(k_mix<1, 0>, 1, 0);
    run(k_mix<5, 0>, 5, 0);
    run(k_mix<2, 0>, 2, 0);
    run(k_mix<3, 0>, 3, 0);
    run(k_mix<4, 0>, 4, 0);
    run(k_mix<1, 2>, 1, 2);
    run(k_mix<1, 3>, 1, 3);
    run(k_mix<1, 4>, 1, 4);
    run(k_mix<2, 4>, 2, 4);
    run(k_mix<3, 4>, 3, 4);
    run(k_mix<3, 2>, 3, 2);
    run(k_mix<5, 3>, 5, 3);
    return 0;
}
