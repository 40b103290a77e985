// fp64_lab.cu — throughput of individual FP64 instruction forms on B200
// (per SM per clock), to explain the MRG32k3a FP64 step's pipe usage.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int IT = 2048, CH = 8;
template <int K>
__global__ void k(double* out, double s, double u)
{
    double a[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < IT; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (K == 0) a[c] = __dadd_rn(a[c], 6755399441055744.0);           // DADD imm
            if (K == 1) a[c] = __dmul_rn(a[c], 1370589.0);                    // DMUL imm
            if (K == 2) a[c] = __fma_rn(a[c], 527612.0, a[(c + 1) % CH]);     // DFMA imm, 2 reg pairs
            if (K == 3) a[c] = __fma_rn(a[c], u, a[(c + 1) % CH]);            // DFMA uniform, 2 pairs
            if (K == 4) a[c] = __fma_rn(a[c], a[(c + 2) % CH], a[(c + 1) % CH]);  // DFMA 3 pairs
            if (K == 5) a[c] = __dadd_rn(a[c], a[(c + 1) % CH]);              // DADD 2 pairs
            if (K == 6) a[c] = __dmul_rn(a[c], a[(c + 1) % CH]);              // DMUL 2 pairs
            if (K == 7) a[c] = __fma_rd(a[c], u, a[(c + 1) % CH]);            // DFMA.RM uniform, 2 pairs
            if (K == 8) a[c] = __fma_rn(a[c], 1e-300, 0.5);                   // DFMA imm + const, 1 pair
        }
    }
    double r = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) r += a[c];
    if (r == 1.2345) out[0] = r;
}
template <class F> float tms(F f) { cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); f(); cudaDeviceSynchronize();
    float best = 1e30f; for (int r = 0; r < 5; ++r) { cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; } return best; }
int main()
{
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* o; cudaMalloc(&o, 8);
    const int blocks = sms * 8, thr = 256;
    const char* names[] = {"dadd_imm", "dmul_imm", "dfma_imm_2pairs", "dfma_ur_2pairs", "dfma_3pairs", "dadd_2pairs", "dmul_2pairs", "dfma_rm_ur_2pairs", "dfma_1pair"};
    float t[9];
    t[0] = tms([&] { k<0><<<blocks, thr>>>(o, 1.0, 0.5); });
    t[1] = tms([&] { k<1><<<blocks, thr>>>(o, 1.0, 0.5); });
    t[2] = tms([&] { k<2><<<blocks, thr>>>(o, 1.0, 0.5); });
    t[3] = tms([&] { k<3><<<blocks, thr>>>(o, 1.0, 0.5); });
    t[4] = tms([&] { k<4><<<blocks, thr>>>(o, 1.0, 0.5); });
    t[5] = tms([&] { k<5><<<blocks, thr>>>(o, 1.0, 0.5); });
    t[6] = tms([&] { k<6><<<blocks, thr>>>(o, 1.0, 0.5); });
    t[7] = tms([&] { k<7><<<blocks, thr>>>(o, 1.0, 0.5); });
    t[8] = tms([&] { k<8><<<blocks, thr>>>(o, 1.0, 0.5); });
    printf("{");
    for (int i = 0; i < 9; ++i)  // ops per SM per ns (divide by GHz for per clock)
        printf("%s\"%s_per_sm_per_ns\": %.2f", i ? ", " : "", names[i], (double)blocks * thr * IT * CH / (t[i] * 1e6) / sms);
    printf("}\n");
}
