// fp64_mix_lab.cu — FP64 throughput of the MRG32k3a floor-reduction instruction
// mix (DMUL, DFMA, DFMA.RM, DADD, DFMA, DADD per component) in S independent
// dependency chains per thread, to separate the pipe's rate for this mix from
// the dependency structure of the real step.
#include <cstdio>
#include <cuda_runtime.h>

template <int S>
__global__ void __launch_bounds__(256) k_mix(double* out, int iters, double inv, double magic, double m)
{
    double x0[S], x1[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        x0[s] = 1000.0 + threadIdx.x + s;
        x1[s] = 7.0 * blockIdx.x + s;
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const double t = __dmul_rn(810728.0, x0[s]);
            const double p = __fma_rn(1403580.0, x1[s], -t);
            const double k = __dadd_rn(__fma_rd(p, inv, magic), -magic);
            const double r = __fma_rn(-k, m, p);
            const double o = __dadd_rn(r, magic);
            x0[s] = x1[s];
            x1[s] = __dadd_rn(r, __hiloint2double(0, __double2loint(o) & 1));  // keep o live, tiny perturbation
        }
    }
    double acc = 0;
#pragma unroll
    for (int s = 0; s < S; ++s) acc += x1[s];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int S>
void run(int sms, double* out)
{
    const int iters = 4096, blocks = sms * 8;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_mix<S><<<blocks, 256>>>(out, 16, 1.0 / 4294967087.0, 6755399441055744.0, 4294967087.0);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a);
        k_mix<S><<<blocks, 256>>>(out, iters, 1.0 / 4294967087.0, 6755399441055744.0, 4294967087.0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    const double ops = (double)blocks * 256 * iters * S * 7;  // 7 FP64 instructions per chain step
    printf("{\"chains\": %d, \"fp64_T_per_s\": %.2f, \"per_sm_per_ns\": %.1f}\n", S, ops / (best * 1e-3) / 1e12,
           ops / (best * 1e6) / sms);
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, (size_t)sms * 8 * 256 * 8);
    run<1>(sms, out);
    run<2>(sms, out);
    run<4>(sms, out);
    return 0;
}
