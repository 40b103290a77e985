// concurrent_lab.cu — MRG32k3a and Philox4x32-10 C5 fills issued on two CUDA
// streams at once (the step's two generators are independent), over a grid of
// per-handle launch configurations (blocks per SM). usage: concurrent_lab lib.so
#include <dlfcn.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/shv.h"
#define F(name) auto name = (decltype(&::name))dlsym(h, #name); if (!name) { printf("missing %s\n", #name); return 1; }
int main(int argc, char** argv)
{
    void* h = dlopen(argv[1], RTLD_NOW | RTLD_LOCAL);
    F(shv_streams_create_ex) F(shv_generate_u32) F(shv_streams_destroy) F(shv_set_launch_config)
    const uint64_t ns = 1 << 20, n = 4096;
    uint32_t *o1, *o2, *st;
    cudaMalloc(&o1, ns * n * 4); cudaMalloc(&o2, ns * n * 4); cudaMalloc(&st, 24 * ns);
    cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t a, b1, b2; cudaEventCreate(&a); cudaEventCreate(&b1); cudaEventCreate(&b2);
    uint32_t seed = 12345;
    shv_streams hm, hp;
    shv_streams_create_ex(&hm, 1, &seed, 1, 0, ns, 1, st, 24 * ns, 0, s1);
    shv_streams_create_ex(&hp, 2, &seed, 1, 0, ns, 0, nullptr, 0, 0, s2);
    int cfg[][2] = {{0, 0}, {3, 0}, {2, 2}, {2, 3}, {1, 4}, {2, 1}, {1, 2}, {3, 2}};
    printf("{\"results\": [");
    for (int c = 0; c < 8; ++c) {
        shv_set_launch_config(hm, cfg[c][0], 0, 0);
        shv_set_launch_config(hp, cfg[c][1], 0, 0);
        float best = 1e30f;
        for (int r = 0; r < 6; ++r) {
            cudaDeviceSynchronize();
            cudaEventRecord(a, s1);
            cudaStreamWaitEvent(s2, a, 0);
            shv_generate_u32(hm, o1, n, s1);
            shv_generate_u32(hp, o2, n, s2);
            cudaEventRecord(b2, s2);
            cudaStreamWaitEvent(s1, b2, 0);
            cudaEventRecord(b1, s1);
            cudaEventSynchronize(b1);
            float ms; cudaEventElapsedTime(&ms, a, b1);
            if (r && ms < best) best = ms;
        }
        printf("%s{\"mrg_bps\": %d, \"philox_bps\": %d, \"ms\": %.4f, \"GBps\": %.1f}", c ? ", " : "", cfg[c][0], cfg[c][1], best, 2.0 * ns * n * 4 / (best * 1e-3) / 1e9);
    }
    printf("], \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
}
