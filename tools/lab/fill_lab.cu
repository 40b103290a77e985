// fill_lab.cu — kernel lab: times the C5 fills (2^20 streams x 4096 u32) of
// one libshv build variant through its C ABI and prints a device checksum, so
// variants (tools/lab/build_variants.sh) can be compared for speed and for
// bit-identical output.   usage: fill_lab <libshv.so> [reps]
#include <dlfcn.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/shv.h"

__global__ void checksum(const uint32_t* v, uint64_t n, unsigned long long* out)
{
    unsigned long long s = 0, x = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        s += v[i];
        x ^= (unsigned long long)v[i] * (2 * i + 1);
    }
    atomicAdd(out, s);
    atomicXor(out + 1, x);
}

#define F(name) auto name = (decltype(&::name))dlsym(h, #name); if (!name) { printf("missing %s\n", #name); return 1; }

int main(int argc, char** argv)
{
    void* h = dlopen(argv[1], RTLD_NOW | RTLD_LOCAL);
    if (!h) { printf("dlopen: %s\n", dlerror()); return 1; }
    const int reps = argc > 2 ? atoi(argv[2]) : 10;
    F(shv_streams_create_ex) F(shv_generate_u32) F(shv_streams_destroy) F(shv_last_error_message) F(shv_generate_f64) F(shv_mc_pi) F(shv_set_launch_config)
    const unsigned tpb = argc > 3 ? (unsigned)atoi(argv[3]) : 0;
    const unsigned bps = argc > 4 ? (unsigned)atoi(argv[4]) : 0;
    const int only_u32 = argc > 5 ? atoi(argv[5]) : 0;
    const uint64_t ns = 1 << 20, n = 4096;
    uint32_t* out; uint32_t* st; unsigned long long* ck;
    cudaMalloc(&out, ns * n * 8); cudaMalloc(&st, 24 * ns); cudaMalloc(&ck, 16);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    uint32_t seed = 12345;
    printf("{\"lib\": \"%s\"", argv[1]);
    for (int gen = 1; gen <= 2; ++gen) {
        for (int kind = 0; kind < (only_u32 ? 1 : 2); ++kind) {
            shv_streams hd;
            uint64_t nsk = kind ? ns / 2 : ns;  // f64: 16 GiB
            if (shv_streams_create_ex(&hd, gen, &seed, 1, 0, nsk, gen == 1 ? 1 : 0, gen == 1 ? st : nullptr, 24 * ns, 0, 0)) {
                printf("create: %s\n", shv_last_error_message()); return 1; }
            if (tpb || bps) shv_set_launch_config(hd, bps, tpb, 0);
            float best = 1e30f, sum = 0;
            for (int r = 0; r < reps + 2; ++r) {
                cudaEventRecord(a);
                int rc = kind ? shv_generate_f64(hd, (double*)out, n, 0) : shv_generate_u32(hd, out, n, 0);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                if (rc) { printf("gen: %s\n", shv_last_error_message()); return 1; }
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (r >= 2) { sum += ms; if (ms < best) best = ms; }
            }
            cudaMemset(ck, 0, 16);
            checksum<<<1184, 256>>>(out, nsk * n * (kind ? 2 : 1), ck);
            unsigned long long hck[2];
            cudaMemcpy(hck, ck, 16, cudaMemcpyDeviceToHost);
            const double bytes = (double)nsk * n * (kind ? 8 : 4);
            printf(", \"%s_%s\": {\"ms_best\": %.4f, \"ms_mean\": %.4f, \"GBps\": %.1f, \"sum\": \"%016llx\", \"wxor\": \"%016llx\"}",
                   gen == 1 ? "mrg" : "philox", kind ? "f64" : "u32", best, sum / reps, bytes / (best * 1e-3) / 1e9, hck[0], hck[1]);
            shv_streams_destroy(hd);
        }
        if (only_u32) continue;
        // MC pi, 2^38 samples
        shv_streams hd;
        shv_streams_create_ex(&hd, gen, &seed, 1, 0, ns, gen == 1 ? 1 : 0, gen == 1 ? st : nullptr, 24 * ns, 0, 0);
        cudaMemset(ck, 0, 8);
        cudaEventRecord(a);
        shv_mc_pi(hd, 1 << 18, (uint64_t*)ck, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        unsigned long long hits; cudaMemcpy(&hits, ck, 8, cudaMemcpyDeviceToHost);
        printf(", \"%s_mc\": {\"ms\": %.2f, \"Gsamples\": %.1f, \"hits\": %llu}", gen == 1 ? "mrg" : "philox", ms, 274877906944.0 / (ms * 1e-3) / 1e9, hits);
        shv_streams_destroy(hd);
    }
    printf("}\n");
    return 0;
}
