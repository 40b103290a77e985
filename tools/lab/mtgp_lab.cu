// mtgp_lab.cu — times the MTGP32 fill (200 states x 2^32/200 u32) of one
// libshv build variant (SHV_MT_THREADS / SHV_MT_EPT) through its C ABI and
// prints a checksum so variants can be compared for speed and identical output.
// Parameter sets: the toolkit's MTGP32-11213 DC table (lab input only).
//   usage: mtgp_lab <libshv.so> [reps]
#include <dlfcn.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include <curand_mtgp32dc_p_11213.h>
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
    const int reps = argc > 2 ? atoi(argv[2]) : 5;
    F(shv_streams_create_mtgp32) F(shv_generate_u32) F(shv_streams_destroy) F(shv_last_error_message) F(shv_mc_pi)
    std::vector<uint32_t> prm;
    for (int i = 0; i < 200; ++i) {
        const mtgp32_params_fast_t& q = mtgp32dc_params_fast_11213[i];
        prm.push_back(q.pos); prm.push_back(q.sh1); prm.push_back(q.sh2); prm.push_back(q.mask);
        for (int j = 0; j < 16; ++j) prm.push_back(q.tbl[j]);
        for (int j = 0; j < 16; ++j) prm.push_back(q.tmp_tbl[j]);
    }
    const uint64_t ns = 200, n = (1ull << 32) / 200;
    uint32_t* out; cudaMalloc(&out, ns * n * 4);
    unsigned long long* cs; cudaMalloc(&cs, 16); cudaMemset(cs, 0, 16);
    shv_streams hd;
    if (shv_streams_create_mtgp32(&hd, prm.data(), 200, 12345, 0, ns, nullptr, 0, 0, nullptr)) { printf("create: %s\n", shv_last_error_message()); return 1; }
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e30f, sum = 0;
    for (int r = 0; r <= reps; ++r) {
        cudaEventRecord(a);
        shv_generate_u32(hd, out, n, nullptr);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (r) { best = ms < best ? ms : best; sum += ms; }
        if (r == 0) checksum<<<1184, 256>>>(out, ns * n, cs);
    }
    unsigned long long* hits; cudaMalloc(&hits, 8); cudaMemset(hits, 0, 8);
    cudaEventRecord(a);
    shv_mc_pi(hd, n / 2, (uint64_t*)hits, nullptr);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float mc; cudaEventElapsedTime(&mc, a, b);
    unsigned long long hc[2], hh; cudaMemcpy(hc, cs, 16, cudaMemcpyDeviceToHost); cudaMemcpy(&hh, hits, 8, cudaMemcpyDeviceToHost);
    printf("{\"lib\": \"%s\", \"ms_best\": %.3f, \"ms_mean\": %.3f, \"Gnum_s\": %.1f, \"sum\": \"%016llx\", \"wxor\": \"%016llx\", \"mc_ms\": %.3f, \"mc_hits\": %llu, \"err\": \"%s\"}\n",
           argv[1], best, sum / reps, ns * n / (best * 1e-3) / 1e9, hc[0], hc[1], mc, hh, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
