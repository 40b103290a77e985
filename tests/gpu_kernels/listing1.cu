// listing1.cu — TEST-ONLY user kernel in the style of the paper's Listing 1
// (P L480-499), written against the public device API include/shv_rng.cuh.
// Built by tests/test_gpu_device_api.py with nvcc; not part of the product.
#include <cstdint>
#include <cuda_runtime.h>
#include "shv_rng.cuh"

template <int GEN, int KIND>
__global__ void fooKernel(void* ddata, shv_device_view v, int per_thread)
{
    const uint64_t i = (uint64_t)blockDim.x * blockIdx.x + threadIdx.x;
    if (i >= v.n_streams) return;
    shv::Rng<GEN> rng(v, i);
    for (int k = 0; k < per_thread; ++k) {
        const uint64_t at = i * per_thread + k;
        if (KIND == 0) static_cast<uint32_t*>(ddata)[at] = rng.next_u32();
        else if (KIND == 1) static_cast<float*>(ddata)[at] = rng.next_f32();
        else static_cast<double*>(ddata)[at] = rng.next_f64();
    }
}

template <int GEN>
static void launch(int kind, void* out, const shv_device_view& v, int per_thread, int blocks, int threads)
{
    if (kind == 0) fooKernel<GEN, 0><<<blocks, threads>>>(out, v, per_thread);
    else if (kind == 1) fooKernel<GEN, 1><<<blocks, threads>>>(out, v, per_thread);
    else fooKernel<GEN, 2><<<blocks, threads>>>(out, v, per_thread);
}

extern "C" int launch_listing1(int gen, int kind, void* out, const shv_device_view* v, int per_thread,
                               int blocks, int threads)
{
    if (gen == SHV_GEN_MRG32K3A) launch<SHV_GEN_MRG32K3A>(kind, out, *v, per_thread, blocks, threads);
    else if (gen == SHV_GEN_TINYMT32) launch<SHV_GEN_TINYMT32>(kind, out, *v, per_thread, blocks, threads);
    else if (gen == SHV_GEN_THREEFRY4X64_20) launch<SHV_GEN_THREEFRY4X64_20>(kind, out, *v, per_thread, blocks, threads);
    else launch<SHV_GEN_PHILOX4X32_10>(kind, out, *v, per_thread, blocks, threads);
    return (int)cudaDeviceSynchronize();
}
