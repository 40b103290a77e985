// step_lab.cu — compute-only throughput of the generator steps in
// shv_device.cuh (no stores): numbers per SM per clock for the integer and
// hybrid MRG32k3a steps, the Philox4x32-10 block, and the MC sample. Also
// checks that the integer and hybrid steps produce identical sequences.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "lab_variants.cuh"
using namespace shv::dev;

constexpr int ITER = 2048;  // x 8 steps

template <class G>
__global__ void k_mrg(uint32_t* out)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    Mrg s0{12345u + t, 12345u, 12345u ^ t, 12345u, 777u + t, 12345u};
    G s;
    if constexpr (sizeof(G) == sizeof(Mrg)) s = s0; else if constexpr (sizeof(G) == sizeof(MrgD)) s = to_fp64(s0); else if constexpr (sizeof(G) == sizeof(MrgS)) s = to_fp64s(s0); else if constexpr (sizeof(G) == sizeof(MrgW)) s = to_fp64w(s0); else s = to_hybrid(s0);
    uint32_t acc = 0;
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = acc * 3u + mrg_next(s);
    }
    out[t] = acc;
}

template <int V>
__global__ void k_mrgv(uint32_t* out)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    Mrg s0{12345u + t, 12345u, 12345u ^ t, 12345u, 777u + t, 12345u};
    MrgDV<V> s = to_fp64v<V>(s0);
    uint32_t acc = 0;
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = acc * 3u + mrg_next(s);
    }
    out[t] = acc;
}

// Two independent streams per thread, interleaved (ILP 2).
__global__ void k_mrg2(uint32_t* out)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    Mrg s0{12345u + t, 12345u, 12345u ^ t, 12345u, 777u + t, 12345u};
    Mrg s1{12345u + t + 7, 12345u, 12345u ^ (t + 7), 12345u, 777u + t + 7, 12345u};
    MrgD a = to_fp64(s0), b = to_fp64(s1);
    uint32_t acc = 0, acc2 = 0;
    for (int i = 0; i < ITER / 2; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) { acc = acc * 3u + mrg_next(a); acc2 = acc2 * 3u + mrg_next(b); }
    }
    out[t] = acc ^ acc2;
}

template <class G>
__global__ void k_mc(uint32_t* out)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    Mrg s0{12345u + t, 12345u, 12345u ^ t, 12345u, 777u + t, 12345u};
    G s;
    if constexpr (sizeof(G) == sizeof(Mrg)) s = s0; else s = to_hybrid(s0);
    uint32_t h = 0;
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) { uint32_t a = mrg_next(s); uint32_t b = mrg_next(s); h += hit(a, b); }
    }
    out[t] = h;
}

__global__ void k_philox(uint32_t* out, uint32_t k0, uint32_t k1)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int i = 0; i < ITER; ++i) {
        W4 a = philox10(i, 0, t, 0, k0, k1);
        W4 b = philox10(i + ITER, 0, t, 0, k0, k1);
        acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
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
    const int threads = 256;
    int occ_i, occ_h, occ_p, occ_mi, occ_mh;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_i, k_mrg<Mrg>, threads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_h, k_mrg<MrgH>, threads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_p, k_philox, threads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_mi, k_mc<Mrg>, threads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_mh, k_mc<MrgH>, threads, 0);
    const int blocks = sms * 8;
    const double thr = (double)blocks * threads;
    uint32_t *o1, *o2; cudaMalloc(&o1, thr * 4); cudaMalloc(&o2, thr * 4);
    // clock
    float ti = tms([&] { k_mrg<Mrg><<<blocks, threads>>>(o1); });
    float th = tms([&] { k_mrg<MrgH><<<blocks, threads>>>(o2); });
    uint32_t* h1 = new uint32_t[(size_t)thr]; uint32_t* h2 = new uint32_t[(size_t)thr];
    cudaMemcpy(h1, o1, thr * 4, cudaMemcpyDeviceToHost); cudaMemcpy(h2, o2, thr * 4, cudaMemcpyDeviceToHost);
    size_t bad = 0; for (size_t i = 0; i < (size_t)thr; ++i) bad += h1[i] != h2[i];
    float td = tms([&] { k_mrg<MrgD><<<blocks, threads>>>(o2); });
    cudaMemcpy(h2, o2, thr * 4, cudaMemcpyDeviceToHost);
    size_t bad3 = 0; for (size_t i = 0; i < (size_t)thr; ++i) bad3 += h1[i] != h2[i];
    float ts = tms([&] { k_mrg<MrgS><<<blocks, threads>>>(o2); });
    cudaMemcpy(h2, o2, thr * 4, cudaMemcpyDeviceToHost);
    size_t bad4 = 0; for (size_t i = 0; i < (size_t)thr; ++i) bad4 += h1[i] != h2[i];
    float tw = tms([&] { k_mrg<MrgW><<<blocks, threads>>>(o2); });
    cudaMemcpy(h2, o2, thr * 4, cudaMemcpyDeviceToHost);
    size_t bad5 = 0; for (size_t i = 0; i < (size_t)thr; ++i) bad5 += h1[i] != h2[i];
    for (int v = 2; v <= 4; ++v) {
        float tv = v == 2 ? tms([&] { k_mrgv<2><<<blocks, threads>>>(o2); }) : v == 3 ? tms([&] { k_mrgv<3><<<blocks, threads>>>(o2); }) : tms([&] { k_mrgv<4><<<blocks, threads>>>(o2); });
        cudaMemcpy(h2, o2, thr * 4, cudaMemcpyDeviceToHost);
        size_t b = 0; for (size_t i = 0; i < (size_t)thr; ++i) b += h1[i] != h2[i];
        printf("{\"variant\": %d, \"Gnum_s\": %.1f, \"mismatch\": %zu}\n", v, thr * ITER * 8 / (tv * 1e6), b);
    }
    float t2 = tms([&] { k_mrg2<<<blocks, threads>>>(o2); });
    int occ2; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_mrg2, threads, 0);
    float t2h = tms([&] { k_mrg2<<<sms * 4, threads>>>(o2); });
    printf("{\"mrg_fp64_ilp2_Gnum_s\": %.1f, \"occ\": %d, \"half_grid_Gnum_s\": %.1f}\n", thr * ITER * 8 / (t2 * 1e6), occ2, thr / 2 * ITER * 8 / (t2h * 1e6));
    float tp = tms([&] { k_philox<<<blocks, threads>>>(o1, 12345, 0); });
    float tmi = tms([&] { k_mc<Mrg><<<blocks, threads>>>(o1); });
    float tmh = tms([&] { k_mc<MrgH><<<blocks, threads>>>(o2); });
    cudaMemcpy(h1, o1, thr * 4, cudaMemcpyDeviceToHost); cudaMemcpy(h2, o2, thr * 4, cudaMemcpyDeviceToHost);
    size_t bad2 = 0; for (size_t i = 0; i < (size_t)thr; ++i) bad2 += h1[i] != h2[i];
    const double n = thr * ITER * 8;
    printf("{\"occ_blocks\": [%d, %d, %d, %d, %d], \"mrg_int_Gnum_s\": %.1f, \"mrg_hybrid_Gnum_s\": %.1f, "
           "\"philox_Gnum_s\": %.1f, \"mc_int_Gsamples_s\": %.1f, \"mc_hybrid_Gsamples_s\": %.1f, "
           "\"int_vs_hybrid_mismatch\": %zu, \"mc_mismatch\": %zu, \"mrg_fp64_Gnum_s\": %.1f, \"fp64_mismatch\": %zu, \"mrg_fp64short_Gnum_s\": %.1f, \"short_mismatch\": %zu, \"mrg_fp64w_Gnum_s\": %.1f, \"w_mismatch\": %zu}\n",
           occ_i, occ_h, occ_p, occ_mi, occ_mh, n / (ti * 1e6), n / (th * 1e6), n / (tp * 1e6),
           n / 2 / (tmi * 1e6), n / 2 / (tmh * 1e6), bad, bad2, n / (td * 1e6), bad3, n / (ts * 1e6), bad4, n / (tw * 1e6), bad5);
    return 0;
}
