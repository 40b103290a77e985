// tma_store_lab.cu — write bandwidth of TMA / bulk-copy store shapes for the
// MRG fill's row layout (2^20 rows x 4096 u32 = 16 GiB): a warp owns 32 rows
// and walks them in rounds; shared memory holds garbage (bandwidth only).
//   A: 2D box 32 rows x 128 B, 128-B swizzle, 1 box per round
//   B: 2D box 32 rows x 256 B, no swizzle
//   C: 2D box 32 rows x 512 B, no swizzle
//   D: 2 A-boxes per round (256 B per row per round)
//   E: 4 A-boxes per round
//   F: 1D bulk copies, one 256-B piece per lane per round
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

constexpr uint64_t NS = 1ull << 20, N = 4096;

template <int MODE, int BOXB, int NBOX>
__global__ void __launch_bounds__(256) k(const __grid_constant__ CUtensorMap tm, uint32_t* out)
{
    extern __shared__ uint8_t sm[];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t base = ((uint32_t)__cvta_generic_to_shared(sm) + 1023u) & ~1023u;
    const uint32_t box = base + warp * (32u * BOXB * NBOX);
    const uint64_t G = NS / 32;
    const uint64_t wstride = (uint64_t)gridDim.x * (blockDim.x >> 5);
    constexpr uint32_t W = BOXB / 4;
    for (uint64_t g = (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp; g < G; g += wstride) {
        for (uint32_t c = 0; c < N; c += W * NBOX) {
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
            // touch shared memory like the fill would (one 16-B store per 8 values)
#pragma unroll
            for (uint32_t q = 0; q < BOXB * NBOX / 16; ++q)
                asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(box + ((lane * BOXB * NBOX + q * 16) % (32u * BOXB * NBOX))), "r"(c) : "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (MODE == 0) {
                if (lane == 0) {
#pragma unroll
                    for (int b = 0; b < NBOX; ++b)
                        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tm),
                                     "r"(box + b * 32u * BOXB), "r"((int)(c + b * W)), "r"((int)(32 * g)) : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
            } else {
                uint32_t* dst = out + (32 * g + lane) * N + c;
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(box + lane * BOXB), "n"(BOXB) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <class F> float tms(F f) { cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); f(); cudaDeviceSynchronize();
    float best = 1e30f; for (int r = 0; r < 5; ++r) { cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; } return best; }

int main()
{
    void* p = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    uint32_t* out; cudaMalloc(&out, NS * N * 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto mk = [&](int boxb, bool swz) { CUtensorMap m; cuuint64_t d[2] = {N, NS}; cuuint64_t st[1] = {N * 4};
        cuuint32_t bx[2] = {(cuuint32_t)boxb / 4, 32}; cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, out, d, st, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r) printf("encode %d failed %d\n", boxb, (int)r); return m; };
    const double bytes = (double)NS * N * 4;
    printf("{");
    auto run = [&](const char* name, auto kern, CUtensorMap m, int smem_per_warp, int tpb) {
        size_t smem = (size_t)(tpb / 32) * smem_per_warp + 1024;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int occ; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, tpb, smem);
        float ms = tms([&] { kern<<<sms * occ, tpb, smem>>>(m, out); });
        cudaError_t e = cudaGetLastError();
        printf("\"%s_tpb%d\": {\"GBps\": %.1f, \"occ\": %d, \"err\": %d}, ", name, tpb, bytes / (ms * 1e-3) / 1e9, occ, (int)e);
    };
    for (int tpb : {128, 256}) {
        run("A_box128swz", k<0, 128, 1>, mk(128, true), 32 * 128, tpb);
        run("B_box256", k<0, 256, 1>, mk(256, false), 32 * 256, tpb);
        run("C_box512", k<0, 512, 1>, mk(512, false), 32 * 512, tpb);
        run("D_2xbox128", k<0, 128, 2>, mk(128, true), 2 * 32 * 128, tpb);
        run("E_4xbox128", k<0, 128, 4>, mk(128, true), 4 * 32 * 128, tpb);
        run("F_bulk256", k<1, 256, 1>, mk(128, true), 32 * 256, tpb);
        run("F_bulk512", k<1, 512, 1>, mk(128, true), 32 * 512, tpb);
    }
    cudaMemset(out, 0, 16);
    float mset = tms([&] { cudaMemsetAsync(out, 1, NS * N * 4); });
    printf("\"memset\": %.1f}\n", bytes / (mset * 1e-3) / 1e9);
}
