// tma_layout_lab.cu — write bandwidth of the MRG fill's store layouts over the
// C5 output (2^20 rows x 4096 u32 = 16 GiB), null generator (bandwidth only).
// The output is viewed as [NS*N/S][S] (segments of S values, contiguous): a
// warp tile is 32 consecutive segments, lane l owns segment l of the tile and
// writes it in rounds of 128 B. S = 4096: the r01/r02 layout (a warp = 32
// stream rows, pieces 16 KB apart); S = 128: a warp = one stream row (pieces
// 512 B apart, the row written in 4 rounds).
//   T (TMA): one 32 x 128-B box per round (128-B swizzle), lane 0 issues it.
//   D (direct): each lane st.global.v8 (32 B) x 4 per round into its segment.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_layout_lab tools/lab/tma_layout_lab.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

constexpr uint64_t NS = 1ull << 20, N = 4096;

template <bool TMA>
__global__ void __launch_bounds__(256) k(const __grid_constant__ CUtensorMap tm, uint32_t* out, uint32_t S)
{
    extern __shared__ uint8_t sm[];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t base = ((uint32_t)__cvta_generic_to_shared(sm) + 1023u) & ~1023u;
    const uint32_t box = base + warp * 4096u;
    const uint64_t G = NS * N / S / 32;
    const uint64_t wstride = (uint64_t)gridDim.x * (blockDim.x >> 5);
    uint32_t v = lane * 77u;
    for (uint64_t g = (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp; g < G; g += wstride) {
        uint32_t* seg = out + (32 * g + lane) * S;
        for (uint32_t c = 0; c < S; c += 32) {
            if (TMA) {
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                __syncwarp();
                const uint32_t rowsw = box + lane * 128u + ((lane & 7u) << 4);
#pragma unroll
                for (unsigned q = 0; q < 8; ++q) {
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowsw ^ (q << 4)), "r"(v), "r"(v + 1),
                                 "r"(v + 2), "r"(v + 3) : "memory");
                    v += 4;
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tm),
                                 "r"(box), "r"((int)c), "r"((int)(32 * g)) : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
            } else {
#pragma unroll
                for (unsigned q = 0; q < 4; ++q) {
                    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(seg + c + 8 * q), "r"(v),
                                 "r"(v + 1), "r"(v + 2), "r"(v + 3), "r"(v + 4), "r"(v + 5), "r"(v + 6), "r"(v + 7)
                                 : "memory");
                    v += 8;
                }
            }
        }
    }
    if (TMA && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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
    void* p = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    uint32_t* out; cudaMalloc(&out, NS * N * 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double bytes = (double)NS * N * 4;
    printf("{");
    for (uint32_t S : {4096u, 2048u, 1024u, 512u, 256u, 128u}) {
        CUtensorMap m; cuuint64_t d[2] = {S, NS * N / S}; cuuint64_t st[1] = {(cuuint64_t)S * 4};
        cuuint32_t bx[2] = {32, 32}; cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, out, d, st, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r) printf("encode failed %d\n", (int)r);
        for (int bps : {2, 4, 6}) {
            const size_t smem = 8 * 4096 + 1024;
            cudaFuncSetAttribute(k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            float mt = tms([&] { k<true><<<sms * bps, 256, smem>>>(m, out, S); });
            float md = tms([&] { k<false><<<sms * bps, 256, 0>>>(m, out, S); });
            printf("\"S%u_b%d\": {\"tma_GBps\": %.1f, \"direct_GBps\": %.1f, \"err\": %d}, ", S, bps,
                   bytes / (mt * 1e-3) / 1e9, bytes / (md * 1e-3) / 1e9, (int)cudaGetLastError());
        }
    }
    float mset = tms([&] { cudaMemsetAsync(out, 1, NS * N * 4); });
    printf("\"memset\": %.1f}\n", bytes / (mset * 1e-3) / 1e9);
}
