// pipe_microbench.cu — M1 roofline denominators for the ShoveRand hot path on
// B200 (SURVEY §8d "M1 microbenchmarks"): integer-pipe instruction throughput
// (IMAD.WIDE.U32, IMAD, IADD3, LOP3, a Philox round mix, a MRG-step-like mix),
// DFMA, and write-only HBM bandwidth (256-bit stores, memset).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_microbench tools/pipe_microbench.cu
//   ./pipe_microbench   -> one JSON object on stdout
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int ITERS = 4096;
constexpr int CH = 8;  // independent chains per thread

__global__ void k_imad_wide(uint64_t* out, uint32_t s)
{
    uint64_t a[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c * 77u + s;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c)
            asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(a[c]) : "r"((uint32_t)(a[(c + 1) % CH] >> 32)), "r"(1403580u), "l"(a[c]));
    }
    uint64_t r = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) r ^= a[c];
    if (r == 0x1234567ull) out[0] = r;
}

__global__ void k_imad(uint32_t* out, uint32_t s)
{
    uint32_t a[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c * 77u + s;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c)
            asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(0x9E3779B9u), "r"(s));
    }
    uint32_t r = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) r ^= a[c];
    if (r == 0x1234567u) out[0] = r;
}

__global__ void k_iadd3(uint32_t* out, uint32_t s)
{
    uint32_t a[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c * 77u + s;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            uint32_t t;
            asm volatile("add.u32 %0, %1, %2;" : "=r"(t) : "r"(a[c]), "r"(s));
            asm volatile("add.u32 %0, %1, %2;" : "=r"(a[c]) : "r"(t), "r"(a[(c + 1) % CH]));
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) r ^= a[c];
    if (r == 0x1234567u) out[0] = r;
}

__global__ void k_lop3(uint32_t* out, uint32_t s)
{
    uint32_t a[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c * 77u + s;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c)
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[c]) : "r"(s), "r"(a[(c + 3) % CH]));
    }
    uint32_t r = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) r ^= a[c];
    if (r == 0x1234567u) out[0] = r;
}

// 2 IMAD.WIDE + 2 LOP3 per "round", like Philox.
__global__ void k_philox_mix(uint32_t* out, uint32_t s)
{
    uint32_t c0[CH / 2], c1[CH / 2], c2[CH / 2], c3[CH / 2];
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) { c0[c] = threadIdx.x + c; c1[c] = s; c2[c] = c * 5u; c3[c] = s ^ c; }
    for (int i = 0; i < ITERS / 2; ++i) {
#pragma unroll
        for (int c = 0; c < CH / 2; ++c) {
            uint64_t p0 = (uint64_t)0xD2511F53u * c0[c];
            uint64_t p1 = (uint64_t)0xCD9E8D57u * c2[c];
            uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1[c] ^ s;
            uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3[c] ^ (s + 1);
            c1[c] = (uint32_t)p1; c3[c] = (uint32_t)p0; c0[c] = n0; c2[c] = n2;
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) r ^= c0[c] ^ c1[c] ^ c2[c] ^ c3[c];
    if (r == 0x1234567u) out[0] = r;
}

__global__ void k_dfma(double* out, double s)
{
    double a[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c * 0.5 + s;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) a[c] = fma(a[c], 0.999999, s);
    }
    double r = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) r += a[c];
    if (r == 1.2345) out[0] = r;
}

__global__ void k_fill256(uint32_t* p, uint64_t n32)
{
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n32; c += nthr) {
        uint32_t v = (uint32_t)c;
        asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p + 8 * c), "r"(v) : "memory");
    }
}

__global__ void k_fill128(uint32_t* p, uint64_t n16)
{
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n16; c += nthr) {
        uint32_t v = (uint32_t)c;
        asm volatile("st.global.v4.b32 [%0], {%1,%1,%1,%1};" ::"l"(p + 4 * c), "r"(v) : "memory");
    }
}

// Scattered full-sector writes: thread t writes 32 B into row t of a
// row-major [rows x rowlen] array, stepping along its row (the MRG fill
// pattern with one work item per thread).
__global__ void k_fill_rows(uint32_t* p, uint64_t rows, uint64_t rowlen)
{
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += nthr) {
        uint32_t* q = p + r * rowlen;
        for (uint64_t t = 0; t < rowlen; t += 8)
            asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(q + t), "r"((uint32_t)t) : "memory");
    }
}

// Warp-per-row: lane k of a group of G lanes writes segment k (length
// rowlen/G) of the group's row, 32 B per step: concurrent writes stay inside
// one row (DRAM-page locality) while each lane still walks its own segment.
template <int G>
__global__ void k_fill_rowseg(uint32_t* p, uint64_t rows, uint64_t rowlen)
{
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t L = rowlen / G;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < rows * G; t += nthr) {
        uint32_t* q = p + (t / G) * rowlen + (t % G) * L;
        for (uint64_t u = 0; u < L; u += 8)
            asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(q + u), "r"((uint32_t)u) : "memory");
    }
}

// Groups of W lanes write W*32 contiguous bytes of one row per instruction;
// the 32/W groups of a warp are in different rows (row = group id).
template <int W>
__global__ void k_fill_rowgroup(uint32_t* p, uint64_t rows, uint64_t rowlen)
{
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < rows * W; t += nthr) {
        uint32_t* q = p + (t / W) * rowlen + (lane % W) * 8;
        for (uint64_t u = 0; u < rowlen; u += 8 * W)
            asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(q + u), "r"((uint32_t)u) : "memory");
    }
}

__global__ void k_spin(long long cycles, long long* out)
{
    long long t0 = clock64();
    while (clock64() - t0 < cycles) {}
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = clock64() - t0;
}

template <typename F>
float time_ms(F f, int reps = 5)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

int main()
{
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    long long* dcl;
    CK(cudaMalloc(&dcl, 8));
    // SM clock under a spin load: cycles / elapsed
    const long long spin = 200000000LL;
    float ms_spin = time_ms([&] { k_spin<<<sms, 32>>>(spin, dcl); }, 2);
    const double mhz = spin / (ms_spin * 1e3);

    void* scratch;
    CK(cudaMalloc(&scratch, 64));
    const int threads = 256, blocks = sms * 8;  // 2048 threads/SM
    const double thr = (double)threads * blocks;
    auto rate = [&](float ms, double ops_per_thread) {
        return ops_per_thread * thr / (ms * 1e-3) / (sms * mhz * 1e6);  // ops per SM per clock
    };
    float t_wide = time_ms([&] { k_imad_wide<<<blocks, threads>>>((uint64_t*)scratch, 1); });
    float t_imad = time_ms([&] { k_imad<<<blocks, threads>>>((uint32_t*)scratch, 1); });
    float t_iadd = time_ms([&] { k_iadd3<<<blocks, threads>>>((uint32_t*)scratch, 1); });
    float t_lop3 = time_ms([&] { k_lop3<<<blocks, threads>>>((uint32_t*)scratch, 1); });
    float t_phx = time_ms([&] { k_philox_mix<<<blocks, threads>>>((uint32_t*)scratch, 1); });
    float t_dfma = time_ms([&] { k_dfma<<<blocks, threads>>>((double*)scratch, 1.0); });

    const uint64_t bytes = 16ull << 30;
    uint32_t* buf;
    CK(cudaMalloc(&buf, bytes));
    float t_f256 = time_ms([&] { k_fill256<<<sms * 8, 256>>>(buf, bytes / 32); });
    float t_f128 = time_ms([&] { k_fill128<<<sms * 8, 256>>>(buf, bytes / 16); });
    float t_rows = time_ms([&] { k_fill_rows<<<sms * 8, 256>>>(buf, 1ull << 20, 4096); });
    float t_rs32 = time_ms([&] { k_fill_rowseg<32><<<sms * 8, 256>>>(buf, 1ull << 20, 4096); });
    float t_rs8 = time_ms([&] { k_fill_rowseg<8><<<sms * 8, 256>>>(buf, 1ull << 20, 4096); });
    float t_rs2 = time_ms([&] { k_fill_rowseg<2><<<sms * 8, 256>>>(buf, 1ull << 20, 4096); });
    float t_rg4 = time_ms([&] { k_fill_rowgroup<4><<<sms * 8, 256>>>(buf, 1ull << 20, 4096); });
    float t_rg8 = time_ms([&] { k_fill_rowgroup<8><<<sms * 8, 256>>>(buf, 1ull << 20, 4096); });
    float t_rg2 = time_ms([&] { k_fill_rowgroup<2><<<sms * 8, 256>>>(buf, 1ull << 20, 4096); });
    float t_mset = time_ms([&] { cudaMemsetAsync(buf, 0x5a, bytes); });
    CK(cudaGetLastError());

    printf("{\"sms\": %d, \"sm_clock_mhz_spin\": %.1f,\n", sms, mhz);
    printf(" \"per_sm_per_clk\": {\"imad_wide_u32\": %.2f, \"imad_u32\": %.2f, \"iadd3\": %.2f, "
           "\"lop3\": %.2f, \"philox_round_mix_rounds\": %.2f, \"dfma\": %.2f},\n",
           rate(t_wide, (double)ITERS * CH), rate(t_imad, (double)ITERS * CH),
           rate(t_iadd, (double)ITERS * CH), rate(t_lop3, (double)ITERS * CH),
           rate(t_phx, (double)ITERS / 2 * CH / 2), rate(t_dfma, (double)ITERS * CH));
    printf(" \"write_GBps\": {\"stg256_flat\": %.1f, \"stg128_flat\": %.1f, \"stg256_rows_1thread_per_row\": %.1f, "
           "\"rowseg32\": %.1f, \"rowseg8\": %.1f, \"rowseg2\": %.1f, \"rowgroup2\": %.1f, \"rowgroup4\": %.1f, \"rowgroup8\": %.1f, \"memset\": %.1f}, \"bytes\": %llu}\n",
           bytes / (t_f256 * 1e-3) / 1e9, bytes / (t_f128 * 1e-3) / 1e9, bytes / (t_rows * 1e-3) / 1e9,
           bytes / (t_rs32 * 1e-3) / 1e9, bytes / (t_rs8 * 1e-3) / 1e9, bytes / (t_rs2 * 1e-3) / 1e9,
           bytes / (t_rg2 * 1e-3) / 1e9, bytes / (t_rg4 * 1e-3) / 1e9, bytes / (t_rg8 * 1e-3) / 1e9,
           bytes / (t_mset * 1e-3) / 1e9, (unsigned long long)bytes);
    return 0;
}
