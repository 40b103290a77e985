// curand_device_pin.cu — TEST-ONLY: NVIDIA cuRAND's own DEVICE implementations
// of MRG32k3a and Philox4x32-10 (curand_kernel.h), compiled for sm_100a, as an
// independent cross-check of libshv's GPU output (tests/test_gpu_curand_xcheck.py).
// Shares no code with libshv or the oracle. Not part of the product.
#include <cstdint>
#include <curand_kernel.h>

// Row i = substream first + i of the MRG32k3a sequence started at state s[6]
// (skipahead_subsequence: 2^76 draws per substream), n u32 draws per row.
__global__ void mrg_rows(uint32_t* out, unsigned long long first, int ns, int n, uint4 s1, uint2 s2)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ns) return;
    curandStateMRG32k3a_t st;
    st.s1[0] = s1.x; st.s1[1] = s1.y; st.s1[2] = s1.z;
    st.s2[0] = s1.w; st.s2[1] = s2.x; st.s2[2] = s2.y;
    skipahead_subsequence(first + (unsigned long long)i, &st);
    // curand() scales z by 2^32/m1; curand_MRG32k3a returns z itself (an integer in [1, m1])
    for (int j = 0; j < n; ++j) out[(size_t)i * n + j] = (uint32_t)curand_MRG32k3a(&st);
}

// Row i = curand_init(seed, first + i, offset) Philox4x32-10 stream, n u32 draws.
__global__ void philox_rows(uint32_t* out, unsigned long long seed, unsigned long long first,
                            unsigned long long offset, int ns, int n)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ns) return;
    curandStatePhilox4_32_10_t st;
    curand_init(seed, first + (unsigned long long)i, offset, &st);
    for (int j = 0; j < n; ++j) out[(size_t)i * n + j] = curand(&st);
}

extern "C" int curand_mrg_rows(uint32_t* d_out, unsigned long long first, int ns, int n, const uint32_t* seed6)
{
    mrg_rows<<<(ns + 127) / 128, 128>>>(d_out, first, ns, n, make_uint4(seed6[0], seed6[1], seed6[2], seed6[3]),
                                        make_uint2(seed6[4], seed6[5]));
    return (int)cudaDeviceSynchronize();
}

extern "C" int curand_philox_rows(uint32_t* d_out, unsigned long long seed, unsigned long long first,
                                  unsigned long long offset, int ns, int n)
{
    philox_rows<<<(ns + 127) / 128, 128>>>(d_out, seed, first, offset, ns, n);
    return (int)cudaDeviceSynchronize();
}
