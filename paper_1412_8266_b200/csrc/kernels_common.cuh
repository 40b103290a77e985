// kernels_common.cuh — pieces shared by the per-generator kernel files
// (kernels_mrg.cu, kernels_philox.cu, kernels_threefry.cu, kernels_tinymt32.cu).
//
// Design: persistent grids sized to the SM count; generator
// state in registers (P L257-258: MRG32k3a "only stores 6 integers"; Philox is
// stateless, P L329-331); numbers leave the SM as 256-byte contiguous runs of
// 32-byte vector stores (st.global.v8.b32 -> STG.E.ENL2.256, sm_100+), or
// never leave it (fused Monte Carlo: warp shuffle + shared-memory block
// reduction + one 64-bit atomic per block). No tensor cores: nothing here is
// a contraction. Generator arithmetic lives in include/shv_device.cuh.
#pragma once
#include <atomic>
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "../../include/shv_device.cuh"
#include "shv_internal.h"

// Bytes each lane stages per round in the staged fills (256: eight 1-KB store
// instructions per round, each covering four rows x 256 B; 128: four
// instructions, eight rows x 128 B each).
#ifndef SHV_MRG_RB
#define SHV_MRG_RB 256
#endif

namespace shv {
namespace {

using namespace dev;

template <int KIND>
using OutT = typename std::conditional<KIND == kF64, double,
                                       typename std::conditional<KIND == kF32, float, uint32_t>::type>::type;

template <int KIND>
__device__ __forceinline__ uint4 pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d)
{
    if (KIND == kF32)
        return make_uint4(__float_as_uint(to_f32(a)), __float_as_uint(to_f32(b)),
                          __float_as_uint(to_f32(c)), __float_as_uint(to_f32(d)));
    return make_uint4(a, b, c, d);
}

constexpr unsigned kRB = SHV_MRG_RB;
constexpr unsigned kPieces = kRB / 16;  // 16-byte pieces per lane per round

// Dynamic shared memory of a staged fill with `threads` threads per block
// (RB bytes per lane per round).
template <unsigned RB = kRB>
constexpr size_t staged_smem(int threads) { return (size_t)(threads / 32) * 32 * RB; }

// Staging slot of 16-byte piece q of lane L, conflict-free for the per-lane
// 128-bit writes (8 lanes, same q) and for the write-out reads (8 lanes that
// read pieces 2p resp. 2p+1 of one source lane (RB=256) or two (RB=128)).
template <unsigned RB = kRB>
__device__ __forceinline__ unsigned slot(unsigned L, unsigned q)
{
    if (RB == 256) return 16 * L + 8 * (q & 1) + (((q >> 1) + L) & 7);
    return 8 * L + ((q + L) & 7);
}

// Write one staged round of the warp: lane L's cnt values (RB bytes at most)
// go to row_L + r values; each store instruction covers 1024/RB source lanes
// x RB contiguous bytes.
template <typename T, unsigned RB = kRB>
__device__ __forceinline__ void write_round(const uint4* wb, unsigned lane, uint32_t r, uint32_t cnt, uint64_t row)
{
    __syncwarp();
#pragma unroll
    for (unsigned k = 0; k < RB / 32; ++k) {
        const unsigned src = (1024 / RB) * k + lane / (RB / 32), p = lane % (RB / 32);
        const uint32_t scnt = __shfl_sync(0xffffffffu, cnt, src);
        const uint64_t srow = __shfl_sync(0xffffffffu, row, src);
        if (32 * p < scnt * sizeof(T))
            st_v8(reinterpret_cast<char*>(srow) + (uint64_t)r * sizeof(T) + 32 * p, wb[slot<RB>(src, 2 * p)],
                  wb[slot<RB>(src, 2 * p + 1)]);
    }
    __syncwarp();
}

template <typename K>
cudaError_t occ(K kernel, int threads, size_t smem, int* out)
{
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, kernel, threads, smem);
}

// Opt a kernel into `bytes` (> 48 KB) of dynamic shared memory once per device
// (the attribute is per function and context); `done` is the caller's
// per-kernel bit set of devices already configured.
template <typename K>
cudaError_t ensure_dyn_smem(K kernel, size_t bytes, std::atomic<uint64_t>& done)
{
    if (bytes <= 48 * 1024) return cudaSuccess;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_release);
    return e;
}

}  // namespace
}  // namespace shv
