// kernels_threefry.cu — Threefry4x64-20 kernels (NEXT-2; R16): bulk fills
// (u32 / f32 / f64) and the fused Monte Carlo pi kernel, same task layout as
// the Philox kernels (one 32-byte block per chunk).
#include "kernels_common.cuh"

namespace shv {
namespace {

template <int KIND>
__device__ __forceinline__ void store_block_tf(void* o, const Q4& v)
{
    const uint32_t w[8] = {(uint32_t)v.x, (uint32_t)(v.x >> 32), (uint32_t)v.y, (uint32_t)(v.y >> 32),
                           (uint32_t)v.z, (uint32_t)(v.z >> 32), (uint32_t)v.w, (uint32_t)(v.w >> 32)};
    if (KIND == kU32) st_v8(o, w[0], w[1], w[2], w[3], w[4], w[5], w[6], w[7]);
    else if (KIND == kF32)
        st_v8f(o, to_f32(w[0]), to_f32(w[1]), to_f32(w[2]), to_f32(w[3]), to_f32(w[4]), to_f32(w[5]),
               to_f32(w[6]), to_f32(w[7]));
    else st_v4d(o, philox_f64(w[0], w[1]), philox_f64(w[2], w[3]), philox_f64(w[4], w[5]), philox_f64(w[6], w[7]));
}

__device__ __forceinline__ uint32_t q4_word(const Q4& v, uint32_t w)
{
    const uint64_t lane = (w >> 1) == 0 ? v.x : (w >> 1) == 1 ? v.y : (w >> 1) == 2 ? v.z : v.w;
    return (w & 1) ? (uint32_t)(lane >> 32) : (uint32_t)lane;
}

struct ThreefryCursor {
    uint64_t g, k0, k1, blk;
    bool valid;
    Q4 v;
    __device__ __forceinline__ uint32_t word(uint64_t b, uint32_t w)
    {
        if (!valid || b != blk) {
            v = threefry20(b, g, k0, k1);
            blk = b;
            valid = true;
        }
        return q4_word(v, w);
    }
};

#ifndef SHV_TF_UNROLL
#define SHV_TF_UNROLL 4  // blocks per iteration of the fast fill chunk loop (6.07 vs 6.14 ms, lab63)
#endif
constexpr int kTfUnroll = SHV_TF_UNROLL;

// Fast: offset word 0, rows a multiple of one block (32 B). Warp tasks as in
// philox_fill_fast_kernel; one block per 32-byte chunk.
template <int KIND>
__global__ void __launch_bounds__(256) threefry_fill_fast_kernel(const __grid_constant__ ThreefryLaunch P)
{
    constexpr uint64_t E = KIND == kF64 ? 4 : 8;
    const unsigned lane = threadIdx.x & 31;
    const uint64_t cpr = P.n / E;
    const uint64_t span = 32ull * P.nseg;
    const uint64_t tpr = (cpr + span - 1) / span;
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    uint64_t task = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (task >= P.items) return;
    uint64_t i = task / tpr, kb = task - i * tpr;
    const uint64_t qs = nw / tpr, rs = nw - qs * tpr;
    for (; task < P.items; task += nw) {
        const uint64_t g = P.g0 + i;
        const uint64_t c0 = kb * span;
        const uint64_t left = cpr - c0;
        const uint32_t nch = (uint32_t)(left < span ? left : span);
        const uint32_t mine = nch > lane ? (nch - lane + 31) / 32 : 0u;
        uint64_t blk = P.o_blk + c0 + lane;
        char* o = reinterpret_cast<char*>(P.out) + ((i * cpr + c0 + lane) << 5);
#pragma unroll kTfUnroll
        for (uint32_t r = 0; r < mine; ++r) {
            store_block_tf<KIND>(o, threefry20(blk, g, P.k0, P.k1));
            blk = add64(blk, 32u);
            o += 1024;
        }
        kb += rs;
        i += qs;
        if (kb >= tpr) {
            kb -= tpr;
            ++i;
        }
    }
}

template <int KIND>
__global__ void __launch_bounds__(256) threefry_fill_generic_kernel(const __grid_constant__ ThreefryLaunch P)
{
    using T = OutT<KIND>;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t total = P.ns * P.n;
    const uint32_t dpv = KIND == kF64 ? 2 : 1;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < P.items; c += nthr) {
        uint64_t e = c * 8;
        uint64_t i = e / P.n;
        uint64_t j = e - i * P.n;
        ThreefryCursor cur{P.g0 + i, P.k0, P.k1, 0, false, {}};
        for (int u = 0; u < 8 && e < total; ++u, ++e) {
            if (cur.g != P.g0 + i) {
                cur.g = P.g0 + i;
                cur.valid = false;
            }
            const uint64_t d = P.o_word + j * dpv;
            const uint32_t w0 = cur.word(P.o_blk + (d >> 3), (uint32_t)(d & 7));
            T* o = reinterpret_cast<T*>(P.out) + e;
            if (KIND == kU32) *o = (T)w0;
            else if (KIND == kF32) *o = (T)to_f32(w0);
            else {
                const uint64_t d1 = d + 1;
                *o = (T)philox_f64(w0, cur.word(P.o_blk + (d1 >> 3), (uint32_t)(d1 & 7)));
            }
            if (++j == P.n) {
                j = 0;
                ++i;
            }
        }
    }
}

// Fused MC. FAST: offset word 0 and segments a multiple of 4 samples (one
// block = 4 samples).
template <bool FAST>
__global__ void __launch_bounds__(256) threefry_mc_kernel(const __grid_constant__ ThreefryLaunch P)
{
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    uint64_t total = 0;
    for (uint64_t it = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; it < P.items; it += nthr) {
        const uint64_t j = it / P.ns;
        const uint64_t i = it - j * P.ns;
        const uint64_t g = P.g0 + i;
        const uint64_t k0 = j * P.seg_len;
        const uint32_t len = (uint32_t)min(P.seg_len, P.n - k0);
        uint32_t h = 0;
        if (FAST) {
            uint64_t b = P.o_blk + k0 / 4;
            uint32_t k = 0;
            for (; k + 4 <= len; k += 4, b = add64(b, 1u)) {
                const Q4 v = threefry20(b, g, P.k0, P.k1);
                h += hit((uint32_t)v.x, (uint32_t)(v.x >> 32)) + hit((uint32_t)v.y, (uint32_t)(v.y >> 32)) +
                     hit((uint32_t)v.z, (uint32_t)(v.z >> 32)) + hit((uint32_t)v.w, (uint32_t)(v.w >> 32));
            }
            if (k < len) {
                const Q4 v = threefry20(b, g, P.k0, P.k1);
                for (uint32_t u = 0; k < len; ++k, ++u) h += hit(q4_word(v, 2 * u), q4_word(v, 2 * u + 1));
            }
        } else {
            ThreefryCursor cur{g, P.k0, P.k1, 0, false, {}};
            for (uint32_t k = 0; k < len; ++k) {
                const uint64_t d = P.o_word + 2 * (k0 + k);
                const uint32_t w0 = cur.word(P.o_blk + (d >> 3), (uint32_t)(d & 7));
                const uint32_t w1 = cur.word(P.o_blk + ((d + 1) >> 3), (uint32_t)((d + 1) & 7));
                h += hit(w0, w1);
            }
        }
        total += h;
        if (P.counts) atomicAdd(P.counts + i, (unsigned long long)h);
    }
    block_reduce_add(total, P.hits);
}

}  // namespace

cudaError_t launch_threefry_fill(const ThreefryLaunch& p, int kind, bool fast, Grid g, cudaStream_t s)
{
    if (fast) {
        if (kind == kU32) threefry_fill_fast_kernel<kU32><<<g.blocks, g.threads, 0, s>>>(p);
        else if (kind == kF32) threefry_fill_fast_kernel<kF32><<<g.blocks, g.threads, 0, s>>>(p);
        else threefry_fill_fast_kernel<kF64><<<g.blocks, g.threads, 0, s>>>(p);
    } else {
        if (kind == kU32) threefry_fill_generic_kernel<kU32><<<g.blocks, g.threads, 0, s>>>(p);
        else if (kind == kF32) threefry_fill_generic_kernel<kF32><<<g.blocks, g.threads, 0, s>>>(p);
        else threefry_fill_generic_kernel<kF64><<<g.blocks, g.threads, 0, s>>>(p);
    }
    return cudaGetLastError();
}

cudaError_t launch_threefry_mc(const ThreefryLaunch& p, bool fast, Grid g, cudaStream_t s)
{
    if (fast) threefry_mc_kernel<true><<<g.blocks, g.threads, 0, s>>>(p);
    else threefry_mc_kernel<false><<<g.blocks, g.threads, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t threefry_occupancy(int kernel, int kind, bool fast, int threads, int* out)
{
    switch (kernel) {
    case kKThreefryFill:
        if (kind == kU32) return fast ? occ(threefry_fill_fast_kernel<kU32>, threads, 0, out)
                                      : occ(threefry_fill_generic_kernel<kU32>, threads, 0, out);
        if (kind == kF32) return fast ? occ(threefry_fill_fast_kernel<kF32>, threads, 0, out)
                                      : occ(threefry_fill_generic_kernel<kF32>, threads, 0, out);
        return fast ? occ(threefry_fill_fast_kernel<kF64>, threads, 0, out)
                    : occ(threefry_fill_generic_kernel<kF64>, threads, 0, out);
    case kKThreefryMc:
        return fast ? occ(threefry_mc_kernel<true>, threads, 0, out) : occ(threefry_mc_kernel<false>, threads, 0, out);
    }
    return cudaErrorInvalidValue;
}

}  // namespace shv
