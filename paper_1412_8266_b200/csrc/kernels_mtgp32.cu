// kernels_mtgp32.cu — MTGP32-11213 (NEXT-4c; [Saito.Matsumoto2012] via P L74-76
// [§2.2], L133-136 [§2.3]; R18): Parameterization, one Dynamic Creator
// parameter set per stream, and the generator's own block-cooperative design
// — the threads of one CTA compute one state's recursion together.
//
// Recursion over N = 351 words: x_{k+N} = rec(x_k, x_{k+1}, x_{k+pos}),
// output_k = temper(x_{k+N}, x_{k+pos-1}). Elements k .. k+R-1 are independent
// when R <= N - pos (every operand is older than the round), so a CTA of 256
// threads computes R = min(256, N - pos) draws per round from a 1024-word
// shared-memory ring, with ONE barrier per round: a round reads ring slots
// [o, o+R+pos) and writes [o+N, o+N+R); the next round's writes
// [o+R+N, o+2R+N) never alias this round's reads (the distance R+N+t-u lies in
// (N-pos, 2R+N) and never reaches 1024). Draw o+t leaves as word t of the
// round: 1 KB contiguous per round (u32/f32); f64 pairs draws (2j, 2j+1) of
// adjacent lanes with a shuffle, as does the Monte Carlo hit test (R7, R9).
// State in HBM: 352 words per stream (the N current words, oldest first, and
// one pad word), read at the start of a call and written back at its end.
#include "kernels_common.cuh"

namespace shv {
namespace {

constexpr uint32_t kN = kMtgpN;
constexpr uint32_t kRing = 1024;

enum MtgpMode : int { kMtU32 = 0, kMtF32 = 1, kMtF64 = 2, kMtMc = 3, kMtSkip = 4 };

// Initial state (the authors' init_state, R18): hidden seed from tbl[4] and
// tbl[8]; every byte of the array set from it; word 0 = seed, word 1 = the
// hidden seed; then Knuth's 1812433253 recursion over words 1..N-1.
__global__ void __launch_bounds__(256) mtgp_seed_kernel(const __grid_constant__ MtgpLaunch P, uint32_t seed_base)
{
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.ns) return;
    const uint32_t* p = P.params + kMtgpParamWords * i;
    const uint32_t hidden = p[4 + 4] ^ (p[4 + 8] << 16);
    uint32_t f = hidden;
    f += f >> 16;
    f += f >> 8;
    const uint32_t fill = (f & 0xffu) * 0x01010101u;
    uint32_t* x = P.state + kMtgpStateWords * i;
    uint32_t prev = seed_base + (uint32_t)(P.first + i) + 1u;
    x[0] = prev;
    for (uint32_t k = 1; k < kN; ++k) {
        prev = (k == 1 ? hidden : fill) ^ (1812433253u * (prev ^ (prev >> 30)) + k);
        x[k] = prev;
    }
    x[kN] = 0u;
}

template <int MODE>
__global__ void __launch_bounds__(256) mtgp_kernel(const __grid_constant__ MtgpLaunch P)
{
    __shared__ uint32_t ring[kRing];
    __shared__ uint32_t tbl[16], ttbl[16], prm[4];
    const unsigned t = threadIdx.x, lane = t & 31;
    // draws per row of this call
    const uint64_t D = (MODE == kMtF64 || MODE == kMtMc) ? 2 * P.n : P.n;
    uint64_t total = 0;
    for (uint64_t i = blockIdx.x; i < P.ns; i += gridDim.x) {
        const uint32_t* pp = P.params + kMtgpParamWords * i;
        if (t < 4) prm[t] = pp[t];
        else if (t < 20) tbl[t - 4] = pp[t];
        else if (t < 36) ttbl[t - 20] = pp[t];
        uint32_t* st = P.state + kMtgpStateWords * i;
        for (uint32_t k = t; k < kN; k += blockDim.x) ring[k] = st[k];
        __syncthreads();
        const uint32_t pos = prm[0], sh1 = prm[1], sh2 = prm[2], mask = prm[3];
        const uint32_t R = min((uint32_t)blockDim.x, (kN - pos) & ~1u);
        uint32_t o = 0;  // ring index of the oldest word
        uint32_t h = 0;
        for (uint64_t d0 = 0; d0 < D; d0 += R) {
            const uint32_t cnt = (uint32_t)min((uint64_t)R, D - d0);
            uint32_t v = 0;
            if (t < cnt) {
                const uint32_t k = o + t;
                const uint32_t x1 = ring[k & (kRing - 1)], x2 = ring[(k + 1) & (kRing - 1)];
                uint32_t y = ring[(k + pos) & (kRing - 1)];
                uint32_t tt = ring[(k + pos - 1) & (kRing - 1)];
                uint32_t x = (x1 & mask) ^ x2;
                x ^= x << sh1;
                y = x ^ (y >> sh2);
                const uint32_t r = y ^ tbl[y & 0x0f];
                ring[(k + kN) & (kRing - 1)] = r;
                tt ^= tt >> 16;
                tt ^= tt >> 8;
                v = r ^ ttbl[tt & 0x0f];
            }
            if (MODE == kMtU32 || MODE == kMtF32) {
                if (t < cnt) {
                    if (MODE == kMtU32) reinterpret_cast<uint32_t*>(P.out)[i * P.n + d0 + t] = v;
                    else reinterpret_cast<float*>(P.out)[i * P.n + d0 + t] = to_f32(v);
                }
            } else if (MODE == kMtF64 || MODE == kMtMc) {
                const uint32_t hi = __shfl_down_sync(0xffffffffu, v, 1);
                if (!(lane & 1) && t < cnt) {  // d0 and t even: draws (d0+t, d0+t+1) = value (d0+t)/2
                    if (MODE == kMtF64) reinterpret_cast<double*>(P.out)[i * P.n + (d0 + t) / 2] = philox_f64(v, hi);
                    else h += hit(v, hi);
                }
            }
            o += cnt;
            __syncthreads();
        }
        for (uint32_t k = t; k < kN; k += blockDim.x) st[k] = ring[(o + k) & (kRing - 1)];
        if (MODE == kMtMc) {
            total += h;
            if (P.counts) {
                uint32_t w = h;
#pragma unroll
                for (int s = 16; s > 0; s >>= 1) w += __shfl_xor_sync(0xffffffffu, w, s);
                if (lane == 0 && w) atomicAdd(P.counts + i, (unsigned long long)w);
            }
        }
        __syncthreads();  // the ring and tables are reloaded for the next stream
    }
    if (MODE == kMtMc) block_reduce_add(total, P.hits);
}

}  // namespace

cudaError_t launch_mtgp_seed(const MtgpLaunch& p, uint32_t seed_base, cudaStream_t s)
{
    if (p.ns == 0) return cudaSuccess;
    mtgp_seed_kernel<<<(unsigned)((p.ns + 255) / 256), 256, 0, s>>>(p, seed_base);
    return cudaGetLastError();
}

// mode: kind (0 u32, 1 f32, 2 f64), 3 Monte Carlo, 4 skip n draws.
cudaError_t launch_mtgp(const MtgpLaunch& p, int mode, unsigned blocks, cudaStream_t s)
{
    if (p.ns == 0) return cudaSuccess;
    switch (mode) {
    case kMtU32: mtgp_kernel<kMtU32><<<blocks, 256, 0, s>>>(p); break;
    case kMtF32: mtgp_kernel<kMtF32><<<blocks, 256, 0, s>>>(p); break;
    case kMtF64: mtgp_kernel<kMtF64><<<blocks, 256, 0, s>>>(p); break;
    case kMtMc: mtgp_kernel<kMtMc><<<blocks, 256, 0, s>>>(p); break;
    default: mtgp_kernel<kMtSkip><<<blocks, 256, 0, s>>>(p); break;
    }
    return cudaGetLastError();
}

}  // namespace shv
