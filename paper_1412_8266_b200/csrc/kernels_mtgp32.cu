// kernels_mtgp32.cu — MTGP32-11213 (NEXT-4c; [Saito.Matsumoto2012] via P L74-76
// [§2.2], L133-136 [§2.3]; R18): Parameterization, one Dynamic Creator
// parameter set per stream, and the generator's own block-cooperative design
// — the threads of one CTA compute one state's recursion together.
//
// Recursion over N = 351 words: x_{k+N} = rec(x_k, x_{k+1}, x_{k+pos}),
// output_k = temper(x_{k+N}, x_{k+pos-1}). Elements k .. k+R-1 are independent
// when R <= N - pos (every operand is older than the round), so the threads of
// a CTA compute R = (N - pos) & ~1 draws per round (128 threads, three
// elements each) from a 1024-word shared-memory ring, with ONE barrier per
// round: a round reads ring slots [o, o+R+pos) and writes [o+N, o+N+R), which
// stay apart (R+pos <= N) and do not wrap onto the live words (N+R <= 699 <
// 1024); the barrier orders one round's writes before the next round's reads.
// Draw o+e leaves as word e of the round: R contiguous words per round
// (u32/f32); f64 pairs draws (2j, 2j+1) of
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

// One round of up to R = (N - pos) & ~1 (<= 348) draws: thread t computes
// elements t, t + 128, t + 256 (kEpt independent chains for latency hiding;
// 4 warps, so the per-round barrier is cheap). Element e is draw d0 + e.
#ifndef SHV_MT_THREADS
#define SHV_MT_THREADS 128
#endif
#ifndef SHV_MT_EPT
#define SHV_MT_EPT 3
#endif
constexpr unsigned kMtThreads = SHV_MT_THREADS, kEpt = SHV_MT_EPT;
static_assert(kMtThreads % 32 == 0, "whole warps");
static_assert(kMtThreads * kEpt >= 348, "a round covers N - pos (<= 348) elements");

template <int MODE>
__global__ void __launch_bounds__(kMtThreads) mtgp_kernel(const __grid_constant__ MtgpLaunch P)
{
    // Mirrored ring: word j lives at j and j + 1024 (j < 1024) and the base o
    // stays below 1024, so every read index o + e + {0, 1, pos - 1, pos}
    // (< 1024 + 348 + 349) needs no wrap mask; each new word is stored twice.
    __shared__ uint32_t ring[2 * kRing];
    __shared__ uint32_t tbl[16], ttbl[16], prm[4];
    const unsigned t = threadIdx.x, lane = t & 31;
    // draws per row of this call
    const uint64_t D = (MODE == kMtF64 || MODE == kMtMc) ? 2 * P.n : P.n;
    uint64_t total = 0;
    for (uint64_t i = blockIdx.x; i < P.ns; i += gridDim.x) {
        const uint32_t* pp = P.params + kMtgpParamWords * i;
        for (uint32_t k = t; k < kMtgpParamWords; k += kMtThreads) {
            if (k < 4) prm[k] = pp[k];
            else if (k < 20) tbl[k - 4] = pp[k];
            else ttbl[k - 20] = pp[k];
        }
        uint32_t* st = P.state + kMtgpStateWords * i;
        for (uint32_t k = t; k < kN; k += kMtThreads) {
            const uint32_t w = st[k];
            ring[k] = w;
            ring[k + kRing] = w;
        }
        __syncthreads();
        const uint32_t pos = prm[0], sh1 = prm[1], sh2 = prm[2], mask = prm[3];
        const uint32_t R = min(kMtThreads * kEpt, (kN - pos) & ~1u);
        uint32_t o = 0;  // ring index of the oldest word, < 1024
        uint32_t h = 0;
        uint32_t* const orow = reinterpret_cast<uint32_t*>(P.out) + (MODE == kMtF64 ? 2 : 1) * i * P.n;
        for (uint64_t d0 = 0; d0 < D; d0 += R) {
            const uint32_t cnt = (uint32_t)min((uint64_t)R, D - d0);
            // all loads of the round first: the ring stores below cannot then
            // order (alias) the next element's loads behind them. Elements past
            // the round (e >= cnt) load the last live element's operands
            // instead: slots past o + R + pos may be this round's stores.
            uint32_t x1[kEpt], x2[kEpt], y[kEpt], tt[kEpt], v[kEpt];
#pragma unroll
            for (unsigned q = 0; q < kEpt; ++q) {
                const uint32_t* rk = ring + o + min(t + q * kMtThreads, cnt - 1);
                x1[q] = rk[0];
                x2[q] = rk[1];
                tt[q] = rk[pos - 1];
                y[q] = rk[pos];
            }
            uint32_t r[kEpt];
#pragma unroll
            for (unsigned q = 0; q < kEpt; ++q) {
                uint32_t x = (x1[q] & mask) ^ x2[q];
                x ^= x << sh1;
                const uint32_t yy = x ^ (y[q] >> sh2);
                r[q] = yy ^ tbl[yy & 0x0f];
                uint32_t u = tt[q];
                u ^= u >> 16;
                u ^= u >> 8;
                v[q] = r[q] ^ ttbl[u & 0x0f];
            }
#pragma unroll
            for (unsigned q = 0; q < kEpt; ++q)
                if (t + q * kMtThreads < cnt) {
                    const uint32_t j = (o + t + q * kMtThreads + kN) & (kRing - 1);
                    ring[j] = r[q];
                    ring[j + kRing] = r[q];
                }
            uint32_t* const ob = orow + (MODE == kMtF64 ? 2 * (d0 / 2) : d0);
#pragma unroll
            for (unsigned q = 0; q < kEpt; ++q) {
                const uint32_t e = t + q * kMtThreads;
                if (MODE == kMtU32 || MODE == kMtF32) {
                    if (e < cnt) {
                        if (MODE == kMtU32) ob[e] = v[q];
                        else reinterpret_cast<float*>(ob)[e] = to_f32(v[q]);
                    }
                } else if (MODE == kMtF64 || MODE == kMtMc) {
                    // d0, R and kMtThreads even: draws (d0+e, d0+e+1) of lanes e, e+1 = value (d0+e)/2
                    const uint32_t hi = __shfl_down_sync(0xffffffffu, v[q], 1);
                    if (!(lane & 1) && e < cnt) {
                        if (MODE == kMtF64)
                            reinterpret_cast<double*>(ob)[e / 2] = philox_f64(v[q], hi);
                        else
                            h += hit(v[q], hi);
                    }
                }
            }
            o = (o + cnt) & (kRing - 1);
            __syncthreads();
        }
        for (uint32_t k = t; k < kN; k += kMtThreads) st[k] = ring[o + k];
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
    case kMtU32: mtgp_kernel<kMtU32><<<blocks, kMtThreads, 0, s>>>(p); break;
    case kMtF32: mtgp_kernel<kMtF32><<<blocks, kMtThreads, 0, s>>>(p); break;
    case kMtF64: mtgp_kernel<kMtF64><<<blocks, kMtThreads, 0, s>>>(p); break;
    case kMtMc: mtgp_kernel<kMtMc><<<blocks, kMtThreads, 0, s>>>(p); break;
    default: mtgp_kernel<kMtSkip><<<blocks, kMtThreads, 0, s>>>(p); break;
    }
    return cudaGetLastError();
}

}  // namespace shv
