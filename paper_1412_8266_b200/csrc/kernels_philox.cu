// kernels_philox.cu — Philox4x32-10 kernels (arXiv 1412.8266 P L326-334
// [§4.1]; counter-split stream layout R6, keyed Parameterization R12): bulk
// fills (u32 / f32 / f64) and the fused Monte Carlo pi kernel. Stateless:
// every value is a pure function of (key, counter), so launches need no state.
#include "kernels_common.cuh"

namespace shv {
namespace {

// Key and counter-stream word of launch stream i. Counter-split layout (R6):
// key = seed, stream g -> ctr[2..3]. KEYED (Parameterization, P L331-334):
// key = (stream id, tag), ctr[2..3] = 0.
template <bool KEYED>
__device__ __forceinline__ void stream_key(const PhiloxLaunch& P, uint64_t i, uint32_t& k0, uint32_t& k1,
                                           uint64_t& g)
{
    if (KEYED) {
        k0 = (uint32_t)(P.g0 + i);
        k1 = P.k1;
        g = 0;
    } else {
        k0 = P.k0;
        k1 = P.k1;
        g = P.g0 + i;
    }
}

// 8 draws (two blocks) -> one 32-byte chunk of u32 / f32 / f64 values.
template <int KIND>
__device__ __forceinline__ void store_chunk(void* o, const W4& a, const W4& d)
{
    if (KIND == kU32) {
        st_v8(o, a.x, a.y, a.z, a.w, d.x, d.y, d.z, d.w);
    } else if (KIND == kF32) {
        st_v8f(o, to_f32(a.x), to_f32(a.y), to_f32(a.z), to_f32(a.w), to_f32(d.x), to_f32(d.y), to_f32(d.z),
               to_f32(d.w));
    } else {
        st_v4d(o, philox_f64(a.x, a.y), philox_f64(a.z, a.w), philox_f64(d.x, d.y), philox_f64(d.z, d.w));
    }
}

// Fast Philox fill: offset lane 0, rows a multiple of E elements, 32-byte
// aligned output. A warp task is (row i, run of 32*R chunks of 32 bytes); lane
// l handles chunks l, l+32, ... so each store instruction writes 1 KB
// contiguous. The round-1 product of the stream word is hoisted per task.
template <int KIND, bool KEYED>
__global__ void __launch_bounds__(256) philox_fill_fast_kernel(const __grid_constant__ PhiloxLaunch P)
{
    constexpr uint64_t E = KIND == kF64 ? 4 : 8;  // elements per 32-byte chunk
    const unsigned lane = threadIdx.x & 31;
    const uint64_t cpr = P.n / E;                  // chunks per row
    const uint64_t span = 32ull * P.nseg;          // chunks per task (nseg = R)
    const uint64_t tpr = (cpr + span - 1) / span;  // tasks per row
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    uint64_t task = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (task >= P.items) return;
    if (P.rpt > 1) {
        // Short rows: a task is rpt whole rows (one run each). The counter
        // block of a lane's chunk depends only on its column, so the round-1
        // product M0*blk_lo is row-invariant; per row only the stream word's
        // products (p1, and q through round 1's output) are recomputed.
        const uint32_t mine = cpr > lane ? (uint32_t)((cpr - lane + 31) / 32) : 0u;
        const uint64_t blk = P.o_blk + 2 * lane;
        const bool nowrap = (uint32_t)blk <= 0xFFFFFFFFu - 64u * mine - 1u;
        const uint64_t pa0 = (uint64_t)kPM0 * (uint32_t)blk;
        for (; task < P.items; task += nw) {
            const uint64_t i0 = task * P.rpt;
            const uint64_t i1 = min(i0 + P.rpt, P.ns);
            char* orow = reinterpret_cast<char*>(P.out) + ((i0 * cpr + lane) << 5);
            for (uint64_t i = i0; i < i1; ++i, orow += cpr << 5) {
                uint32_t k0, k1;
                uint64_t g;
                stream_key<KEYED>(P, i, k0, k1, g);
                const uint64_t p1 = (uint64_t)kPM1 * (uint32_t)g;
                char* o = orow;
                if (nowrap) {
                    const uint32_t c0r1 = (uint32_t)(p1 >> 32) ^ (uint32_t)(blk >> 32) ^ k0;
                    const uint64_t q = (uint64_t)kPM0 * c0r1;
                    uint64_t pa = pa0;
                    for (uint32_t r = 0; r < mine; ++r) {
                        const uint64_t pb = add64w(pa, kPM0);
                        const W4 a = philox10_from_r2<true>(pa, q, (uint32_t)p1, (uint32_t)(g >> 32), k0, k1);
                        const W4 d = philox10_from_r2<true>(pb, q, (uint32_t)p1, (uint32_t)(g >> 32), k0, k1);
                        store_chunk<KIND>(o, a, d);
                        pa = add64w(pa, 64ull * kPM0);
                        o += 1024;
                    }
                } else {
                    uint64_t b = blk;
                    for (uint32_t r = 0; r < mine; ++r) {
                        const uint64_t b1 = add64(b, 1u);
                        const W4 a = philox_blk(b, g, k0, k1);
                        const W4 d = philox_blk(b1, g, k0, k1);
                        store_chunk<KIND>(o, a, d);
                        b = add64(b, 64u);
                        o += 1024;
                    }
                }
            }
        }
        return;
    }
    uint64_t i = task / tpr, kb = task - i * tpr;
    const uint64_t qs = nw / tpr, rs = nw - qs * tpr;
    for (; task < P.items; task += nw) {
        uint32_t k0, k1;
        uint64_t g;
        stream_key<KEYED>(P, i, k0, k1, g);
        const uint64_t p1 = (uint64_t)kPM1 * (uint32_t)g;  // round-1 product, task-invariant
        const uint64_t c0 = kb * span;
        const uint64_t left = cpr - c0;
        const uint32_t nch = (uint32_t)(left < span ? left : span);
        const uint32_t mine = nch > lane ? (nch - lane + 31) / 32 : 0u;
        uint64_t blk = P.o_blk + 2 * (c0 + lane);
        char* o = reinterpret_cast<char*>(P.out) + ((i * cpr + c0 + lane) << 5);
        // Fast sub-path: the low counter word does not wrap inside this task,
        // so blk_hi is fixed, round 2's M0 product is hoisted, and the round-1
        // products M0*blk_lo advance by additions (M0*(b+1) = M0*b + M0).
        if ((uint32_t)blk <= 0xFFFFFFFFu - 64u * mine - 1u) {
            const uint32_t c0r1 = (uint32_t)(p1 >> 32) ^ (uint32_t)(blk >> 32) ^ k0;
            const uint64_t q = (uint64_t)kPM0 * c0r1;
            uint64_t pa = (uint64_t)kPM0 * (uint32_t)blk;
            for (uint32_t r = 0; r < mine; ++r) {
                const uint64_t pb = add64w(pa, kPM0);
                const W4 a = philox10_from_r2<true>(pa, q, (uint32_t)p1, (uint32_t)(g >> 32), k0, k1);
                const W4 d = philox10_from_r2<true>(pb, q, (uint32_t)p1, (uint32_t)(g >> 32), k0, k1);
                store_chunk<KIND>(o, a, d);
                pa = add64w(pa, 64ull * kPM0);
                o += 1024;
            }
        } else {
            for (uint32_t r = 0; r < mine; ++r) {
                const uint64_t b1 = add64(blk, 1u);
                const uint64_t pa = (uint64_t)kPM0 * (uint32_t)blk;
                const uint64_t pb = (uint64_t)kPM0 * (uint32_t)b1;
                const W4 a = philox10_from_r1((uint32_t)(pa >> 32), (uint32_t)pa, (uint32_t)(p1 >> 32), (uint32_t)p1,
                                              (uint32_t)(blk >> 32), (uint32_t)(g >> 32), k0, k1);
                const W4 d = philox10_from_r1((uint32_t)(pb >> 32), (uint32_t)pb, (uint32_t)(p1 >> 32), (uint32_t)p1,
                                              (uint32_t)(b1 >> 32), (uint32_t)(g >> 32), k0, k1);
                store_chunk<KIND>(o, a, d);
                blk = add64(blk, 64u);
                o += 1024;
            }
        }
        kb += rs;
        i += qs;
        if (kb >= tpr) {
            kb -= tpr;
            ++i;
        }
    }
}

// Generic Philox fill: any offset, any row length, element-aligned output.
// Work item = up to 8 consecutive elements of the flat stream-major array.
template <int KIND, bool KEYED>
__global__ void __launch_bounds__(256) philox_fill_generic_kernel(const __grid_constant__ PhiloxLaunch P)
{
    using T = OutT<KIND>;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t total = P.ns * P.n;
    const uint32_t dpv = KIND == kF64 ? 2 : 1;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < P.items; c += nthr) {
        uint64_t e = c * 8;
        uint64_t i = e / P.n;
        uint64_t j = e - i * P.n;
        PhiloxCursor cur{0, 0, 0, 0, false, {}};
        stream_key<KEYED>(P, i, cur.k0, cur.k1, cur.g);
        uint64_t ci = i;
        for (int u = 0; u < 8 && e < total; ++u, ++e) {
            if (ci != i) {
                ci = i;
                stream_key<KEYED>(P, i, cur.k0, cur.k1, cur.g);
                cur.valid = false;
            }
            const uint64_t d = P.o_lane + j * dpv;  // draw index relative to 4*o_blk
            const uint32_t w0 = cur.word(P.o_blk + (d >> 2), (uint32_t)(d & 3));
            T* o = reinterpret_cast<T*>(P.out) + e;
            if (KIND == kU32) {
                *o = (T)w0;
            } else if (KIND == kF32) {
                *o = (T)to_f32(w0);
            } else {
                const uint64_t d1 = d + 1;
                const uint32_t w1 = cur.word(P.o_blk + (d1 >> 2), (uint32_t)(d1 & 3));
                *o = (T)philox_f64(w0, w1);
            }
            if (++j == P.n) {
                j = 0;
                ++i;
            }
        }
    }
}

#ifndef SHV_PHILOX_MC_UNROLL
#define SHV_PHILOX_MC_UNROLL 2  // two blocks in flight per thread: 412 -> 398 ms for C4 (tools/lab)
#endif
constexpr int kPhiloxMcUnroll = SHV_PHILOX_MC_UNROLL;

#ifndef SHV_PHILOX_MC_HIT
#define SHV_PHILOX_MC_HIT 2  // 2 = hit_fp64_cvt (XU conversions: 393.8 vs 396.7 ms, lab38), 1 = hit_fp64
#endif
#define PHILOX_MC_HIT(a, b) (SHV_PHILOX_MC_HIT == 2 ? hit_fp64_cvt(a, b) : hit_fp64(a, b))

// Fused Philox Monte Carlo. FAST: offset lane 0 and even segment length, so
// sample pairs never straddle a counter block (two samples per block).
template <bool FAST, bool KEYED>
__global__ void __launch_bounds__(256) philox_mc_kernel(const __grid_constant__ PhiloxLaunch P)
{
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    uint64_t total = 0;
    for (uint64_t it = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; it < P.items; it += nthr) {
        const uint64_t j = it / P.ns;
        const uint64_t i = it - j * P.ns;
        uint32_t key0, key1;
        uint64_t g;
        stream_key<KEYED>(P, i, key0, key1, g);
        const uint64_t k0 = j * P.seg_len;
        const uint32_t len = (uint32_t)min(P.seg_len, P.n - k0);
        uint32_t h = 0;
        if (FAST) {
            const uint64_t p1 = (uint64_t)kPM1 * (uint32_t)g;
            uint64_t b = P.o_blk + k0 / 2;
            const uint32_t nb = len / 2;
            if ((uint32_t)b <= 0xFFFFFFFFu - nb - 1u) {
                // no wrap of the low counter word: hoisted round-2 product,
                // round-1 products by addition (see philox_fill_fast_kernel)
                const uint32_t c0r1 = (uint32_t)(p1 >> 32) ^ (uint32_t)(b >> 32) ^ key0;
                const uint64_t q = (uint64_t)kPM0 * c0r1;
                uint64_t pa = (uint64_t)kPM0 * (uint32_t)b;
#pragma unroll kPhiloxMcUnroll
                for (uint32_t r = 0; r < nb; ++r) {
                    const W4 a = philox10_from_r2(pa, q, (uint32_t)p1, (uint32_t)(g >> 32), key0, key1);
                    h += PHILOX_MC_HIT(a.x, a.y) + PHILOX_MC_HIT(a.z, a.w);
                    pa = add64w(pa, kPM0);
                }
                b = add64(b, nb);
            } else {
                for (uint32_t r = 0; r < nb; ++r) {
                    const uint64_t pa = (uint64_t)kPM0 * (uint32_t)b;
                    const W4 a = philox10_from_r1((uint32_t)(pa >> 32), (uint32_t)pa, (uint32_t)(p1 >> 32),
                                                  (uint32_t)p1, (uint32_t)(b >> 32), (uint32_t)(g >> 32), key0, key1);
                    h += PHILOX_MC_HIT(a.x, a.y) + PHILOX_MC_HIT(a.z, a.w);
                    b = add64(b, 1u);
                }
            }
            if (len & 1) {
                const W4 a = philox_blk(b, g, key0, key1);
                h += hit(a.x, a.y);
            }
        } else {
            PhiloxCursor cur{g, key0, key1, 0, false, {}};
            for (uint32_t k = 0; k < len; ++k) {
                const uint64_t d = P.o_lane + 2 * (k0 + k);
                const uint32_t w0 = cur.word(P.o_blk + (d >> 2), (uint32_t)(d & 3));
                const uint32_t w1 = cur.word(P.o_blk + ((d + 1) >> 2), (uint32_t)((d + 1) & 3));
                h += hit(w0, w1);
            }
        }
        total += h;
        if (P.counts) atomicAdd(P.counts + i, (unsigned long long)h);
    }
    block_reduce_add(total, P.hits);
}

}  // namespace

template <bool KEYED>
cudaError_t launch_philox_fill_t(const PhiloxLaunch& p, int kind, bool fast, Grid g, cudaStream_t s)
{
    if (fast) {
        if (kind == kU32) philox_fill_fast_kernel<kU32, KEYED><<<g.blocks, g.threads, 0, s>>>(p);
        else if (kind == kF32) philox_fill_fast_kernel<kF32, KEYED><<<g.blocks, g.threads, 0, s>>>(p);
        else philox_fill_fast_kernel<kF64, KEYED><<<g.blocks, g.threads, 0, s>>>(p);
    } else {
        if (kind == kU32) philox_fill_generic_kernel<kU32, KEYED><<<g.blocks, g.threads, 0, s>>>(p);
        else if (kind == kF32) philox_fill_generic_kernel<kF32, KEYED><<<g.blocks, g.threads, 0, s>>>(p);
        else philox_fill_generic_kernel<kF64, KEYED><<<g.blocks, g.threads, 0, s>>>(p);
    }
    return cudaGetLastError();
}

cudaError_t launch_philox_fill(const PhiloxLaunch& p, int kind, bool fast, Grid g, cudaStream_t s)
{
    return p.keyed ? launch_philox_fill_t<true>(p, kind, fast, g, s) : launch_philox_fill_t<false>(p, kind, fast, g, s);
}

cudaError_t launch_philox_mc(const PhiloxLaunch& p, bool fast, Grid g, cudaStream_t s)
{
    if (p.keyed) {
        if (fast) philox_mc_kernel<true, true><<<g.blocks, g.threads, 0, s>>>(p);
        else philox_mc_kernel<false, true><<<g.blocks, g.threads, 0, s>>>(p);
    } else {
        if (fast) philox_mc_kernel<true, false><<<g.blocks, g.threads, 0, s>>>(p);
        else philox_mc_kernel<false, false><<<g.blocks, g.threads, 0, s>>>(p);
    }
    return cudaGetLastError();
}

cudaError_t philox_occupancy(int kernel, int kind, bool fast, int threads, int* out)
{
    switch (kernel) {
    case kKPhiloxFill:
        if (kind == kU32) return fast ? occ(philox_fill_fast_kernel<kU32, false>, threads, 0, out)
                                      : occ(philox_fill_generic_kernel<kU32, false>, threads, 0, out);
        if (kind == kF32) return fast ? occ(philox_fill_fast_kernel<kF32, false>, threads, 0, out)
                                      : occ(philox_fill_generic_kernel<kF32, false>, threads, 0, out);
        return fast ? occ(philox_fill_fast_kernel<kF64, false>, threads, 0, out)
                    : occ(philox_fill_generic_kernel<kF64, false>, threads, 0, out);
    case kKPhiloxFillKeyed:
        if (kind == kU32) return fast ? occ(philox_fill_fast_kernel<kU32, true>, threads, 0, out)
                                      : occ(philox_fill_generic_kernel<kU32, true>, threads, 0, out);
        if (kind == kF32) return fast ? occ(philox_fill_fast_kernel<kF32, true>, threads, 0, out)
                                      : occ(philox_fill_generic_kernel<kF32, true>, threads, 0, out);
        return fast ? occ(philox_fill_fast_kernel<kF64, true>, threads, 0, out)
                    : occ(philox_fill_generic_kernel<kF64, true>, threads, 0, out);
    case kKPhiloxMc:
        return fast ? occ(philox_mc_kernel<true, false>, threads, 0, out)
                    : occ(philox_mc_kernel<false, false>, threads, 0, out);
    case kKPhiloxMcKeyed:
        return fast ? occ(philox_mc_kernel<true, true>, threads, 0, out)
                    : occ(philox_mc_kernel<false, true>, threads, 0, out);
    }
    return cudaErrorInvalidValue;
}

}  // namespace shv
