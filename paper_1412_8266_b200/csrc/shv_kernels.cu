// shv_kernels.cu — sm_100a kernels of the ShoveRand hot path (arXiv 1412.8266).
//
// Design: one persistent grid sized to the SM count; generator
// state lives in registers (P L257-258: MRG32k3a "only stores 6 integers";
// Philox is stateless, P L329-331); numbers leave the SM as full 32-byte
// sectors (st.global.v8.b32 -> STG.E.ENL2.256, sm_100+), or never leave it
// (fused Monte Carlo: warp shuffle + shared-memory block reduction + one
// 64-bit atomic per block). No tensor cores: nothing here is a contraction.
//
// Arithmetic (exact, integer only; bounds in DESIGN.md §4.2):
//   MRG32k3a step  p1 = a12*x1 + a13n*(m1-x0) folded with 2^32 = 209 (mod m1)
//                  p2 = a21*y2 + a23n*(m2-y0) folded twice with 2^32 = 22853 (mod m2)
//                  z  = p1 - p2 (+ m1 if p1 <= p2), z in [1, m1]         (R1, R2)
//   Philox4x32-10  10 rounds of two 32x32->64 multiplies and two 3-way XORs;
//                  the key schedule is warp-uniform (uniform datapath).    (R5, R6)
#include <cstdint>
#include <cuda_runtime.h>

#include "shv_internal.h"

namespace shv {
namespace {

// [LEcuyer1999] MRG32k3a parameters (PAPER.md L255 cites them; not restated there).
constexpr uint32_t kM1 = 4294967087u;  // 2^32 - 209
constexpr uint32_t kM2 = 4294944443u;  // 2^32 - 22853
constexpr uint32_t kC1 = 209u;
constexpr uint32_t kC2 = 22853u;
constexpr uint32_t kA12 = 1403580u;
constexpr uint32_t kA13n = 810728u;
constexpr uint32_t kA21 = 527612u;
constexpr uint32_t kA23n = 1370589u;
// [Salmon.etal.2011] Philox4x32 multipliers and Weyl key increments.
constexpr uint32_t kPM0 = 0xD2511F53u;
constexpr uint32_t kPM1 = 0xCD9E8D57u;
constexpr uint32_t kPW0 = 0x9E3779B9u;
constexpr uint32_t kPW1 = 0xBB67AE85u;

// Jump tables: [0][b] = A^(2^(76+b)) (substreams, b < 51),
//              [1][b] = A^(2^(127+b)) (streams, b < 64).
__device__ MatPair g_jump_tab[2][64];

// ------------------------------------------------------------------ MRG32k3a

struct Mrg {
    uint32_t x0, x1, x2;  // component 1, oldest -> newest (R1)
    uint32_t y0, y1, y2;  // component 2
};

__device__ __forceinline__ uint32_t mrg_next(Mrg& s)
{
    // Component 1. P < 2^53.06, hi < 2^21.1, hi*209 < 2^29: one 32-bit fold
    // whose carry-out or a result >= m1 both mean "subtract m1" = "+209".
    const uint64_t p = (uint64_t)kA12 * s.x1 + (uint64_t)kA13n * (kM1 - s.x0);
    const uint32_t lo = (uint32_t)p;
    const uint32_t r = lo + (uint32_t)(p >> 32) * kC1;
    const uint32_t p1 = r + ((r < lo) | (r >= kM1) ? kC1 : 0u);
    s.x0 = s.x1;
    s.x1 = s.x2;
    s.x2 = p1;
    // Component 2. Q < 2^52.9, hi*22853 < 2^35.4: fold to T < 2^35.6, then a
    // second 32-bit fold as above with c = 22853.
    const uint64_t q = (uint64_t)kA21 * s.y2 + (uint64_t)kA23n * (kM2 - s.y0);
    const uint64_t t = (uint64_t)(uint32_t)(q >> 32) * kC2 + (uint32_t)q;
    const uint32_t tlo = (uint32_t)t;
    const uint32_t r2 = tlo + (uint32_t)(t >> 32) * kC2;
    const uint32_t p2 = r2 + ((r2 < tlo) | (r2 >= kM2) ? kC2 : 0u);
    s.y0 = s.y1;
    s.y1 = s.y2;
    s.y2 = p2;
    // Combination: (p1 - p2) mod m1 with 0 -> m1 (R2); exact in wrap-around.
    const uint32_t z = p1 - p2;
    return p1 > p2 ? z : z + kM1;
}

// x mod (2^32 - c) for any 64-bit x (c < 2^15): two folds + one subtraction.
template <uint32_t C>
__device__ __forceinline__ uint32_t red64(uint64_t x)
{
    x = (x >> 32) * C + (uint32_t)x;  // < 2^47.1
    x = (x >> 32) * C + (uint32_t)x;  // < 2^32 + 2^30
    const uint64_t m = (1ull << 32) - C;
    return (uint32_t)(x >= m ? x - m : x);
}

template <uint32_t C>
__device__ __forceinline__ void matvec(const uint32_t* M, uint32_t& v0, uint32_t& v1, uint32_t& v2)
{
    uint32_t r[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const uint64_t s = (uint64_t)red64<C>((uint64_t)M[3 * k] * v0) +
                           red64<C>((uint64_t)M[3 * k + 1] * v1) +
                           red64<C>((uint64_t)M[3 * k + 2] * v2);
        r[k] = red64<C>(s);
    }
    v0 = r[0];
    v1 = r[1];
    v2 = r[2];
}

__device__ __forceinline__ void apply(const MatPair& P, Mrg& s)
{
    matvec<kC1>(P.a, s.x0, s.x1, s.x2);
    matvec<kC2>(P.b, s.y0, s.y1, s.y2);
}

__device__ __forceinline__ Mrg load_state(const uint32_t* __restrict__ st, uint64_t stride, uint64_t i)
{
    Mrg s;
    s.x0 = __ldg(st + i);
    s.x1 = __ldg(st + stride + i);
    s.x2 = __ldg(st + 2 * stride + i);
    s.y0 = __ldg(st + 3 * stride + i);
    s.y1 = __ldg(st + 4 * stride + i);
    s.y2 = __ldg(st + 5 * stride + i);
    return s;
}

// ------------------------------------------------------------------ Philox

struct W4 {
    uint32_t x, y, z, w;
};

__device__ __forceinline__ W4 philox10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                       uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)kPM0 * c0;
        const uint64_t p1 = (uint64_t)kPM1 * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
        k0 += kPW0;
        k1 += kPW1;
    }
    return W4{c0, c1, c2, c3};
}

__device__ __forceinline__ W4 philox_blk(uint64_t blk, uint64_t g, uint32_t k0, uint32_t k1)
{
    return philox10((uint32_t)blk, (uint32_t)(blk >> 32), (uint32_t)g, (uint32_t)(g >> 32), k0, k1);
}

__device__ __forceinline__ uint32_t lane_of(const W4& v, uint32_t l)
{
    return l == 0 ? v.x : l == 1 ? v.y : l == 2 ? v.z : v.w;
}

// Generic per-draw access with a one-block cache (arbitrary offsets).
struct PhiloxCursor {
    uint64_t g;
    uint32_t k0, k1;
    uint64_t blk;
    bool valid;
    W4 v;
    __device__ __forceinline__ uint32_t word(uint64_t b, uint32_t lane)
    {
        if (!valid || b != blk) {
            v = philox_blk(b, g, k0, k1);
            blk = b;
            valid = true;
        }
        return lane_of(v, lane);
    }
};

// ------------------------------------------------------------------ conversions (R7)

__device__ __forceinline__ float to_f32(uint32_t w)
{
    return __fmul_rn(__uint2float_rn(w >> 8), 0x1p-24f);
}

__device__ __forceinline__ double mrg_f64(uint32_t z)
{
    return __dmul_rn(__uint2double_rn(z), 0x1.000000d00000bp-32);
}

__device__ __forceinline__ double philox_f64(uint32_t lo, uint32_t hi)
{
    const uint64_t b = (((uint64_t)hi << 32) | lo) >> 11;
    return __dmul_rn(__ull2double_rn(b), 0x1p-53);
}

// ------------------------------------------------------------------ stores

// One full 32-byte sector per thread: STG.E.ENL2.256 on sm_100a.
__device__ __forceinline__ void st_v8(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                      uint32_t e, uint32_t f, uint32_t g, uint32_t h)
{
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(a),
                 "r"(b), "r"(c), "r"(d), "r"(e), "r"(f), "r"(g), "r"(h)
                 : "memory");
}

__device__ __forceinline__ void st_v8f(void* p, float a, float b, float c, float d, float e,
                                       float f, float g, float h)
{
    st_v8(p, __float_as_uint(a), __float_as_uint(b), __float_as_uint(c), __float_as_uint(d),
          __float_as_uint(e), __float_as_uint(f), __float_as_uint(g), __float_as_uint(h));
}

__device__ __forceinline__ void st_v4d(void* p, double a, double b, double c, double d)
{
    st_v8(p, __double2loint(a), __double2hiint(a), __double2loint(b), __double2hiint(b),
          __double2loint(c), __double2hiint(c), __double2loint(d), __double2hiint(d));
}

// ------------------------------------------------------------------ reduction

__device__ __forceinline__ void block_reduce_add(uint64_t v, unsigned long long* dst)
{
    __shared__ unsigned long long part[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) part[warp] = v;
    __syncthreads();
    if (warp == 0) {
        const unsigned nw = (blockDim.x + 31) >> 5;
        v = lane < nw ? part[lane] : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && v) atomicAdd(dst, (unsigned long long)v);
    }
}

__device__ __forceinline__ uint32_t hit(uint32_t w0, uint32_t w1)
{
    const uint32_t X = w0 >> 8, Y = w1 >> 8;
    const uint64_t r2 = (uint64_t)X * X + (uint64_t)Y * Y;  // < 2^49
    return (uint32_t)(r2 >> 48) == 0u;
}

// ================================================================== kernels

__global__ void __launch_bounds__(256) mrg_seed_kernel(uint32_t* __restrict__ state, uint64_t n,
                                                       uint32_t b0, uint32_t b1, uint32_t b2,
                                                       uint32_t b3, uint32_t b4, uint32_t b5,
                                                       int table)
{
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Mrg s{b0, b1, b2, b3, b4, b5};
    uint64_t bits = i;
    for (int b = 0; bits; ++b, bits >>= 1)
        if (bits & 1) apply(g_jump_tab[table][b], s);
    state[i] = s.x0;
    state[n + i] = s.x1;
    state[2 * n + i] = s.x2;
    state[3 * n + i] = s.y0;
    state[4 * n + i] = s.y1;
    state[5 * n + i] = s.y2;
}

template <int KIND, bool VEC>
__global__ void __launch_bounds__(256) mrg_fill_kernel(const __grid_constant__ MrgLaunch P)
{
    using T = typename std::conditional<KIND == kF64, double,
                                        typename std::conditional<KIND == kF32, float, uint32_t>::type>::type;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t it = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; it < P.items; it += nthr) {
        const uint64_t j = it / P.ns;
        const uint64_t i = it - j * P.ns;
        Mrg s = load_state(P.state, P.stride, P.stream_begin + i);
        apply(P.seg[j], s);
        const uint64_t c0 = j * P.seg_len;
        const uint64_t len = min(P.seg_len, P.n - c0);
        T* o = reinterpret_cast<T*>(P.out) + i * P.n + c0;
        if (VEC) {
            for (uint64_t t = 0; t < len; t += 8) {
                uint32_t v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = mrg_next(s);
                if (KIND == kU32) {
                    st_v8(o + t, v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7]);
                } else if (KIND == kF32) {
                    st_v8f(o + t, to_f32(v[0]), to_f32(v[1]), to_f32(v[2]), to_f32(v[3]),
                           to_f32(v[4]), to_f32(v[5]), to_f32(v[6]), to_f32(v[7]));
                } else {
                    st_v4d(o + t, mrg_f64(v[0]), mrg_f64(v[1]), mrg_f64(v[2]), mrg_f64(v[3]));
                    st_v4d(o + t + 4, mrg_f64(v[4]), mrg_f64(v[5]), mrg_f64(v[6]), mrg_f64(v[7]));
                }
            }
        } else {
            for (uint64_t t = 0; t < len; ++t) {
                const uint32_t z = mrg_next(s);
                if (KIND == kU32) o[t] = (T)z;
                else if (KIND == kF32) o[t] = (T)to_f32(z);
                else o[t] = (T)mrg_f64(z);
            }
        }
    }
}

__global__ void __launch_bounds__(256) mrg_mc_kernel(const __grid_constant__ MrgLaunch P)
{
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    uint64_t total = 0;
    for (uint64_t it = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; it < P.items; it += nthr) {
        const uint64_t j = it / P.ns;
        const uint64_t i = it - j * P.ns;
        Mrg s = load_state(P.state, P.stride, P.stream_begin + i);
        apply(P.seg[j], s);
        const uint64_t c0 = j * P.seg_len;
        const uint32_t len = (uint32_t)min(P.seg_len, P.n - c0);
        uint32_t h = 0;
        uint32_t k = 0;
        for (; k + 4 <= len; k += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t w0 = mrg_next(s);
                const uint32_t w1 = mrg_next(s);
                h += hit(w0, w1);
            }
        }
        for (; k < len; ++k) {
            const uint32_t w0 = mrg_next(s);
            const uint32_t w1 = mrg_next(s);
            h += hit(w0, w1);
        }
        total += h;
        if (P.counts) atomicAdd(P.counts + i, (unsigned long long)h);
    }
    block_reduce_add(total, P.hits);
}

// Fast Philox fill: offset lane 0, rows a multiple of E elements, 32-byte
// aligned output. Work item = one 32-byte chunk = two counter blocks.
template <int KIND>
__global__ void __launch_bounds__(256) philox_fill_fast_kernel(const __grid_constant__ PhiloxLaunch P)
{
    constexpr uint64_t E = KIND == kF64 ? 4 : 8;  // elements per 32-byte chunk
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= P.items) return;
    // (i, j) of the chunk's first element, advanced incrementally by the stride.
    uint64_t i = (c * E) / P.n;
    uint64_t j = c * E - i * P.n;
    const uint64_t stride_e = nthr * E;
    const uint64_t qs = stride_e / P.n, rs = stride_e - qs * P.n;
    for (; c < P.items; c += nthr) {
        const uint64_t g = P.g0 + i;
        // u32/f32: draws j..j+7 = blocks b, b+1. f64: draws 2j..2j+7, same.
        const uint64_t b = P.o_blk + (KIND == kF64 ? j / 2 : j / 4);
        const W4 a = philox_blk(b, g, P.k0, P.k1);
        const W4 d = philox_blk(b + 1, g, P.k0, P.k1);
        void* o = reinterpret_cast<char*>(P.out) + (c * 32);
        if (KIND == kU32) {
            st_v8(o, a.x, a.y, a.z, a.w, d.x, d.y, d.z, d.w);
        } else if (KIND == kF32) {
            st_v8f(o, to_f32(a.x), to_f32(a.y), to_f32(a.z), to_f32(a.w), to_f32(d.x),
                   to_f32(d.y), to_f32(d.z), to_f32(d.w));
        } else {
            st_v4d(o, philox_f64(a.x, a.y), philox_f64(a.z, a.w), philox_f64(d.x, d.y),
                   philox_f64(d.z, d.w));
        }
        j += rs;
        i += qs;
        if (j >= P.n) {
            j -= P.n;
            ++i;
        }
    }
}

// Generic Philox fill: any offset, any row length, element-aligned output.
// Work item = up to 8 consecutive elements of the flat stream-major array.
template <int KIND>
__global__ void __launch_bounds__(256) philox_fill_generic_kernel(const __grid_constant__ PhiloxLaunch P)
{
    using T = typename std::conditional<KIND == kF64, double,
                                        typename std::conditional<KIND == kF32, float, uint32_t>::type>::type;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t total = P.ns * P.n;
    const uint32_t dpv = KIND == kF64 ? 2 : 1;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < P.items; c += nthr) {
        uint64_t e = c * 8;
        uint64_t i = e / P.n;
        uint64_t j = e - i * P.n;
        PhiloxCursor cur{P.g0 + i, P.k0, P.k1, 0, false, {}};
        for (int u = 0; u < 8 && e < total; ++u, ++e) {
            if (cur.g != P.g0 + i) {
                cur.g = P.g0 + i;
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

// Fused Philox Monte Carlo. FAST: offset lane 0 and even segment length, so
// sample pairs never straddle a counter block (two samples per block).
template <bool FAST>
__global__ void __launch_bounds__(256) philox_mc_kernel(const __grid_constant__ PhiloxLaunch P)
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
            const uint64_t b0 = P.o_blk + k0 / 2;
            const uint32_t nb = len / 2;
            uint32_t q = 0;
            for (; q + 2 <= nb; q += 2) {
                const W4 a = philox_blk(b0 + q, g, P.k0, P.k1);
                const W4 b = philox_blk(b0 + q + 1, g, P.k0, P.k1);
                h += hit(a.x, a.y) + hit(a.z, a.w) + hit(b.x, b.y) + hit(b.z, b.w);
            }
            for (; q < nb; ++q) {
                const W4 a = philox_blk(b0 + q, g, P.k0, P.k1);
                h += hit(a.x, a.y) + hit(a.z, a.w);
            }
            if (len & 1) {
                const W4 a = philox_blk(b0 + nb, g, P.k0, P.k1);
                h += hit(a.x, a.y);
            }
        } else {
            PhiloxCursor cur{g, P.k0, P.k1, 0, false, {}};
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

template <typename K>
cudaError_t occ(K kernel, int threads, int* out)
{
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, kernel, threads, 0);
}

}  // namespace

cudaError_t upload_jump_tables(const MatPair* sub51, const MatPair* str64)
{
    MatPair h[2][64] = {};
    for (int b = 0; b < 51; ++b) h[0][b] = sub51[b];
    for (int b = 0; b < 64; ++b) h[1][b] = str64[b];
    return cudaMemcpyToSymbol(g_jump_tab, h, sizeof h);
}

cudaError_t launch_mrg_seed(uint32_t* state, uint64_t n, const uint32_t base[6], int table, Grid g,
                            cudaStream_t s)
{
    mrg_seed_kernel<<<g.blocks, g.threads, 0, s>>>(state, n, base[0], base[1], base[2], base[3],
                                                   base[4], base[5], table);
    return cudaGetLastError();
}

cudaError_t launch_mrg_fill(const MrgLaunch& p, int kind, bool vec, Grid g, cudaStream_t s)
{
#define SHV_MRG_FILL(K, V) mrg_fill_kernel<K, V><<<g.blocks, g.threads, 0, s>>>(p)
    if (kind == kU32) vec ? SHV_MRG_FILL(kU32, true) : SHV_MRG_FILL(kU32, false);
    else if (kind == kF32) vec ? SHV_MRG_FILL(kF32, true) : SHV_MRG_FILL(kF32, false);
    else vec ? SHV_MRG_FILL(kF64, true) : SHV_MRG_FILL(kF64, false);
#undef SHV_MRG_FILL
    return cudaGetLastError();
}

cudaError_t launch_mrg_mc(const MrgLaunch& p, Grid g, cudaStream_t s)
{
    mrg_mc_kernel<<<g.blocks, g.threads, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_philox_fill(const PhiloxLaunch& p, int kind, bool fast, Grid g, cudaStream_t s)
{
    if (fast) {
        if (kind == kU32) philox_fill_fast_kernel<kU32><<<g.blocks, g.threads, 0, s>>>(p);
        else if (kind == kF32) philox_fill_fast_kernel<kF32><<<g.blocks, g.threads, 0, s>>>(p);
        else philox_fill_fast_kernel<kF64><<<g.blocks, g.threads, 0, s>>>(p);
    } else {
        if (kind == kU32) philox_fill_generic_kernel<kU32><<<g.blocks, g.threads, 0, s>>>(p);
        else if (kind == kF32) philox_fill_generic_kernel<kF32><<<g.blocks, g.threads, 0, s>>>(p);
        else philox_fill_generic_kernel<kF64><<<g.blocks, g.threads, 0, s>>>(p);
    }
    return cudaGetLastError();
}

cudaError_t launch_philox_mc(const PhiloxLaunch& p, bool fast, Grid g, cudaStream_t s)
{
    if (fast) philox_mc_kernel<true><<<g.blocks, g.threads, 0, s>>>(p);
    else philox_mc_kernel<false><<<g.blocks, g.threads, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t max_blocks_per_sm(int kernel, int kind, bool fast, int threads, int* out)
{
    switch (kernel) {
    case kKSeed:
        return occ(mrg_seed_kernel, threads, out);
    case kKMrgFill:
        if (kind == kU32) return fast ? occ(mrg_fill_kernel<kU32, true>, threads, out)
                                      : occ(mrg_fill_kernel<kU32, false>, threads, out);
        if (kind == kF32) return fast ? occ(mrg_fill_kernel<kF32, true>, threads, out)
                                      : occ(mrg_fill_kernel<kF32, false>, threads, out);
        return fast ? occ(mrg_fill_kernel<kF64, true>, threads, out)
                    : occ(mrg_fill_kernel<kF64, false>, threads, out);
    case kKMrgMc:
        return occ(mrg_mc_kernel, threads, out);
    case kKPhiloxFill:
        if (kind == kU32) return fast ? occ(philox_fill_fast_kernel<kU32>, threads, out)
                                      : occ(philox_fill_generic_kernel<kU32>, threads, out);
        if (kind == kF32) return fast ? occ(philox_fill_fast_kernel<kF32>, threads, out)
                                      : occ(philox_fill_generic_kernel<kF32>, threads, out);
        return fast ? occ(philox_fill_fast_kernel<kF64>, threads, out)
                    : occ(philox_fill_generic_kernel<kF64>, threads, out);
    case kKPhiloxMc:
        return fast ? occ(philox_mc_kernel<true>, threads, out)
                    : occ(philox_mc_kernel<false>, threads, out);
    }
    return cudaErrorInvalidValue;
}

}  // namespace shv
