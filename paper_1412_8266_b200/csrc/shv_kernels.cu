// shv_kernels.cu — sm_100a kernels of the ShoveRand hot path (arXiv 1412.8266).
//
// Design: persistent grids sized to the SM count; generator
// state in registers (P L257-258: MRG32k3a "only stores 6 integers"; Philox is
// stateless, P L329-331); numbers leave the SM as 256-byte contiguous runs of
// 32-byte vector stores (st.global.v8.b32 -> STG.E.ENL2.256, sm_100+), or
// never leave it (fused Monte Carlo: warp shuffle + shared-memory block
// reduction + one 64-bit atomic per block). No tensor cores: nothing here is
// a contraction. Generator arithmetic lives in shv_device.cuh.
//
// Compile-time variants (the kernel lab, tools/lab/, builds each):
//   SHV_MRG_STEP  0 = all-integer step, 2 = both components on the FP64 pipe
//                 (default; fastest measured; other forms live in tools/lab/)
//   SHV_MRG_STAGE 0 = each lane stores its own row directly (32-byte vector
//                 stores); 2 = lanes stage 256 B in shared memory and the warp
//                 writes 256-byte runs; 1 (default) = stage the 8-byte (f64)
//                 outputs only: the compute-bound u32/f32 fills run faster
//                 without staging (more warps), the HBM-bound f64 fill needs it
#include <atomic>
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "../../include/shv_device.cuh"
#include "shv_internal.h"

#ifndef SHV_MRG_STEP
#define SHV_MRG_STEP 2
#endif
#ifndef SHV_MRG_STAGE
#define SHV_MRG_STAGE 1
#endif

namespace shv {

// Jump tables: [0][b] = A^(2^(76+b)) (substreams, b < 51),
//              [1][b] = A^(2^(127+b)) (streams, b < 64).
__device__ MatPair g_jump_tab[2][64];

namespace {

using namespace dev;

template <int KIND>
using OutT = typename std::conditional<KIND == kF64, double,
                                       typename std::conditional<KIND == kF32, float, uint32_t>::type>::type;

#if SHV_MRG_STEP == 2
using Gen = MrgD;
__device__ __forceinline__ Gen make_gen(const Mrg& s) { return to_fp64(s); }
#else
using Gen = Mrg;
__device__ __forceinline__ Gen make_gen(const Mrg& s) { return s; }
#endif

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

// Start state of work item (stream i of the launch, segment j).
__device__ __forceinline__ Gen item_state(const MrgLaunch& P, uint64_t i, uint64_t j)
{
    Mrg s = load_state(P.state, P.stride, P.stream_begin + i);
    apply(P.seg[j].a, P.seg[j].b, s);
    return make_gen(s);
}

template <int KIND>
__device__ __forceinline__ uint4 pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d)
{
    if (KIND == kF32)
        return make_uint4(__float_as_uint(to_f32(a)), __float_as_uint(to_f32(b)),
                          __float_as_uint(to_f32(c)), __float_as_uint(to_f32(d)));
    return make_uint4(a, b, c, d);
}

// Bytes each lane stages per round (256: eight 1-KB store instructions per
// round, each covering four rows x 256 B; 128: four instructions, eight rows
// x 128 B each), and the min-blocks hint of the vector kernel.
#ifndef SHV_MRG_RB
#define SHV_MRG_RB 256
#endif
#ifndef SHV_MRG_MINB
#define SHV_MRG_MINB 4  // <= 64 registers (fewer spill or slow the FP64 step; lab)
#endif
constexpr unsigned kRB = SHV_MRG_RB;
constexpr unsigned kPieces = kRB / 16;  // 16-byte pieces per lane per round

// Staging slot of 16-byte piece q of lane L, conflict-free for the per-lane
// 128-bit writes (8 lanes, same q) and for the write-out reads (8 lanes that
// read pieces 2p resp. 2p+1 of one source lane (kRB=256) or two (kRB=128)).
__device__ __forceinline__ unsigned slot(unsigned L, unsigned q)
{
    if (kRB == 256) return 16 * L + 8 * (q & 1) + (((q >> 1) + L) & 7);
    return 8 * L + ((q + L) & 7);
}

// 8 values -> staging pieces (u32/f32: 2 pieces; f64: 4 pieces).
template <int KIND>
__device__ __forceinline__ void stage8(uint4* wb, unsigned lane, unsigned q0, Gen& s)
{
    uint32_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = mrg_next(s);
    if (KIND == kF64) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double a = mrg_f64(v[2 * u]), b = mrg_f64(v[2 * u + 1]);
            wb[slot(lane, q0 + u)] = make_uint4(__double2loint(a), __double2hiint(a),
                                                __double2loint(b), __double2hiint(b));
        }
    } else {
        wb[slot(lane, q0)] = pack4<KIND>(v[0], v[1], v[2], v[3]);
        wb[slot(lane, q0 + 1)] = pack4<KIND>(v[4], v[5], v[6], v[7]);
    }
}

// Write one staged round of the warp: lane L's cnt values (kRB bytes at most)
// go to row_L + r values; each store instruction covers 1024/kRB source lanes
// x kRB contiguous bytes.
template <typename T>
__device__ __forceinline__ void write_round(const uint4* wb, unsigned lane, uint32_t r, uint32_t cnt, uint64_t row)
{
    __syncwarp();
#pragma unroll
    for (unsigned k = 0; k < kRB / 32; ++k) {
        const unsigned src = (1024 / kRB) * k + lane / (kRB / 32), p = lane % (kRB / 32);
        const uint32_t scnt = __shfl_sync(0xffffffffu, cnt, src);
        const uint64_t srow = __shfl_sync(0xffffffffu, row, src);
        if (32 * p < scnt * sizeof(T))
            st_v8(reinterpret_cast<char*>(srow) + (uint64_t)r * sizeof(T) + 32 * p, wb[slot(src, 2 * p)],
                  wb[slot(src, 2 * p + 1)]);
    }
    __syncwarp();
}

// TinyMT32: 8 values -> staging pieces (u32/f32: 8 words; f64: 16 words, two
// per value like Philox, R7/R15).
template <int KIND>
__device__ __forceinline__ void stage8_tm(uint4* wb, unsigned lane, unsigned q0, TinyMT& t)
{
    if (KIND == kF64) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t a0 = tinymt_next(t), a1 = tinymt_next(t), b0 = tinymt_next(t), b1 = tinymt_next(t);
            const double a = philox_f64(a0, a1), b = philox_f64(b0, b1);
            wb[slot(lane, q0 + u)] = make_uint4(__double2loint(a), __double2hiint(a), __double2loint(b),
                                                __double2hiint(b));
        }
    } else {
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = tinymt_next(t);
        wb[slot(lane, q0)] = pack4<KIND>(v[0], v[1], v[2], v[3]);
        wb[slot(lane, q0 + 1)] = pack4<KIND>(v[4], v[5], v[6], v[7]);
    }
}

__device__ __forceinline__ TinyMT tm_load(const TinyMtLaunch& P, uint64_t i)
{
    const uint64_t n = P.stride;
    const uint32_t* pr = P.params + 3 * ((P.first + i) / P.group_size - P.group0);
    return TinyMT{__ldg(P.state + i), __ldg(P.state + n + i), __ldg(P.state + 2 * n + i),
                  __ldg(P.state + 3 * n + i), __ldg(pr), __ldg(pr + 1), __ldg(pr + 2)};
}

__device__ __forceinline__ void tm_store(const TinyMtLaunch& P, uint64_t i, const TinyMT& t)
{
    const uint64_t n = P.stride;
    P.state[i] = t.s0;
    P.state[n + i] = t.s1;
    P.state[2 * n + i] = t.s2;
    P.state[3 * n + i] = t.s3;
}

// ================================================================== kernels

// Per-stream start states (row a3). Thread t of T handles streams t, t+T,
// t+2T, ...: its first state is the product of the per-bit jump tables for t
// (<= log2 T mat-vecs), each next one is one mat-vec with step = A^(T*spacing)
// (host-built). ~2 mat-vecs per stream instead of popcount(i) <= 20; the SoA
// stores of a warp are coalesced.
__global__ void __launch_bounds__(256) mrg_seed_kernel(uint32_t* __restrict__ state, uint64_t n,
                                                       uint32_t b0, uint32_t b1, uint32_t b2,
                                                       uint32_t b3, uint32_t b4, uint32_t b5,
                                                       int table, MatPair step)
{
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    Mrg s{b0, b1, b2, b3, b4, b5};
    uint64_t bits = t;
    for (int b = 0; bits; ++b, bits >>= 1)
        if (bits & 1) apply(g_jump_tab[table][b].a, g_jump_tab[table][b].b, s);
    for (uint64_t i = t; i < n; i += T) {
        state[i] = s.x0;
        state[n + i] = s.x1;
        state[2 * n + i] = s.x2;
        state[3 * n + i] = s.y0;
        state[4 * n + i] = s.y1;
        state[5 * n + i] = s.y2;
        if (i + T < n) apply(step.a, step.b, s);
    }
}

// MRG32k3a fill, vector path (32-byte aligned rows, seg_len % 8 == 0).
// Staged: each lane generates 256 B of its row into shared memory per round,
// then the warp writes them as eight 1-KB store instructions, each covering
// four rows x 256 contiguous bytes.
template <int KIND>
__host__ __device__ constexpr bool mrg_staged()
{
    return SHV_MRG_STAGE == 2 || (SHV_MRG_STAGE == 1 && KIND == kF64);
}

template <int KIND>
__global__ void __launch_bounds__(256, SHV_MRG_MINB) mrg_fill_vec_kernel(const __grid_constant__ MrgLaunch P)
{
    using T = OutT<KIND>;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if constexpr (mrg_staged<KIND>()) {
    extern __shared__ uint4 smem[];
    uint4* wb = smem + warp * (32 * kPieces);
    constexpr uint32_t G = kRB / sizeof(T);  // values per lane per round
    const uint64_t wstride = (uint64_t)gridDim.x * (blockDim.x >> 5) * 32;
    for (uint64_t base = ((uint64_t)blockIdx.x * (blockDim.x >> 5) + warp) * 32; base < P.items;
         base += wstride) {
        const uint64_t it = base + lane;
        uint32_t len = 0;
        uint64_t row = 0;
        Gen s{};
        if (it < P.items) {
            const uint64_t j = it / P.ns;
            const uint64_t i = it - j * P.ns;
            s = item_state(P, i, j);
            const uint64_t c0 = j * P.seg_len;
            len = (uint32_t)min(P.seg_len, P.n - c0);
            row = (uint64_t)P.out + (i * P.n + c0) * sizeof(T);
        }
        const uint32_t maxlen = __reduce_max_sync(0xffffffffu, len);
        for (uint32_t r = 0; r < maxlen; r += G) {
            const uint32_t cnt = len > r ? min(G, len - r) : 0u;
            if (cnt == G) {
#pragma unroll
                for (unsigned g = 0; g < G / 8; ++g) stage8<KIND>(wb, lane, g * (KIND == kF64 ? 4 : 2), s);
            } else {
                for (unsigned g = 0; g < cnt / 8; ++g) stage8<KIND>(wb, lane, g * (KIND == kF64 ? 4 : 2), s);
            }
            write_round<T>(wb, lane, r, cnt, row);
        }
    }
    } else {
    (void)lane;
    (void)warp;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t it = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; it < P.items; it += nthr) {
        const uint64_t j = it / P.ns;
        const uint64_t i = it - j * P.ns;
        Gen s = item_state(P, i, j);
        const uint64_t c0 = j * P.seg_len;
        const uint64_t len = min(P.seg_len, P.n - c0);
        T* o = reinterpret_cast<T*>(P.out) + i * P.n + c0;
        for (uint64_t t = 0; t < len; t += 8) {
            uint32_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = mrg_next(s);
            if (KIND == kU32) {
                st_v8(o + t, v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7]);
            } else if (KIND == kF32) {
                st_v8f(o + t, to_f32(v[0]), to_f32(v[1]), to_f32(v[2]), to_f32(v[3]), to_f32(v[4]),
                       to_f32(v[5]), to_f32(v[6]), to_f32(v[7]));
            } else {
                st_v4d(o + t, mrg_f64(v[0]), mrg_f64(v[1]), mrg_f64(v[2]), mrg_f64(v[3]));
                st_v4d(o + t + 4, mrg_f64(v[4]), mrg_f64(v[5]), mrg_f64(v[6]), mrg_f64(v[7]));
            }
        }
    }
    }
}

// MRG32k3a fill, scalar path (any row length / element-aligned pointer).
template <int KIND>
__global__ void __launch_bounds__(256) mrg_fill_scalar_kernel(const __grid_constant__ MrgLaunch P)
{
    using T = OutT<KIND>;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t it = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; it < P.items; it += nthr) {
        const uint64_t j = it / P.ns;
        const uint64_t i = it - j * P.ns;
        Gen s = item_state(P, i, j);
        const uint64_t c0 = j * P.seg_len;
        const uint64_t len = min(P.seg_len, P.n - c0);
        T* o = reinterpret_cast<T*>(P.out) + i * P.n + c0;
        for (uint64_t t = 0; t < len; ++t) {
            const uint32_t z = mrg_next(s);
            if (KIND == kU32) o[t] = (T)z;
            else if (KIND == kF32) o[t] = (T)to_f32(z);
            else o[t] = (T)mrg_f64(z);
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
        Gen s = item_state(P, i, j);
        const uint64_t c0 = j * P.seg_len;
        const uint32_t len = (uint32_t)min(P.seg_len, P.n - c0);
        uint32_t h = 0;
        uint32_t k = 0;
        for (; k + 12 <= len; k += 12) {
#pragma unroll
            for (int u = 0; u < 12; ++u) {
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
                const W4 a = philox10_from_r2(pa, q, (uint32_t)p1, (uint32_t)(g >> 32), k0, k1);
                const W4 d = philox10_from_r2(pb, q, (uint32_t)p1, (uint32_t)(g >> 32), k0, k1);
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
                for (uint32_t r = 0; r < nb; ++r) {
                    const W4 a = philox10_from_r2(pa, q, (uint32_t)p1, (uint32_t)(g >> 32), key0, key1);
                    h += hit_fp64(a.x, a.y) + hit_fp64(a.z, a.w);
                    pa = add64w(pa, kPM0);
                }
                b = add64(b, nb);
            } else {
                for (uint32_t r = 0; r < nb; ++r) {
                    const uint64_t pa = (uint64_t)kPM0 * (uint32_t)b;
                    const W4 a = philox10_from_r1((uint32_t)(pa >> 32), (uint32_t)pa, (uint32_t)(p1 >> 32),
                                                  (uint32_t)p1, (uint32_t)(b >> 32), (uint32_t)(g >> 32), key0, key1);
                    h += hit_fp64(a.x, a.y) + hit_fp64(a.z, a.w);
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


// ------------------------------------------------------------------ Threefry4x64-20 (NEXT-2)

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

// ------------------------------------------------------------------ TinyMT32 (NEXT-3)

// One block of 128 threads per parameter set: thread c builds column c of the
// transition T (next_state of unit vector e_c), then the block squares the
// matrix 64 times (T^(2^64), the slice length) and log2_gs - 1 more times,
// storing (T^(2^64))^(2^b) for b < log2_gs.
__global__ void __launch_bounds__(128) tinymt_prep_kernel(const uint32_t* __restrict__ params, int log2_gs,
                                                          uint32_t* __restrict__ tables)
{
    __shared__ uint4 M[128], N[128];
    const unsigned c = threadIdx.x;
    const uint32_t* pr = params + 3 * blockIdx.x;
    TinyMT t{0, 0, 0, 0, pr[0], pr[1], pr[2]};
    (c < 32 ? t.s0 : c < 64 ? t.s1 : c < 96 ? t.s2 : t.s3) = 1u << (c & 31);
    tinymt_next_state(t);
    M[c] = make_uint4(t.s0, t.s1, t.s2, t.s3);
    __syncthreads();
    for (int k = 0; k < 64 + log2_gs; ++k) {
        if (k >= 64) {  // M = (T^(2^64))^(2^(k-64)): emit table entry k-64
            reinterpret_cast<uint4*>(tables)[((size_t)blockIdx.x * log2_gs + (k - 64)) * 128 + c] = M[c];
            if (k == 64 + log2_gs - 1) break;
        }
        const uint4 x = M[c];  // column c of M*M = M applied to column c of M
        const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
        uint4 y = make_uint4(0, 0, 0, 0);
        for (int b = 0; b < 128; ++b)
            if ((xs[b >> 5] >> (b & 31)) & 1u) {
                const uint4 col = M[b];
                y.x ^= col.x;
                y.y ^= col.y;
                y.z ^= col.z;
                y.w ^= col.w;
            }
        N[c] = y;
        __syncthreads();
        M[c] = N[c];
        __syncthreads();
    }
}

// Stream i: init(params of its group, seed), then slice s = g % group_size
// via the per-bit tables (popcount(s) GF(2) mat-vecs).
__global__ void __launch_bounds__(256) tinymt_seed_kernel(const TinyMtLaunch P, uint32_t seed,
                                                          const uint32_t* __restrict__ tables, int log2_gs)
{
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.ns) return;
    const uint64_t g = P.first + i;
    const uint64_t grp = g / P.group_size - P.group0;
    const uint32_t* pr = P.params + 3 * grp;
    TinyMT t;
    tinymt_init(t, pr[0], pr[1], pr[2], seed);
    const uint32_t slice = (uint32_t)(g % P.group_size);
    for (int b = 0; b < log2_gs; ++b)
        if ((slice >> b) & 1u) gf2_apply(tables + ((size_t)grp * log2_gs + b) * 512, t);
    tm_store(P, i, t);
}

// Vector fill: one stream per lane, staged 256-byte runs (as the MRG kernel).
template <int KIND>
__global__ void __launch_bounds__(256, 4) tinymt_fill_vec_kernel(const __grid_constant__ TinyMtLaunch P)
{
    using T = OutT<KIND>;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    extern __shared__ uint4 smem[];
    uint4* wb = smem + warp * (32 * kPieces);
    constexpr uint32_t G = kRB / sizeof(T);
    const uint64_t wstride = (uint64_t)gridDim.x * (blockDim.x >> 5) * 32;
    for (uint64_t base = ((uint64_t)blockIdx.x * (blockDim.x >> 5) + warp) * 32; base < P.ns; base += wstride) {
        const uint64_t i = base + lane;
        const bool on = i < P.ns;
        TinyMT t = on ? tm_load(P, i) : TinyMT{};
        const uint32_t len = on ? (uint32_t)P.n : 0u;
        const uint64_t row = on ? (uint64_t)P.out + i * P.n * sizeof(T) : 0;
        for (uint32_t r = 0; r < (uint32_t)P.n; r += G) {
            const uint32_t cnt = len > r ? min(G, len - r) : 0u;
            for (unsigned g = 0; g < cnt / 8; ++g) stage8_tm<KIND>(wb, lane, g * (KIND == kF64 ? 4 : 2), t);
            write_round<T>(wb, lane, r, cnt, row);
        }
        if (on) tm_store(P, i, t);
    }
}

template <int KIND>
__global__ void __launch_bounds__(256) tinymt_fill_scalar_kernel(const __grid_constant__ TinyMtLaunch P)
{
    using T = OutT<KIND>;
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.ns) return;
    TinyMT t = tm_load(P, i);
    T* o = reinterpret_cast<T*>(P.out) + i * P.n;
    for (uint64_t j = 0; j < P.n; ++j) {
        if (KIND == kU32) o[j] = (T)tinymt_next(t);
        else if (KIND == kF32) o[j] = (T)to_f32(tinymt_next(t));
        else {
            const uint32_t lo = tinymt_next(t);
            o[j] = (T)philox_f64(lo, tinymt_next(t));
        }
    }
    tm_store(P, i, t);
}

// Sequential advance by P.steps draws (TinyMT32 jumps, S L355).
__global__ void __launch_bounds__(256) tinymt_advance_kernel(const TinyMtLaunch P)
{
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.ns) return;
    TinyMT t = tm_load(P, i);
    for (uint64_t k = 0; k < P.steps; ++k) tinymt_next_state(t);
    tm_store(P, i, t);
}

__global__ void __launch_bounds__(256) tinymt_mc_kernel(const __grid_constant__ TinyMtLaunch P)
{
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t h = 0;
    if (i < P.ns) {
        TinyMT t = tm_load(P, i);
        for (uint64_t k = 0; k < P.n; ++k) {
            const uint32_t w0 = tinymt_next(t);
            h += hit(w0, tinymt_next(t));
        }
        tm_store(P, i, t);
        if (P.counts) atomicAdd(P.counts + i, (unsigned long long)h);
    }
    block_reduce_add(h, P.hits);
}

template <typename K>
cudaError_t occ(K kernel, int threads, size_t smem, int* out)
{
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, kernel, threads, smem);
}

// Opt the vector fill kernels into > 48 KB of dynamic shared memory, once per
// device (the attribute is per function and context).
template <int KIND>
cudaError_t ensure_smem_attr()
{
    static std::atomic<uint64_t> done{0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(mrg_fill_vec_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)mrg_fill_smem(256, KIND));
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_release);
    return e;
}

template <int KIND>
cudaError_t launch_vec(const MrgLaunch& p, Grid g, cudaStream_t s)
{
    const size_t smem = mrg_fill_smem((int)g.threads, KIND);
    if (smem > 48 * 1024) {
        cudaError_t e = ensure_smem_attr<KIND>();
        if (e != cudaSuccess) return e;
    }
    mrg_fill_vec_kernel<KIND><<<g.blocks, g.threads, smem, s>>>(p);
    return cudaGetLastError();
}

}  // namespace

size_t mrg_fill_smem(int threads, int kind)
{
    const bool staged = kind == kU32 ? mrg_staged<kU32>() : kind == kF32 ? mrg_staged<kF32>() : mrg_staged<kF64>();
    return staged ? (size_t)(threads / 32) * 32 * kRB : 0;
}

cudaError_t upload_jump_tables(const MatPair* sub51, const MatPair* str64)
{
    MatPair h[2][64] = {};
    for (int b = 0; b < 51; ++b) h[0][b] = sub51[b];
    for (int b = 0; b < 64; ++b) h[1][b] = str64[b];
    return cudaMemcpyToSymbol(g_jump_tab, h, sizeof h);
}

cudaError_t launch_mrg_seed(uint32_t* state, uint64_t n, const uint32_t base[6], int table,
                            const MatPair& step, Grid g, cudaStream_t s)
{
    mrg_seed_kernel<<<g.blocks, g.threads, 0, s>>>(state, n, base[0], base[1], base[2], base[3],
                                                   base[4], base[5], table, step);
    return cudaGetLastError();
}

cudaError_t launch_mrg_fill(const MrgLaunch& p, int kind, bool vec, Grid g, cudaStream_t s)
{
    if (vec) {
        if (kind == kU32) return launch_vec<kU32>(p, g, s);
        if (kind == kF32) return launch_vec<kF32>(p, g, s);
        return launch_vec<kF64>(p, g, s);
    }
    if (kind == kU32) mrg_fill_scalar_kernel<kU32><<<g.blocks, g.threads, 0, s>>>(p);
    else if (kind == kF32) mrg_fill_scalar_kernel<kF32><<<g.blocks, g.threads, 0, s>>>(p);
    else mrg_fill_scalar_kernel<kF64><<<g.blocks, g.threads, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_mrg_mc(const MrgLaunch& p, Grid g, cudaStream_t s)
{
    mrg_mc_kernel<<<g.blocks, g.threads, 0, s>>>(p);
    return cudaGetLastError();
}

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

cudaError_t launch_tinymt_prep(const uint32_t* params, uint64_t n_groups, int log2_gs, uint32_t* tables,
                               cudaStream_t s)
{
    if (log2_gs == 0 || n_groups == 0) return cudaSuccess;
    tinymt_prep_kernel<<<(unsigned)n_groups, 128, 0, s>>>(params, log2_gs, tables);
    return cudaGetLastError();
}

cudaError_t launch_tinymt_seed(const TinyMtLaunch& p, uint32_t seed, const uint32_t* tables, int log2_gs, Grid g,
                               cudaStream_t s)
{
    tinymt_seed_kernel<<<g.blocks, g.threads, 0, s>>>(p, seed, tables, log2_gs);
    return cudaGetLastError();
}

template <int KIND>
cudaError_t launch_tm_vec(const TinyMtLaunch& p, Grid g, cudaStream_t s)
{
    const size_t smem = (size_t)(g.threads / 32) * 32 * kRB;
    static std::atomic<uint64_t> done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (!(done.load() & bit)) {
        cudaError_t e = cudaFuncSetAttribute(tinymt_fill_vec_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)((256 / 32) * 32 * kRB));
        if (e != cudaSuccess) return e;
        done.fetch_or(bit);
    }
    tinymt_fill_vec_kernel<KIND><<<g.blocks, g.threads, smem, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_tinymt_fill(const TinyMtLaunch& p, int kind, bool vec, Grid g, cudaStream_t s)
{
    if (vec) {
        if (kind == kU32) return launch_tm_vec<kU32>(p, g, s);
        if (kind == kF32) return launch_tm_vec<kF32>(p, g, s);
        return launch_tm_vec<kF64>(p, g, s);
    }
    if (kind == kU32) tinymt_fill_scalar_kernel<kU32><<<g.blocks, g.threads, 0, s>>>(p);
    else if (kind == kF32) tinymt_fill_scalar_kernel<kF32><<<g.blocks, g.threads, 0, s>>>(p);
    else tinymt_fill_scalar_kernel<kF64><<<g.blocks, g.threads, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_tinymt_advance(const TinyMtLaunch& p, Grid g, cudaStream_t s)
{
    tinymt_advance_kernel<<<g.blocks, g.threads, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_tinymt_mc(const TinyMtLaunch& p, Grid g, cudaStream_t s)
{
    tinymt_mc_kernel<<<g.blocks, g.threads, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t max_blocks_per_sm(int kernel, int kind, bool fast, int threads, int* out)
{
    switch (kernel) {
    case kKSeed:
        return occ(mrg_seed_kernel, threads, 0, out);
    case kKMrgFill: {
        const size_t sm = fast ? mrg_fill_smem(threads, kind) : 0;
        if (fast && sm > 48 * 1024) {
            cudaError_t e = kind == kU32 ? ensure_smem_attr<kU32>()
                          : kind == kF32 ? ensure_smem_attr<kF32>() : ensure_smem_attr<kF64>();
            if (e != cudaSuccess) return e;
        }
        if (kind == kU32) return fast ? occ(mrg_fill_vec_kernel<kU32>, threads, sm, out)
                                      : occ(mrg_fill_scalar_kernel<kU32>, threads, 0, out);
        if (kind == kF32) return fast ? occ(mrg_fill_vec_kernel<kF32>, threads, sm, out)
                                      : occ(mrg_fill_scalar_kernel<kF32>, threads, 0, out);
        return fast ? occ(mrg_fill_vec_kernel<kF64>, threads, sm, out)
                    : occ(mrg_fill_scalar_kernel<kF64>, threads, 0, out);
    }
    case kKMrgMc:
        return occ(mrg_mc_kernel, threads, 0, out);
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
    case kKTinyFill: {
        const size_t sm = (size_t)(threads / 32) * 32 * kRB;
        if (kind == kU32) {
            cudaFuncSetAttribute(tinymt_fill_vec_kernel<kU32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(8 * 32 * kRB));
            return occ(tinymt_fill_vec_kernel<kU32>, threads, sm, out);
        }
        if (kind == kF32) {
            cudaFuncSetAttribute(tinymt_fill_vec_kernel<kF32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(8 * 32 * kRB));
            return occ(tinymt_fill_vec_kernel<kF32>, threads, sm, out);
        }
        cudaFuncSetAttribute(tinymt_fill_vec_kernel<kF64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(8 * 32 * kRB));
        return occ(tinymt_fill_vec_kernel<kF64>, threads, sm, out);
    }
    case kKTinyMc:
        return occ(tinymt_mc_kernel, threads, 0, out);
    case kKThreefryFill:
        if (kind == kU32) return fast ? occ(threefry_fill_fast_kernel<kU32>, threads, 0, out)
                                      : occ(threefry_fill_generic_kernel<kU32>, threads, 0, out);
        if (kind == kF32) return fast ? occ(threefry_fill_fast_kernel<kF32>, threads, 0, out)
                                      : occ(threefry_fill_generic_kernel<kF32>, threads, 0, out);
        return fast ? occ(threefry_fill_fast_kernel<kF64>, threads, 0, out)
                    : occ(threefry_fill_generic_kernel<kF64>, threads, 0, out);
    case kKThreefryMc:
        return fast ? occ(threefry_mc_kernel<true>, threads, 0, out) : occ(threefry_mc_kernel<false>, threads, 0, out);
    case kKPhiloxMcKeyed:
        return fast ? occ(philox_mc_kernel<true, true>, threads, 0, out)
                    : occ(philox_mc_kernel<false, true>, threads, 0, out);
    }
    return cudaErrorInvalidValue;
}

}  // namespace shv
