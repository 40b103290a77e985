// kernels_tinymt32.cu — TinyMT32 kernels (NEXT-3; R15; S L355): GF(2)
// jump tables, per-stream seeding, staged bulk fills, sequential advance and
// the fused Monte Carlo pi kernel. Stateful: every launch writes the SoA state
// back.
#include "kernels_common.cuh"

#ifndef SHV_TM_RB
#define SHV_TM_RB 256  // bytes per lane per staged round of the TinyMT32 vector fill (128: 3.72 vs 3.37 ms, lab41)
#endif

namespace shv {
namespace {

constexpr unsigned kTmRB = SHV_TM_RB;

using u128 = unsigned __int128;

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
            wb[slot<kTmRB>(lane, q0 + u)] = make_uint4(__double2loint(a), __double2hiint(a), __double2loint(b),
                                                    __double2hiint(b));
        }
    } else {
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = tinymt_next(t);
        wb[slot<kTmRB>(lane, q0)] = pack4<KIND>(v[0], v[1], v[2], v[3]);
        wb[slot<kTmRB>(lane, q0 + 1)] = pack4<KIND>(v[4], v[5], v[6], v[7]);
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

// Vector fill: one stream per lane, staged 256-byte runs (as the MRG kernel;
// 128-byte runs give four blocks per SM instead of three but measured slower).
template <int KIND>
__global__ void __launch_bounds__(256, 4) tinymt_fill_vec_kernel(const __grid_constant__ TinyMtLaunch P)
{
    using T = OutT<KIND>;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    extern __shared__ uint4 smem[];
    uint4* wb = smem + warp * (32 * (kTmRB / 16));
    constexpr uint32_t G = kTmRB / sizeof(T);
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
            write_round<T, kTmRB>(wb, lane, r, cnt, row);
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

// ---- jump-ahead by a polynomial (shv_jump on TinyMT32 handles, any n) ----
// The transition T (tinymt_next_state) is linear over GF(2) on the 128-bit
// state (bit 31 of s0 is masked out of the recurrence but carried into the
// next s0, so it is part of the vector). For a state v, let m(x) be the
// minimal polynomial of v under T: m(T) T^k v = 0 for every k, so all states
// of v's orbit (the streams of one parameter set are slices of one sequence)
// share it. Then T^n w = r(T) w with r = x^n mod m, for every w of the orbit:
// the jump costs deg(m) <= 128 transition steps per stream, whatever n is.

struct Poly256 {
    uint32_t w[9];  // bits 0..287 (coefficient i = bit i)
};

__device__ __forceinline__ int poly_deg(const uint32_t* a, int words)
{
    for (int k = words - 1; k >= 0; --k)
        if (a[k]) return 32 * k + 31 - __clz(a[k]);
    return -1;
}

// a (< 2^(2*128)) reduced mod m (deg dm), in place.
__device__ __forceinline__ void poly_mod(uint32_t* a, const uint32_t* m, int dm)
{
    for (int i = 255; i >= dm; --i) {
        if ((a[i >> 5] >> (i & 31)) & 1u) {
            const int sh = i - dm;
            // a ^= m << sh (m has dm+1 <= 129 bits: 5 words)
            const int ws = sh >> 5, bs = sh & 31;
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                const uint32_t lo = m[k] << bs;
                const uint32_t hi = bs ? (m[k] >> (32 - bs)) : 0u;
                if (ws + k < 9) a[ws + k] ^= lo;
                if (ws + k + 1 < 9) a[ws + k + 1] ^= hi;
            }
        }
    }
}

// One thread per parameter set present in the launch (absolute group
// G = P.first / group_size + g): minimal polynomial of the state of the first
// launch stream of group G by Krylov elimination, then
// r_g = x^n mod m_g by left-to-right squaring (squaring over GF(2) spreads
// the bits) and multiplication by x. out[4g..4g+3] = r_g (degree < 128).
__global__ void __launch_bounds__(64) tinymt_jump_poly_kernel(const TinyMtLaunch P, uint64_t ngroups, uint64_t n,
                                                              uint32_t* __restrict__ out)
{
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ngroups) return;
    const uint64_t G = P.first / P.group_size + g;
    TinyMT t = tm_load(P, (G * P.group_size > P.first ? G * P.group_size : P.first) - P.first);
    // echelon basis of the Krylov vectors indexed by pivot (highest set bit),
    // each with its polynomial tag; a new vector is reduced in decreasing pivot
    // order, so a XOR never sets a pivot bit already cleared
    uint32_t bv[128][4], bt[128][5];
    uint32_t have[4] = {0, 0, 0, 0};
    uint32_t m[5] = {0, 0, 0, 0, 0};
    for (int k = 0; k <= 128; ++k) {
        uint32_t v[4] = {t.s0, t.s1, t.s2, t.s3};
        uint32_t tag[5] = {0, 0, 0, 0, 0};
        tag[k >> 5] |= 1u << (k & 31);
        for (int p = 127; p >= 0; --p) {
            if (((v[p >> 5] & have[p >> 5]) >> (p & 31)) & 1u) {
#pragma unroll
                for (int q = 0; q < 4; ++q) v[q] ^= bv[p][q];
#pragma unroll
                for (int q = 0; q < 5; ++q) tag[q] ^= bt[p][q];
            }
        }
        const int d = poly_deg(v, 4);
        if (d < 0) {  // T^k v is a combination of the earlier ones: m = tag
#pragma unroll
            for (int q = 0; q < 5; ++q) m[q] = tag[q];
            break;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) bv[d][q] = v[q];
#pragma unroll
        for (int q = 0; q < 5; ++q) bt[d][q] = tag[q];
        have[d >> 5] |= 1u << (d & 31);
        tinymt_next_state(t);
    }
    const int dm = poly_deg(m, 5);
    uint32_t r[9] = {1, 0, 0, 0, 0, 0, 0, 0, 0};  // x^0
    if (dm == 0) r[0] = 0;  // v = 0: the zero state stays zero
    for (int b = 63; b >= 0 && dm > 0; --b) {
        uint32_t sq[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // r^2: bit i -> bit 2i
            uint32_t lo = r[k] & 0xFFFFu, hi = r[k] >> 16;
            lo = (lo | (lo << 8)) & 0x00FF00FFu;
            lo = (lo | (lo << 4)) & 0x0F0F0F0Fu;
            lo = (lo | (lo << 2)) & 0x33333333u;
            lo = (lo | (lo << 1)) & 0x55555555u;
            hi = (hi | (hi << 8)) & 0x00FF00FFu;
            hi = (hi | (hi << 4)) & 0x0F0F0F0Fu;
            hi = (hi | (hi << 2)) & 0x33333333u;
            hi = (hi | (hi << 1)) & 0x55555555u;
            sq[2 * k] = lo;
            sq[2 * k + 1] = hi;
        }
        poly_mod(sq, m, dm);
        if ((n >> b) & 1u) {  // * x
            for (int k = 8; k > 0; --k) sq[k] = (sq[k] << 1) | (sq[k - 1] >> 31);
            sq[0] <<= 1;
            poly_mod(sq, m, dm);
        }
#pragma unroll
        for (int k = 0; k < 9; ++k) r[k] = sq[k];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) out[4 * g + k] = r[k];
}

// Per stream: state <- r_g(T) state by Horner's rule (deg r_g < 128 steps).
__global__ void __launch_bounds__(256) tinymt_jump_apply_kernel(const TinyMtLaunch P, const uint32_t* __restrict__ poly)
{
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.ns) return;
    const uint32_t* r = poly + 4 * ((P.first + i) / P.group_size - P.first / P.group_size);
    const TinyMT v = tm_load(P, i);
    TinyMT acc = v;
    acc.s0 = acc.s1 = acc.s2 = acc.s3 = 0;
    const int d = poly_deg(r, 4);
    for (int k = d; k >= 0; --k) {
        tinymt_next_state(acc);
        if ((r[k >> 5] >> (k & 31)) & 1u) {
            acc.s0 ^= v.s0;
            acc.s1 ^= v.s1;
            acc.s2 ^= v.s2;
            acc.s3 ^= v.s3;
        }
    }
    tm_store(P, i, acc);
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

// ------------------------------------------------------------------ TinyMT32 Leap Frog (R19)
// Buffer (u32 words, TmLeapLaunch::buf): [0..2] mat1, mat2, tmat; [4..7] the
// base state after init(params, seed); [8, 520) T^(K-1) (columns of 4 words);
// [520 + 512 b, ...) T^(2^b), b < 128.
constexpr uint32_t kTmBase = 4, kTmSkip = 8, kTmTab = 520;

// One block of 128 threads: T from unit vectors, then 127 squarings.
__global__ void __launch_bounds__(128) tm_leap_tables_kernel(uint32_t* __restrict__ buf)
{
    __shared__ uint4 M[128], N[128];
    const unsigned c = threadIdx.x;
    TinyMT t{0, 0, 0, 0, buf[0], buf[1], buf[2]};
    (c < 32 ? t.s0 : c < 64 ? t.s1 : c < 96 ? t.s2 : t.s3) = 1u << (c & 31);
    tinymt_next_state(t);
    M[c] = make_uint4(t.s0, t.s1, t.s2, t.s3);
    __syncthreads();
    for (int b = 0; b < 128; ++b) {
        reinterpret_cast<uint4*>(buf + kTmTab + 512 * b)[c] = M[c];
        if (b == 127) break;
        const uint4 x = M[c];
        const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
        uint4 y = make_uint4(0, 0, 0, 0);
        for (int k = 0; k < 128; ++k)
            if ((xs[k >> 5] >> (k & 31)) & 1u) {
                const uint4 col = M[k];
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

// One block of 128 threads: the skip matrix T^e (e = K - 1) as a product of
// table entries (column c of A*R = A applied to column c of R), and the base
// state init(params, seed).
__global__ void __launch_bounds__(128) tm_leap_skip_kernel(uint32_t* __restrict__ buf, uint64_t e, uint32_t seed)
{
    __shared__ uint4 R[128];
    const unsigned c = threadIdx.x;
    R[c] = make_uint4(c < 32 ? 1u << c : 0u, c >= 32 && c < 64 ? 1u << (c - 32) : 0u,
                      c >= 64 && c < 96 ? 1u << (c - 64) : 0u, c >= 96 ? 1u << (c - 96) : 0u);
    __syncthreads();
    for (int b = 0; b < 64; ++b) {
        if (!((e >> b) & 1u)) continue;
        TinyMT t{R[c].x, R[c].y, R[c].z, R[c].w, 0, 0, 0};
        gf2_apply(buf + kTmTab + 512 * b, t);
        __syncthreads();
        R[c] = make_uint4(t.s0, t.s1, t.s2, t.s3);
        __syncthreads();
    }
    reinterpret_cast<uint4*>(buf + kTmSkip)[c] = R[c];
    if (c == 0) {
        TinyMT t;
        tinymt_init(t, buf[0], buf[1], buf[2], seed);
        buf[kTmBase] = t.s0;
        buf[kTmBase + 1] = t.s1;
        buf[kTmBase + 2] = t.s2;
        buf[kTmBase + 3] = t.s3;
    }
}

// Player first + i, segment j: the base state after
// d = first + i + K*(o + j*seg_draws) draws (per-bit tables), then each draw
// serves the next base draw and skips K - 1.
struct TmLeapCursor {
    TinyMT t;
    __device__ __forceinline__ void init(const TmLeapLaunch& P, uint64_t i, uint64_t j)
    {
        const uint32_t* b = P.buf;
        t = TinyMT{b[kTmBase], b[kTmBase + 1], b[kTmBase + 2], b[kTmBase + 3], b[0], b[1], b[2]};
        const u128 d = (u128)(P.first + i) +
                       (u128)P.players * ((((u128)P.o_hi << 64) | P.o_lo) + (u128)j * P.seg_draws);
        for (int k = 0; k < 128; ++k)
            if ((uint64_t)(d >> k) & 1u) gf2_apply(b + kTmTab + 512 * k, t);
    }
    __device__ __forceinline__ uint32_t next(const TmLeapLaunch& P)
    {
        const uint32_t w = tinymt_next(t);
        if (P.players - 1 > 64) {
            gf2_apply(P.buf + kTmSkip, t);
        } else {
            for (uint64_t k = 1; k < P.players; ++k) tinymt_next_state(t);
        }
        return w;
    }
};

template <int KIND>
__global__ void __launch_bounds__(256) tm_leap_fill_kernel(const __grid_constant__ TmLeapLaunch P)
{
    using T = OutT<KIND>;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t it = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; it < P.items; it += nthr) {
        const uint64_t j = it / P.ns, i = it - j * P.ns;
        const uint64_t c0 = j * P.seg_len, len = min(P.seg_len, P.n - c0);
        TmLeapCursor cur;
        cur.init(P, i, j);
        T* o = reinterpret_cast<T*>(P.out) + i * P.n + c0;
        for (uint64_t k = 0; k < len; ++k) {
            const uint32_t w = cur.next(P);
            if (KIND == kU32) o[k] = (T)w;
            else if (KIND == kF32) o[k] = (T)to_f32(w);
            else o[k] = (T)philox_f64(w, cur.next(P));  // two player draws per double (R7)
        }
    }
}

__global__ void __launch_bounds__(256) tm_leap_mc_kernel(const __grid_constant__ TmLeapLaunch P)
{
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    uint64_t total = 0;
    for (uint64_t it = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; it < P.items; it += nthr) {
        const uint64_t j = it / P.ns, i = it - j * P.ns;
        const uint64_t len = min(P.seg_len, P.n - j * P.seg_len);
        TmLeapCursor cur;
        cur.init(P, i, j);
        uint32_t h = 0;
        for (uint64_t k = 0; k < len; ++k) {
            const uint32_t w0 = cur.next(P);
            h += hit(w0, cur.next(P));
        }
        total += h;
        if (P.counts) atomicAdd(P.counts + i, (unsigned long long)h);
    }
    block_reduce_add(total, P.hits);
}

// Transposed TinyMT32 Leap Frog fill (as leap_mrg_tr_kernel, kernels_leapfrog.cu):
// out[p][t] = base draw (first + p) + K*(o + t) is the transpose of the base
// sequence laid out as rows of K draws, so a lane (one t-row) steps through
// consecutive base draws — consecutive players — with one TinyMT32 step per
// value, after one GF(2) jump to its start (per-bit tables T^(2^b)). Draw
// (p, t) is word t of box row p; each 128-player box leaves by TMA.
constexpr unsigned kTmTrWarps = 4;
#ifndef SHV_TM_LEAP_UNROLL
#define SHV_TM_LEAP_UNROLL 1  // 8-value groups per iteration of the transposed fill's box loop
#endif
constexpr int kTmLeapUnroll = SHV_TM_LEAP_UNROLL;
template <int KIND>
__global__ void __launch_bounds__(kTmTrWarps * 32)
    tm_leap_tr_kernel(const __grid_constant__ TmLeapLaunch P, const __grid_constant__ CUtensorMap tmap)
{
    extern __shared__ uint8_t tm_tr_buf[];
    const unsigned lane = threadIdx.x & 31, warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
    const uint32_t base = ((uint32_t)__cvta_generic_to_shared(tm_tr_buf) + 1023u) & ~1023u;
    const uint32_t box = base + warp * (kTmTrRows * 128u);
    uint32_t off[8];
#pragma unroll
    for (uint32_t k = 0; k < 8; ++k) off[k] = ((((lane >> 2) ^ k)) << 4) + (lane & 3u) * 4u;
    const uint32_t* b = P.buf;
    const uint64_t items = P.tr_tb * P.tr_ps;
    const uint64_t wstride = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t it = (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp; it < items; it += wstride) {
        const uint64_t ps = it / P.tr_tb, tb = it - ps * P.tr_tb;
        const uint64_t t = 32 * tb + lane;
        const uint64_t p0 = ps * P.tr_pl, p1 = min(P.ns, p0 + P.tr_pl);
        TinyMT g{b[kTmBase], b[kTmBase + 1], b[kTmBase + 2], b[kTmBase + 3], b[0], b[1], b[2]};
        const u128 d = (u128)(P.first + p0) + (u128)P.players * ((((u128)P.o_hi << 64) | P.o_lo) + t);
        for (int k = 0; k < 128; ++k)
            if ((uint64_t)(d >> k) & 1u) gf2_apply(b + kTmTab + 512 * k, g);
        for (uint64_t pc = p0; pc < p1; pc += kTmTrRows) {
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
#pragma unroll kTmLeapUnroll
            for (uint32_t q8 = 0; q8 < kTmTrRows; q8 += 8) {
                const uint32_t rb = box + q8 * 128u;
#pragma unroll
                for (uint32_t k = 0; k < 8; ++k) {
                    const uint32_t z = tinymt_next(g);
                    const uint32_t w = KIND == kF32 ? __float_as_uint(to_f32(z)) : z;
                    asm volatile("st.shared.b32 [%0], %1;" ::"r"(rb + k * 128u + off[k]), "r"(w) : "memory");
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tmap),
                             "r"(box), "r"((int)(32 * tb)), "r"((int)pc)
                             : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

constexpr size_t tm_tr_smem() { return (size_t)kTmTrWarps * kTmTrRows * 128 + 1024; }

template <int KIND>
cudaError_t tm_tr_attr()
{
    static std::atomic<uint64_t> done{0};
    return ensure_dyn_smem(tm_leap_tr_kernel<KIND>, tm_tr_smem(), done);
}

template <int KIND>
cudaError_t ensure_tm_smem()
{
    static std::atomic<uint64_t> done{0};
    return ensure_dyn_smem(tinymt_fill_vec_kernel<KIND>, staged_smem<kTmRB>(256), done);
}

template <int KIND>
cudaError_t launch_tm_vec(const TinyMtLaunch& p, Grid g, cudaStream_t s)
{
    const cudaError_t e = ensure_tm_smem<KIND>();
    if (e != cudaSuccess) return e;
    tinymt_fill_vec_kernel<KIND><<<g.blocks, g.threads, staged_smem<kTmRB>((int)g.threads), s>>>(p);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_tm_leap_tr(const TmLeapLaunch& p, const CUtensorMap& tmap, int kind, unsigned blocks, cudaStream_t s)
{
    cudaError_t e = kind == kF32 ? tm_tr_attr<kF32>() : tm_tr_attr<kU32>();
    if (e != cudaSuccess) return e;
    if (kind == kF32) tm_leap_tr_kernel<kF32><<<blocks, kTmTrWarps * 32, tm_tr_smem(), s>>>(p, tmap);
    else tm_leap_tr_kernel<kU32><<<blocks, kTmTrWarps * 32, tm_tr_smem(), s>>>(p, tmap);
    return cudaGetLastError();
}

cudaError_t tm_leap_tr_blocks_per_sm(int kind, int* out)
{
    cudaError_t e = kind == kF32 ? tm_tr_attr<kF32>() : tm_tr_attr<kU32>();
    if (e != cudaSuccess) return e;
    return kind == kF32 ? occ(tm_leap_tr_kernel<kF32>, kTmTrWarps * 32, tm_tr_smem(), out)
                        : occ(tm_leap_tr_kernel<kU32>, kTmTrWarps * 32, tm_tr_smem(), out);
}

cudaError_t launch_tm_leap_prep(uint32_t* buf, uint64_t players, uint32_t seed, cudaStream_t s)
{
    tm_leap_tables_kernel<<<1, 128, 0, s>>>(buf);
    tm_leap_skip_kernel<<<1, 128, 0, s>>>(buf, players - 1, seed);
    return cudaGetLastError();
}

cudaError_t launch_tm_leap(const TmLeapLaunch& p, int mode, Grid g, cudaStream_t s)
{
    if (mode == kU32) tm_leap_fill_kernel<kU32><<<g.blocks, g.threads, 0, s>>>(p);
    else if (mode == kF32) tm_leap_fill_kernel<kF32><<<g.blocks, g.threads, 0, s>>>(p);
    else if (mode == kF64) tm_leap_fill_kernel<kF64><<<g.blocks, g.threads, 0, s>>>(p);
    else tm_leap_mc_kernel<<<g.blocks, g.threads, 0, s>>>(p);
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

cudaError_t launch_tinymt_jump(const TinyMtLaunch& p, uint64_t n, uint32_t* d_poly, cudaStream_t s)
{
    const uint64_t ngroups = (p.first + p.ns - 1) / p.group_size - p.first / p.group_size + 1;
    tinymt_jump_poly_kernel<<<(unsigned)((ngroups + 63) / 64), 64, 0, s>>>(p, ngroups, n, d_poly);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    tinymt_jump_apply_kernel<<<(unsigned)((p.ns + 255) / 256), 256, 0, s>>>(p, d_poly);
    return cudaGetLastError();
}

cudaError_t launch_tinymt_mc(const TinyMtLaunch& p, Grid g, cudaStream_t s)
{
    tinymt_mc_kernel<<<g.blocks, g.threads, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t tinymt_occupancy(int kernel, int kind, bool fast, int threads, int* out)
{
    (void)fast;
    switch (kernel) {
    case kKTinyFill: {
        const cudaError_t e = kind == kU32 ? ensure_tm_smem<kU32>()
                            : kind == kF32 ? ensure_tm_smem<kF32>() : ensure_tm_smem<kF64>();
        if (e != cudaSuccess) return e;
        const size_t sm = staged_smem<kTmRB>(threads);
        if (kind == kU32) return occ(tinymt_fill_vec_kernel<kU32>, threads, sm, out);
        if (kind == kF32) return occ(tinymt_fill_vec_kernel<kF32>, threads, sm, out);
        return occ(tinymt_fill_vec_kernel<kF64>, threads, sm, out);
    }
    case kKTinyMc:
        return occ(tinymt_mc_kernel, threads, 0, out);
    }
    return cudaErrorInvalidValue;
}

}  // namespace shv
