// kernels_leapfrog.cu — Leap Frog partition kernels (NEXT-4; P L118-122
// [§2.3]: one base sequence "dealt" round-robin to K players; R17): bulk fills
// (u32 / f32 / f64) and the fused Monte Carlo pi kernel for MRG32k3a,
// Philox4x32-10 and Threefry4x64-20 handles.
//
// Player p's draw t is base draw p + K*t. Counter-based generators compute it
// directly (one block per draw; a cached block serves K < words-per-block);
// Philox with K % 4 == 0 evaluates each block once for the four players that
// share it (leap_fill_grouped_kernel).
// MRG32k3a cannot skip K-1 draws for free, so each component of the player's
// subsequence is stepped by the order-3 linear recurrence that the
// characteristic polynomial of B = A^K gives (Cayley-Hamilton: B^3 = tr(B) B^2
// - M2(B) B + det(B) I, so u_{t+3} = tr u_{t+2} - M2 u_{t+1} + det u_t for any
// linear functional u_t of B^t w): 3 modular products per component and draw,
// independent of K. The host builds the coefficients, B, and
// the segment start jumps.
#include "kernels_common.cuh"

#ifndef SHV_LEAP_MRG_UNROLL
#define SHV_LEAP_MRG_UNROLL 4  // 8-value groups per box unrolled in the transposed MRG32k3a fill (4: 3.28 vs 3.49 ms, lab61)
#endif
constexpr int kLeapMrgUnroll = SHV_LEAP_MRG_UNROLL;
// the same for the counter-based transposed fills (lab62): Philox 1 (3.16 vs
// 3.53-3.64 ms unrolled), Threefry 4 (6.00 vs 6.20 ms)
#ifndef SHV_LEAP_PHILOX_COLS
#define SHV_LEAP_PHILOX_COLS 1  // t-columns per lane of the transposed Philox fill (2: 256-B box rows)
#endif
__host__ __device__ constexpr uint32_t leap_ctr_cols_of(int lgen) { return lgen == 1 ? SHV_LEAP_PHILOX_COLS : 1; }
#ifndef SHV_LEAP_PHILOX_UNROLL
#define SHV_LEAP_PHILOX_UNROLL 1
#endif
#ifndef SHV_LEAP_THREEFRY_UNROLL
#define SHV_LEAP_THREEFRY_UNROLL 4
#endif

namespace shv {
namespace {

// (c0 u0 + c1 u1 + c2 u2) mod (2^32 - C), all operands < 2^32 - C. The three
// 64-bit products are summed with carries (s = cy*2^64 + s2), then folded with
// 2^32 = C and 2^64 = C^2: x < 2^46.6, one more fold gives < 2m.
template <uint32_t C>
__device__ __forceinline__ uint32_t dot3(uint32_t c0, uint32_t u0, uint32_t c1, uint32_t u1, uint32_t c2,
                                         uint32_t u2)
{
    const uint64_t p0 = (uint64_t)c0 * u0, p1 = (uint64_t)c1 * u1, p2 = (uint64_t)c2 * u2;
    const uint64_t s = p0 + p1;
    const uint64_t s2 = s + p2;
    const uint32_t cy = (uint32_t)(s < p0) + (uint32_t)(s2 < s);
    uint64_t x = (s2 >> 32) * C + (uint32_t)s2 + (uint64_t)cy * ((uint64_t)C * C);
    x = (x >> 32) * C + (uint32_t)x;
    const uint64_t m = (1ull << 32) - C;
    return (uint32_t)(x >= m ? x - m : x);
}

using u128 = unsigned __int128;

template <int G>
struct LeapCursor;

// MRG32k3a player: (x0, x1, x2) = newest component-1 words of the states at
// player draws t, t+1, t+2 (likewise y for component 2); draw t is their
// combination (R2).
template <>
struct LeapCursor<kLeapMrg> {
    uint32_t x0, x1, x2, y0, y1, y2;

    __device__ __forceinline__ void init(const LeapLaunch& P, uint64_t i, uint64_t j)
    {
        const uint32_t* st = P.state;
        const uint64_t n = P.stride, q = P.stream_begin + i;
        Mrg s{__ldg(st + q), __ldg(st + n + q), __ldg(st + 2 * n + q),
              __ldg(st + 3 * n + q), __ldg(st + 4 * n + q), __ldg(st + 5 * n + q)};
        apply(P.start.a, P.start.b, s);  // A^(1 + K*o) A^p seed: state of player draw o
        for (int b = 0; j; ++b, j >>= 1)  // segment j starts j*seg_draws player draws later
            if (j & 1) apply(P.segpow[b].a, P.segpow[b].b, s);
        x0 = s.x2;
        y0 = s.y2;
        apply(P.B.a, P.B.b, s);
        x1 = s.x2;
        y1 = s.y2;
        apply(P.B.a, P.B.b, s);
        x2 = s.x2;
        y2 = s.y2;
    }

    __device__ __forceinline__ uint32_t next(const LeapLaunch& P)
    {
        const uint32_t z = mrg_combine(x0, y0);
        const uint32_t nx = dot3<kC1>(P.cp1[0], x0, P.cp1[1], x1, P.cp1[2], x2);
        const uint32_t ny = dot3<kC2>(P.cp2[0], y0, P.cp2[1], y1, P.cp2[2], y2);
        x0 = x1;
        x1 = x2;
        x2 = nx;
        y0 = y1;
        y1 = y2;
        y2 = ny;
        return z;
    }
};

// Counter-based player: next base draw index d (u128), advanced by K.
template <>
struct LeapCursor<kLeapPhilox> {
    u128 d;
    uint64_t cb;
    bool valid;
    W4 v;

    __device__ __forceinline__ void init(const LeapLaunch& P, uint64_t i, uint64_t j)
    {
        const u128 o = ((u128)P.o_hi << 64) | P.o_lo;
        d = (u128)(P.first + i) + (u128)P.players * (o + (u128)j * P.seg_draws);
        valid = false;
    }

    __device__ __forceinline__ uint32_t next(const LeapLaunch& P)
    {
        const uint64_t b = (uint64_t)(d >> 2);
        if (!valid || b != cb) {
            v = philox_blk(b, 0, (uint32_t)P.k0, (uint32_t)P.k1);
            cb = b;
            valid = true;
        }
        const uint32_t w = (uint32_t)d & 3;
        d += P.players;
        return w == 0 ? v.x : w == 1 ? v.y : w == 2 ? v.z : v.w;
    }
};

template <>
struct LeapCursor<kLeapThreefry> {
    u128 d;
    uint64_t cb;
    bool valid;
    Q4 v;

    __device__ __forceinline__ void init(const LeapLaunch& P, uint64_t i, uint64_t j)
    {
        const u128 o = ((u128)P.o_hi << 64) | P.o_lo;
        d = (u128)(P.first + i) + (u128)P.players * (o + (u128)j * P.seg_draws);
        valid = false;
    }

    __device__ __forceinline__ uint32_t next(const LeapLaunch& P)
    {
        const uint64_t b = (uint64_t)(d >> 3);
        if (!valid || b != cb) {
            v = threefry20(b, 0, P.k0, P.k1);
            cb = b;
            valid = true;
        }
        const uint32_t w = (uint32_t)d & 7;
        d += P.players;
        const uint64_t lane = (w >> 1) == 0 ? v.x : (w >> 1) == 1 ? v.y : (w >> 1) == 2 ? v.z : v.w;
        return (w & 1) ? (uint32_t)(lane >> 32) : (uint32_t)lane;
    }
};

template <int G, int KIND>
__device__ __forceinline__ OutT<KIND> leap_value(LeapCursor<G>& c, const LeapLaunch& P)
{
    const uint32_t w = c.next(P);
    if constexpr (KIND == kU32) return w;
    else if constexpr (KIND == kF32) return to_f32(w);
    else if constexpr (G == kLeapMrg) return mrg_f64(w);
    else return philox_f64(w, c.next(P));  // two player draws per double (R7)
}

// Fill: each thread writes one segment of one row. VEC: 32-byte aligned
// rows and seg_len % 8 == 0, so every 8 values (u32/f32) or 4 (f64) leave as
// one 32-byte store.
template <int G, int KIND, bool VEC>
__global__ void __launch_bounds__(256) leap_fill_kernel(const __grid_constant__ LeapLaunch P)
{
    using T = OutT<KIND>;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t it = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; it < P.items; it += nthr) {
        const uint64_t j = it / P.ns;
        const uint64_t i = it - j * P.ns;
        const uint64_t c0 = j * P.seg_len;
        const uint64_t len = min(P.seg_len, P.n - c0);
        LeapCursor<G> cur;
        cur.init(P, i, j);
        T* o = reinterpret_cast<T*>(P.out) + i * P.n + c0;
        if (VEC) {
            for (uint64_t t = 0; t < len; t += 8) {
                if (KIND == kF64) {
                    const double a = leap_value<G, KIND>(cur, P), b = leap_value<G, KIND>(cur, P),
                                 c = leap_value<G, KIND>(cur, P), d = leap_value<G, KIND>(cur, P);
                    st_v4d(o + t, a, b, c, d);
                    const double e = leap_value<G, KIND>(cur, P), f = leap_value<G, KIND>(cur, P),
                                 g = leap_value<G, KIND>(cur, P), h = leap_value<G, KIND>(cur, P);
                    st_v4d(o + t + 4, e, f, g, h);
                } else {
                    uint32_t v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const T x = leap_value<G, KIND>(cur, P);
                        v[u] = KIND == kF32 ? __float_as_uint((float)x) : (uint32_t)x;
                    }
                    st_v8(o + t, v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7]);
                }
            }
        } else {
            for (uint64_t t = 0; t < len; ++t) o[t] = leap_value<G, KIND>(cur, P);
        }
    }
}

// Fused Monte Carlo: sample k of a player uses its draws 2k, 2k+1 (R9).
template <int G>
__global__ void __launch_bounds__(256) leap_mc_kernel(const __grid_constant__ LeapLaunch P)
{
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    uint64_t total = 0;
    for (uint64_t it = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; it < P.items; it += nthr) {
        const uint64_t j = it / P.ns;
        const uint64_t i = it - j * P.ns;
        const uint64_t k0 = j * P.seg_len;
        const uint32_t len = (uint32_t)min(P.seg_len, P.n - k0);
        LeapCursor<G> cur;
        cur.init(P, i, j);
        uint32_t h = 0;
        for (uint32_t k = 0; k < len; ++k) {
            const uint32_t w0 = cur.next(P);
            h += hit(w0, cur.next(P));
        }
        total += h;
        if (P.counts) atomicAdd(P.counts + i, (unsigned long long)h);
    }
    block_reduce_add(total, P.hits);
}

// Grouped Philox players (K % 4 == 0): players 4G .. 4G+3 read the four words
// of ONE counter block for every draw t (base draw p + K t lies in block
// G + (K/4) t, word p & 3), so a work item (group G, segment j) evaluates each
// block once and serves up to four rows from it — a quarter of the per-value
// block evaluations of the per-player cursor. Rows outside the launch are not
// written (partial groups at the launch edges).
struct LeapGroup {
    uint64_t b, step;      // next block, blocks per player draw (K/4)
    int64_t row0;          // launch row of player 4G (may be < 0)
    __device__ __forceinline__ void init(const LeapLaunch& P, uint64_t g, uint64_t j)
    {
        const uint64_t G = P.g0 + g;
        const u128 o = ((u128)P.o_hi << 64) | P.o_lo;
        step = P.players >> 2;
        b = (uint64_t)((u128)G + (u128)step * (o + (u128)j * P.seg_draws));
        row0 = (int64_t)(4 * G) - (int64_t)P.first;
    }
    __device__ __forceinline__ W4 next(const LeapLaunch& P)
    {
        const W4 v = philox_blk(b, 0, (uint32_t)P.k0, (uint32_t)P.k1);
        b += step;
        return v;
    }
    __device__ __forceinline__ bool live(const LeapLaunch& P, int l) const
    {
        return row0 + l >= 0 && row0 + l < (int64_t)P.ns;
    }
};

__device__ __forceinline__ uint32_t lane_of(const W4& v, int l)
{
    return l == 0 ? v.x : l == 1 ? v.y : l == 2 ? v.z : v.w;
}

template <int KIND, bool VEC>
__global__ void __launch_bounds__(256) leap_fill_grouped_kernel(const __grid_constant__ LeapLaunch P)
{
    using T = OutT<KIND>;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t it = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; it < P.items; it += nthr) {
        const uint64_t j = it / P.ngroups;
        const uint64_t g = it - j * P.ngroups;
        const uint64_t c0 = j * P.seg_len;
        const uint64_t len = min(P.seg_len, P.n - c0);
        LeapGroup cur;
        cur.init(P, g, j);
        T* base = reinterpret_cast<T*>(P.out) + c0;
        if (VEC && KIND != kF64) {
            for (uint64_t t = 0; t < len; t += 8) {
                W4 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = cur.next(P);
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    if (!cur.live(P, l)) continue;
                    uint32_t w[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const uint32_t x = lane_of(v[u], l);
                        w[u] = KIND == kF32 ? __float_as_uint(to_f32(x)) : x;
                    }
                    st_v8(base + (uint64_t)(cur.row0 + l) * P.n + t, w[0], w[1], w[2], w[3], w[4], w[5], w[6], w[7]);
                }
            }
        } else if (VEC) {  // f64: two player draws per value, four values per 32-byte store
            for (uint64_t t = 0; t < len; t += 4) {
                W4 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = cur.next(P);
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    if (!cur.live(P, l)) continue;
                    st_v4d(base + (uint64_t)(cur.row0 + l) * P.n + t,
                           philox_f64(lane_of(v[0], l), lane_of(v[1], l)), philox_f64(lane_of(v[2], l), lane_of(v[3], l)),
                           philox_f64(lane_of(v[4], l), lane_of(v[5], l)), philox_f64(lane_of(v[6], l), lane_of(v[7], l)));
                }
            }
        } else {
            for (uint64_t t = 0; t < len; ++t) {
                const W4 a = cur.next(P);
                W4 b2{};
                if (KIND == kF64) b2 = cur.next(P);
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    if (!cur.live(P, l)) continue;
                    T* o = base + (uint64_t)(cur.row0 + l) * P.n + t;
                    if (KIND == kU32) *o = (T)lane_of(a, l);
                    else if (KIND == kF32) *o = (T)to_f32(lane_of(a, l));
                    else *o = (T)philox_f64(lane_of(a, l), lane_of(b2, l));
                }
            }
        }
    }
}

// Grouped Philox fill with TMA stores (u32/f32; n % 32 == 0). A warp owns a
// tile of 32 consecutive groups = 128 rows x one segment. Each round a lane
// evaluates 32 blocks for its group — 32 values for each of its four rows —
// into the warp's 16-KB shared-memory box (128 rows x 128 B, 128-B swizzle:
// chunk c of box row r at c ^ (r & 7)); at store step s lane L writes row
// 4L + ((s + L) & 3), so the eight chunk slots of a 512-B wavefront group are
// all distinct. One lane then hands the box to the TMA engine. Rows past the
// launch (the last partial group, tiles past the last group) lie outside the
// tensor map and are clipped by it; a first group that starts before the
// launch (first player not 4-aligned) has the warp store its rows itself.
constexpr unsigned kLeapTmaWarps = 4;
template <int KIND>
__global__ void __launch_bounds__(kLeapTmaWarps * 32)
    leap_fill_tma_kernel(const __grid_constant__ LeapLaunch P, const __grid_constant__ CUtensorMap tmap)
{
    extern __shared__ uint8_t leap_smem[];
    const unsigned lane = threadIdx.x & 31, warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
    const uint32_t base = ((uint32_t)__cvta_generic_to_shared(leap_smem) + 1023u) & ~1023u;
    const uint32_t box = base + warp * 16384u;
    const uint64_t nseg = P.items / P.ngroups;
    const uint64_t T = (P.ngroups + 31) / 32, ntiles = T * nseg;
    const uint64_t wstride = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t tile = (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp; tile < ntiles; tile += wstride) {
        const uint64_t j = tile / T, gt = tile - j * T;
        LeapGroup cur;
        cur.init(P, 32 * gt + lane, j);
        const int64_t row_base = (int64_t)(4 * (P.g0 + 32 * gt)) - (int64_t)P.first;
        const uint64_t c0 = j * P.seg_len;
        const uint32_t len = (uint32_t)min(P.seg_len, P.n - c0);  // multiple of 32
        for (uint32_t r = 0; r < len; r += 32) {
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
#pragma unroll 2
            for (uint32_t c = 0; c < 8; ++c) {
                const W4 v0 = cur.next(P), v1 = cur.next(P), v2 = cur.next(P), v3 = cur.next(P);
#pragma unroll
                for (uint32_t st = 0; st < 4; ++st) {
                    const int l = (int)((st + lane) & 3);
                    const uint32_t row = 4 * lane + l;
                    const uint32_t addr = box + row * 128u + ((c ^ (row & 7u)) << 4);
                    uint32_t a = lane_of(v0, l), b = lane_of(v1, l), d = lane_of(v2, l), e = lane_of(v3, l);
                    if (KIND == kF32) {
                        a = __float_as_uint(to_f32(a));
                        b = __float_as_uint(to_f32(b));
                        d = __float_as_uint(to_f32(d));
                        e = __float_as_uint(to_f32(e));
                    }
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(d), "r"(e)
                                 : "memory");
                }
            }
            if (row_base < 0) {
                // first tile of a launch whose first player is not 4-aligned: the
                // TMA engine rejects negative box coordinates, so the warp copies
                // the box's live rows itself (lane = word of the row)
                __syncwarp();
                for (uint32_t rr = 0; rr < 128; ++rr) {
                    const int64_t trow = row_base + rr;
                    if (trow < 0 || trow >= (int64_t)P.ns) continue;
                    uint32_t w;
                    asm volatile("ld.shared.b32 %0, [%1];"
                                 : "=r"(w)
                                 : "r"(box + rr * 128u + ((((lane >> 2) ^ (rr & 7u))) << 4) + (lane & 3u) * 4u)
                                 : "memory");
                    reinterpret_cast<uint32_t*>(P.out)[(uint64_t)trow * P.n + c0 + r + lane] = w;
                }
                __syncwarp();
                continue;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tmap),
                             "r"(box), "r"((int)(c0 + r)), "r"((int)row_base)
                             : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

constexpr size_t leap_tma_smem() { return (size_t)kLeapTmaWarps * 16384 + 1024; }

template <int KIND>
cudaError_t leap_tma_attr()
{
    static std::atomic<uint64_t> done{0};
    return ensure_dyn_smem(leap_fill_tma_kernel<KIND>, leap_tma_smem(), done);
}

// MRG32k3a Leap Frog by transposition (u32/f32). out[p][t] = base draw
// (first + p) + K*(o + t): the output is the TRANSPOSE of the base sequence
// laid out as rows of K consecutive draws. A warp owns 32 consecutive t (lane
// = t) and a segment of tr_pl players; each lane runs the FP64 MRG step
// through consecutive base draws (players p, p+1, ...) of its t-row, starting
// from A^(p_begin + K*t) * tr_s0 (per-bit tables: one jump per lane per
// segment), and writes draw (p, t) as word t of box row p: all 32 lanes write
// distinct words of one 128-B row (conflict-free, unswizzled box). Each
// kTrRows-player box (kTrRows rows x 32 values) leaves by TMA; rows past the launch
// and columns past n are clipped by the tensor map. Per value: the MRG step
// (MrgIF) and one shared store, against three modular products per component
// for the per-player recurrence.
#ifndef SHV_LEAP_TR_WARPS
#define SHV_LEAP_TR_WARPS 4
#endif
constexpr unsigned kTrWarps = SHV_LEAP_TR_WARPS;
// warps per block of the transposed MRG32k3a fill (8: 3.22 vs 3.28 ms with 4-warp grid sizing, lab64; 3.34-3.43 with 8-warp sizing)
#ifndef SHV_LEAP_MRG_WARPS
#define SHV_LEAP_MRG_WARPS 4
#endif
constexpr unsigned kTrWarpsMrg = SHV_LEAP_MRG_WARPS;
// Players per transposed box (rows of the 128-B wide box): 32 keeps a warp's
// box at 4 KB, so up to 48 warps per SM stay resident (128-row, 16-KB boxes
// held the transposed fills to 12 warps per SM: ncu 0.74 eligible warps per
// scheduler, issue 51 %).
#ifndef SHV_LEAP_TR_ROWS
#define SHV_LEAP_TR_ROWS 32
#endif
constexpr uint32_t kTrRows = SHV_LEAP_TR_ROWS;
#ifndef SHV_LEAP_CKMASK
#define SHV_LEAP_CKMASK 22  // no three-register-pair DFMA: 4.21 -> 3.99 ms at the C5 shape (tools/lab)
#endif
// FP64 step constants from constant memory (bit i of SHV_LEAP_CKMASK) or the
// launch parameters, as in kernels_mrg.cu (operand placement).
__constant__ double c_leap_fpk[6] = {6755399441055744.0, 1.0 / 4294967087.0, 0x1.000059451f212p-32,
                                     4294967087.0, 4294944443.0, 5886603609186927.0};
// MrgSN constants (MrgFpK::sn_* order) from constant memory: the DFMA.RM
// multiplicands become uniform-register operands (kernels_mrg.cu, lab50).
__constant__ double c_leap_snk[5] = {0x0.317b9fd79a126p-1022, 0x1.4e9d5b50f226fp-1022, 0x1.000000d10000bp+980,
                                     0x1.000059451f212p+978, 0x1.8p-12};
#ifndef SHV_LEAP_STEP
#define SHV_LEAP_STEP 3  // step of the transposed MRG32k3a Leap Frog fill: 3 = MrgIF, 5 = MrgSN (3.69 vs 3.48 ms, lab51)
#endif
using LeapMrgGen = std::conditional<SHV_LEAP_STEP == 5, MrgSN,
                                    std::conditional<SHV_LEAP_STEP == 7, MrgMF, MrgIF>::type>::type;
__device__ __forceinline__ void make_leap_gen(const Mrg& m, MrgSN& g) { g = to_mrg_sn(m); }
__device__ __forceinline__ void make_leap_gen(const Mrg& m, MrgMF& g) { g = to_mrg_mf(m); }
__device__ __forceinline__ void make_leap_gen(const Mrg& m, MrgIF& g) { g = to_mrg_if(m); }
template <int KIND>
__global__ void __launch_bounds__(kTrWarpsMrg * 32)
    leap_mrg_tr_kernel(const __grid_constant__ LeapLaunch P, const __grid_constant__ CUtensorMap tmap)
{
    extern __shared__ uint8_t tr_smem[];
    const unsigned lane = threadIdx.x & 31, warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
    const uint32_t base = ((uint32_t)__cvta_generic_to_shared(tr_smem) + 1023u) & ~1023u;
    const uint32_t box = base + warp * (kTrRows * 128u);
#define SHV_TRF(i) (((SHV_LEAP_CKMASK >> (i)) & 1) ? c_leap_fpk[i] : P.fpk[i])
    MrgFpK K{SHV_TRF(0), SHV_TRF(1), SHV_TRF(2), SHV_TRF(3), SHV_TRF(4), SHV_TRF(5), P.imul[0], P.imul[1]};
#undef SHV_TRF
    K.sn_c1q = c_leap_snk[0];
    K.sn_c2p = c_leap_snk[1];
    K.sn_c1s = c_leap_snk[2];
    K.sn_c2s = c_leap_snk[3];
    K.sn_M = c_leap_snk[4];
    const uint32_t lo4 = lane * 4u;  // unswizzled box: word `lane` of each 128-B row
    const uint64_t items = P.tr_tb * P.tr_ps;
    const uint64_t wstride = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t it = (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp; it < items; it += wstride) {
        const uint64_t ps = it / P.tr_tb, tb = it - ps * P.tr_tb;
        const uint64_t t = 32 * tb + lane;
        const uint64_t p0 = ps * P.tr_pl;
        const uint64_t p1 = min(P.ns, p0 + P.tr_pl);
        Mrg m{P.tr_s0[0], P.tr_s0[1], P.tr_s0[2], P.tr_s0[3], P.tr_s0[4], P.tr_s0[5]};
        for (uint64_t b = 0, x = t; x; ++b, x >>= 1)
            if (x & 1) apply(P.segpow[b].a, P.segpow[b].b, m);
        for (uint64_t b = 0, x = ps; x; ++b, x >>= 1)
            if (x & 1) apply(P.tr_ppow[b].a, P.tr_ppow[b].b, m);
        LeapMrgGen g;
        make_leap_gen(m, g);
        for (uint64_t pc = p0; pc < p1; pc += kTrRows) {
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
#pragma unroll kLeapMrgUnroll
            for (uint32_t q8 = 0; q8 < kTrRows; q8 += 8) {
                const uint32_t rb = box + q8 * 128u;
#pragma unroll
                for (uint32_t k = 0; k < 8; ++k) {
                    const uint32_t z = mrg_next(g, K);
                    const uint32_t w = KIND == kF32 ? __float_as_uint(to_f32(z)) : z;
                    asm volatile("st.shared.b32 [%0], %1;" ::"r"(rb + lo4 + k * 128u), "r"(w) : "memory");
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

// One player segment [p0, p1) of a lane's t-row, in kTrRows-player boxes.
// HOIST (Philox, the low counter word does not wrap within the run): round 1
// is hoisted (M0*b_lo by addition, M0*c0' constant; counter words 2, 3 = 0).
// A separate instantiation per HOIST keeps ptxas from merging the two round
// bodies into one with selects (18 extra adds per block measured in SASS).
#ifndef SHV_LEAP_NOSTORE
#define SHV_LEAP_NOSTORE 0  // lab knob: compute only (profiles/r02_labs/lab23: 3.03 of 3.38 ms)
#endif
template <int KIND, int G, bool HOIST>
__device__ __forceinline__ void leap_ctr_run(const LeapLaunch& P, const CUtensorMap* tmap, unsigned lane, uint32_t box,
                                             uint32_t lo4, uint64_t tb, uint64_t p0, uint64_t p1, uint64_t b,
                                             uint64_t b2)
{
    constexpr int kUnroll = G == kLeapPhilox ? SHV_LEAP_PHILOX_UNROLL : SHV_LEAP_THREEFRY_UNROLL;
    constexpr uint32_t kCols = leap_ctr_cols_of(G), kRowB = 128u * kCols;
    const uint64_t q = (uint64_t)kPM0 * ((uint32_t)(b >> 32) ^ (uint32_t)P.k0);
    uint64_t pa = (uint64_t)kPM0 * (uint32_t)b;
    const uint64_t q2 = (uint64_t)kPM0 * ((uint32_t)(b2 >> 32) ^ (uint32_t)P.k0);
    uint64_t pa2 = (uint64_t)kPM0 * (uint32_t)b2;
    for (uint64_t pc = p0; pc < p1; pc += kTrRows) {
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
#pragma unroll kUnroll
        for (uint32_t q8 = 0; q8 < kTrRows; q8 += 8) {
            const uint32_t rb = box + q8 * kRowB;
            if constexpr (kCols == 2) {  // second column t + 32 (Philox only): word 32 + lane of the 256-B row
                uint32_t y[8];
                W4 u0, u1;
                if constexpr (HOIST) {
                    u0 = philox10_from_r2(pa2, q2, 0u, 0u, (uint32_t)P.k0, (uint32_t)P.k1);
                    pa2 = add64w(pa2, kPM0);
                    u1 = philox10_from_r2(pa2, q2, 0u, 0u, (uint32_t)P.k0, (uint32_t)P.k1);
                    pa2 = add64w(pa2, kPM0);
                } else {
                    u0 = philox_blk(b2, 0, (uint32_t)P.k0, (uint32_t)P.k1);
                    u1 = philox_blk(b2 + 1, 0, (uint32_t)P.k0, (uint32_t)P.k1);
                }
                b2 += 2;
                y[0] = u0.x; y[1] = u0.y; y[2] = u0.z; y[3] = u0.w;
                y[4] = u1.x; y[5] = u1.y; y[6] = u1.z; y[7] = u1.w;
#pragma unroll
                for (uint32_t k = 0; k < 8; ++k) {
                    const uint32_t w = KIND == kF32 ? __float_as_uint(to_f32(y[k])) : y[k];
                    asm volatile("st.shared.b32 [%0], %1;" ::"r"(rb + 128u + lo4 + k * kRowB), "r"(w) : "memory");
                }
            }
            uint32_t z[8];
            if constexpr (G == kLeapPhilox) {
                W4 v0, v1;
                if constexpr (HOIST) {
                    v0 = philox10_from_r2(pa, q, 0u, 0u, (uint32_t)P.k0, (uint32_t)P.k1);
                    pa = add64w(pa, kPM0);
                    v1 = philox10_from_r2(pa, q, 0u, 0u, (uint32_t)P.k0, (uint32_t)P.k1);
                    pa = add64w(pa, kPM0);
                } else {
                    v0 = philox_blk(b, 0, (uint32_t)P.k0, (uint32_t)P.k1);
                    v1 = philox_blk(b + 1, 0, (uint32_t)P.k0, (uint32_t)P.k1);
                }
                b += 2;
                z[0] = v0.x; z[1] = v0.y; z[2] = v0.z; z[3] = v0.w;
                z[4] = v1.x; z[5] = v1.y; z[6] = v1.z; z[7] = v1.w;
            } else {  // Threefry4x64-20: words (lo, hi) of lanes 0..3 (R16)
                const Q4 v = threefry20(b, 0, P.k0, P.k1);
                b += 1;
                z[0] = (uint32_t)v.x; z[1] = (uint32_t)(v.x >> 32); z[2] = (uint32_t)v.y; z[3] = (uint32_t)(v.y >> 32);
                z[4] = (uint32_t)v.z; z[5] = (uint32_t)(v.z >> 32); z[6] = (uint32_t)v.w; z[7] = (uint32_t)(v.w >> 32);
            }
#if SHV_LEAP_NOSTORE  // lab knob: compute only (the store path's share of the time)
            uint32_t x = 0;
#pragma unroll
            for (uint32_t k = 0; k < 8; ++k) x ^= z[k];
            if (x == 0x9E3779B9u) asm volatile("st.shared.b32 [%0], %1;" ::"r"(rb), "r"(x) : "memory");
        }
    }
#else
#pragma unroll
            for (uint32_t k = 0; k < 8; ++k) {
                const uint32_t w = KIND == kF32 ? __float_as_uint(to_f32(z[k])) : z[k];
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(rb + lo4 + k * kRowB), "r"(w) : "memory");
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tmap),
                         "r"(box), "r"((int)(32 * kCols * tb)), "r"((int)pc)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
#endif
}

// Counter-based Leap Frog by the same transposition (Philox: K % 4 == 0 and
// first % 4 == 0; Threefry: K % 8 == 0 and first % 8 == 0): a lane's
// consecutive base draws are consecutive words of consecutive counter blocks
// of stream 0, so one block serves 4 (Philox) or 8 (Threefry) players of the
// lane's t-row (the per-player kernels evaluate one block per value).
template <int KIND, int G>
__global__ void __launch_bounds__(kTrWarps * 32)
    leap_ctr_tr_kernel(const __grid_constant__ LeapLaunch P, const __grid_constant__ CUtensorMap tmap)
{
    extern __shared__ uint8_t trp_smem[];
    const unsigned lane = threadIdx.x & 31, warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
    const uint32_t base = ((uint32_t)__cvta_generic_to_shared(trp_smem) + 1023u) & ~1023u;
    constexpr uint32_t kCols = leap_ctr_cols_of(G);
    const uint32_t box = base + warp * (kTrRows * 128u * kCols);
    const uint32_t lo4 = lane * 4u;  // unswizzled box: word `lane` (and 32 + lane) of each row
    const uint64_t items = P.tr_tb * P.tr_ps;
    const uint64_t wstride = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const u128 o = ((u128)P.o_hi << 64) | P.o_lo;
    for (uint64_t it = (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp; it < items; it += wstride) {
        const uint64_t ps = it / P.tr_tb, tb = it - ps * P.tr_tb;
        const uint64_t t = 32 * kCols * tb + lane;
        const uint64_t p0 = ps * P.tr_pl;
        const uint64_t p1 = min(P.ns, p0 + P.tr_pl);
        // words per block: 4 (Philox) or 8 (Threefry); the run starts block-aligned
        const uint64_t b = (uint64_t)(((u128)(P.first + p0) + (u128)P.players * (o + t)) >> (G == kLeapPhilox ? 2 : 3));
        const uint64_t b2 =
            kCols == 2 ? (uint64_t)(((u128)(P.first + p0) + (u128)P.players * (o + t + 32)) >> 2) : 0;
        const uint64_t nblk = (p1 - p0 + 3) / 4 + 2;
        const uint32_t lim = 0xFFFFFFFFu - (uint32_t)min(nblk, (uint64_t)0xFFFFFFFFu);
        const bool hoist = G == kLeapPhilox && (uint32_t)b <= lim && (kCols == 1 || (uint32_t)b2 <= lim);
        if (__all_sync(0xffffffffu, hoist))
            leap_ctr_run<KIND, G, G == kLeapPhilox>(P, &tmap, lane, box, lo4, tb, p0, p1, b, b2);
        else leap_ctr_run<KIND, G, false>(P, &tmap, lane, box, lo4, tb, p0, p1, b, b2);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

constexpr size_t leap_tr_smem(uint32_t cols = 1) { return (size_t)kTrWarps * kTrRows * 128 * cols + 1024; }
constexpr size_t leap_tr_smem_mrg() { return (size_t)kTrWarpsMrg * kTrRows * 128 + 1024; }

template <int KIND, int G>
cudaError_t leap_trp_attr()
{
    static std::atomic<uint64_t> done{0};
    return ensure_dyn_smem(leap_ctr_tr_kernel<KIND, G>, leap_tr_smem(leap_ctr_cols_of(G)), done);
}

template <int KIND>
cudaError_t leap_tr_attr()
{
    static std::atomic<uint64_t> done{0};
    return ensure_dyn_smem(leap_mrg_tr_kernel<KIND>, leap_tr_smem_mrg(), done);
}

__global__ void __launch_bounds__(256) leap_mc_grouped_kernel(const __grid_constant__ LeapLaunch P)
{
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    uint64_t total = 0;
    for (uint64_t it = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; it < P.items; it += nthr) {
        const uint64_t j = it / P.ngroups;
        const uint64_t g = it - j * P.ngroups;
        const uint32_t len = (uint32_t)min(P.seg_len, P.n - j * P.seg_len);
        LeapGroup cur;
        cur.init(P, g, j);
        uint32_t h[4] = {0, 0, 0, 0};
        for (uint32_t k = 0; k < len; ++k) {
            const W4 a = cur.next(P), b = cur.next(P);
            h[0] += hit_fp64(a.x, b.x);
            h[1] += hit_fp64(a.y, b.y);
            h[2] += hit_fp64(a.z, b.z);
            h[3] += hit_fp64(a.w, b.w);
        }
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            if (!cur.live(P, l)) continue;
            total += h[l];
            if (P.counts) atomicAdd(P.counts + cur.row0 + l, (unsigned long long)h[l]);
        }
    }
    block_reduce_add(total, P.hits);
}

template <int G>
cudaError_t fill_g(const LeapLaunch& p, int kind, bool vec, Grid g, cudaStream_t s)
{
    if (G == kLeapPhilox && p.ngroups) {
        if (vec) {
            if (kind == kU32) leap_fill_grouped_kernel<kU32, true><<<g.blocks, g.threads, 0, s>>>(p);
            else if (kind == kF32) leap_fill_grouped_kernel<kF32, true><<<g.blocks, g.threads, 0, s>>>(p);
            else leap_fill_grouped_kernel<kF64, true><<<g.blocks, g.threads, 0, s>>>(p);
        } else {
            if (kind == kU32) leap_fill_grouped_kernel<kU32, false><<<g.blocks, g.threads, 0, s>>>(p);
            else if (kind == kF32) leap_fill_grouped_kernel<kF32, false><<<g.blocks, g.threads, 0, s>>>(p);
            else leap_fill_grouped_kernel<kF64, false><<<g.blocks, g.threads, 0, s>>>(p);
        }
        return cudaGetLastError();
    }
    if (vec) {
        if (kind == kU32) leap_fill_kernel<G, kU32, true><<<g.blocks, g.threads, 0, s>>>(p);
        else if (kind == kF32) leap_fill_kernel<G, kF32, true><<<g.blocks, g.threads, 0, s>>>(p);
        else leap_fill_kernel<G, kF64, true><<<g.blocks, g.threads, 0, s>>>(p);
    } else {
        if (kind == kU32) leap_fill_kernel<G, kU32, false><<<g.blocks, g.threads, 0, s>>>(p);
        else if (kind == kF32) leap_fill_kernel<G, kF32, false><<<g.blocks, g.threads, 0, s>>>(p);
        else leap_fill_kernel<G, kF64, false><<<g.blocks, g.threads, 0, s>>>(p);
    }
    return cudaGetLastError();
}

template <int G>
cudaError_t occ_fill_g(int kind, bool vec, int threads, int* out)
{
    if (kind == kU32) return vec ? occ(leap_fill_kernel<G, kU32, true>, threads, 0, out)
                                 : occ(leap_fill_kernel<G, kU32, false>, threads, 0, out);
    if (kind == kF32) return vec ? occ(leap_fill_kernel<G, kF32, true>, threads, 0, out)
                                 : occ(leap_fill_kernel<G, kF32, false>, threads, 0, out);
    return vec ? occ(leap_fill_kernel<G, kF64, true>, threads, 0, out)
               : occ(leap_fill_kernel<G, kF64, false>, threads, 0, out);
}

}  // namespace

cudaError_t launch_leap_fill(const LeapLaunch& p, int lgen, int kind, bool vec, Grid g, cudaStream_t s)
{
    if (lgen == kLeapMrg) return fill_g<kLeapMrg>(p, kind, vec, g, s);
    if (lgen == kLeapPhilox) return fill_g<kLeapPhilox>(p, kind, vec, g, s);
    return fill_g<kLeapThreefry>(p, kind, vec, g, s);
}

cudaError_t launch_leap_fill_tma(const LeapLaunch& p, const CUtensorMap& tmap, int kind, Grid g, cudaStream_t s)
{
    cudaError_t e = kind == kF32 ? leap_tma_attr<kF32>() : leap_tma_attr<kU32>();
    if (e != cudaSuccess) return e;
    if (kind == kF32) leap_fill_tma_kernel<kF32><<<g.blocks, kLeapTmaWarps * 32, leap_tma_smem(), s>>>(p, tmap);
    else leap_fill_tma_kernel<kU32><<<g.blocks, kLeapTmaWarps * 32, leap_tma_smem(), s>>>(p, tmap);
    return cudaGetLastError();
}

cudaError_t leap_tma_blocks_per_sm(int kind, int* out)
{
    cudaError_t e = kind == kF32 ? leap_tma_attr<kF32>() : leap_tma_attr<kU32>();
    if (e != cudaSuccess) return e;
    return kind == kF32 ? occ(leap_fill_tma_kernel<kF32>, kLeapTmaWarps * 32, leap_tma_smem(), out)
                        : occ(leap_fill_tma_kernel<kU32>, kLeapTmaWarps * 32, leap_tma_smem(), out);
}

cudaError_t launch_leap_mrg_tr(const LeapLaunch& p, const CUtensorMap& tmap, int kind, unsigned blocks, cudaStream_t s)
{
    cudaError_t e = kind == kF32 ? leap_tr_attr<kF32>() : leap_tr_attr<kU32>();
    if (e != cudaSuccess) return e;
    if (kind == kF32) leap_mrg_tr_kernel<kF32><<<blocks, kTrWarpsMrg * 32, leap_tr_smem_mrg(), s>>>(p, tmap);
    else leap_mrg_tr_kernel<kU32><<<blocks, kTrWarpsMrg * 32, leap_tr_smem_mrg(), s>>>(p, tmap);
    return cudaGetLastError();
}

template <int G>
cudaError_t launch_ctr_tr_g(const LeapLaunch& p, const CUtensorMap& tmap, int kind, unsigned blocks, cudaStream_t s)
{
    cudaError_t e = kind == kF32 ? leap_trp_attr<kF32, G>() : leap_trp_attr<kU32, G>();
    if (e != cudaSuccess) return e;
    if (kind == kF32) leap_ctr_tr_kernel<kF32, G><<<blocks, kTrWarps * 32, leap_tr_smem(leap_ctr_cols_of(G)), s>>>(p, tmap);
    else leap_ctr_tr_kernel<kU32, G><<<blocks, kTrWarps * 32, leap_tr_smem(leap_ctr_cols_of(G)), s>>>(p, tmap);
    return cudaGetLastError();
}

cudaError_t launch_leap_ctr_tr(const LeapLaunch& p, const CUtensorMap& tmap, int lgen, int kind, unsigned blocks,
                               cudaStream_t s)
{
    return lgen == kLeapPhilox ? launch_ctr_tr_g<kLeapPhilox>(p, tmap, kind, blocks, s)
                               : launch_ctr_tr_g<kLeapThreefry>(p, tmap, kind, blocks, s);
}

uint32_t leap_tr_rows() { return kTrRows; }
uint32_t leap_ctr_cols(int lgen) { return leap_ctr_cols_of(lgen); }
uint32_t leap_tr_warps(bool mrg) { return mrg ? kTrWarpsMrg : kTrWarps; }

cudaError_t leap_ctr_tr_blocks_per_sm(int lgen, int kind, int* out)
{
    if (lgen == kLeapPhilox) {
        const cudaError_t e = kind == kF32 ? leap_trp_attr<kF32, kLeapPhilox>() : leap_trp_attr<kU32, kLeapPhilox>();
        if (e != cudaSuccess) return e;
        return kind == kF32 ? occ(leap_ctr_tr_kernel<kF32, kLeapPhilox>, kTrWarps * 32, leap_tr_smem(leap_ctr_cols_of(kLeapPhilox)), out)
                            : occ(leap_ctr_tr_kernel<kU32, kLeapPhilox>, kTrWarps * 32, leap_tr_smem(leap_ctr_cols_of(kLeapPhilox)), out);
    }
    const cudaError_t e = kind == kF32 ? leap_trp_attr<kF32, kLeapThreefry>() : leap_trp_attr<kU32, kLeapThreefry>();
    if (e != cudaSuccess) return e;
    return kind == kF32 ? occ(leap_ctr_tr_kernel<kF32, kLeapThreefry>, kTrWarps * 32, leap_tr_smem(), out)
                        : occ(leap_ctr_tr_kernel<kU32, kLeapThreefry>, kTrWarps * 32, leap_tr_smem(), out);
}

cudaError_t leap_mrg_tr_blocks_per_sm(int kind, int* out)
{
    cudaError_t e = kind == kF32 ? leap_tr_attr<kF32>() : leap_tr_attr<kU32>();
    if (e != cudaSuccess) return e;
    return kind == kF32 ? occ(leap_mrg_tr_kernel<kF32>, kTrWarpsMrg * 32, leap_tr_smem_mrg(), out)
                        : occ(leap_mrg_tr_kernel<kU32>, kTrWarpsMrg * 32, leap_tr_smem_mrg(), out);
}

cudaError_t launch_leap_mc(const LeapLaunch& p, int lgen, Grid g, cudaStream_t s)
{
    if (lgen == kLeapPhilox && p.ngroups) leap_mc_grouped_kernel<<<g.blocks, g.threads, 0, s>>>(p);
    else if (lgen == kLeapMrg) leap_mc_kernel<kLeapMrg><<<g.blocks, g.threads, 0, s>>>(p);
    else if (lgen == kLeapPhilox) leap_mc_kernel<kLeapPhilox><<<g.blocks, g.threads, 0, s>>>(p);
    else leap_mc_kernel<kLeapThreefry><<<g.blocks, g.threads, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t leap_occupancy(int kernel, int kind, bool fast, int threads, int* out)
{
    switch (kernel) {
    case leap_kernel_id(kKLeapFill, kLeapMrg): return occ_fill_g<kLeapMrg>(kind, fast, threads, out);
    case leap_kernel_id(kKLeapFill, kLeapPhilox): return occ_fill_g<kLeapPhilox>(kind, fast, threads, out);
    case leap_kernel_id(kKLeapFill, kLeapThreefry): return occ_fill_g<kLeapThreefry>(kind, fast, threads, out);
    case leap_kernel_id(kKLeapMc, kLeapMrg): return occ(leap_mc_kernel<kLeapMrg>, threads, 0, out);
    case leap_kernel_id(kKLeapMc, kLeapPhilox): return occ(leap_mc_kernel<kLeapPhilox>, threads, 0, out);
    case leap_kernel_id(kKLeapMc, kLeapThreefry): return occ(leap_mc_kernel<kLeapThreefry>, threads, 0, out);
    }
    return cudaErrorInvalidValue;
}

}  // namespace shv
