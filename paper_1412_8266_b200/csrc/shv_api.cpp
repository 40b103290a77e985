// shv_api.cpp — the C ABI (include/shv.h): handle registry, validation,
// host-side jump-matrix math (H1), partitioning and work split (H2), launches.
//
// Host math: 3x3 matrices mod m = 2^32 - c with entries < m; products folded
// with 2^32 = c (mod m). A process-wide table P[b] = A^(2^b), b < 192, built
// once by repeated squaring, turns any jump A^e (e < 2^192) into a product over
// the set bits of e (P L112-117 [§2.3]: jump-ahead; P L264-268 [§4.1]: streams
// 2^127 and substreams 2^76 apart).
#include "../../include/shv.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>

#include "shv_internal.h"

#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled

#ifndef SHV_MRG_ORDER
#define SHV_MRG_ORDER 0  // lab: 0 = by row length, 1 = streams fastest, 2 = segments fastest
#endif
#ifndef SHV_MRG_ROWS
#define SHV_MRG_ROWS 1  // MRG32k3a u32/f32 fills in row tiles (0: stream-per-lane tiles only; lab A/B)
#endif
#ifndef SHV_MRG_ROWS_F64
#define SHV_MRG_ROWS_F64 1  // f64 fills in row tiles too (0: the staged vector kernel)
#endif
#ifndef SHV_MRG_TMA
#define SHV_MRG_TMA 1  // MRG32k3a fills store through TMA (0: per-lane vector stores; lab A/B)
#endif

#include <nvtx3/nvToolsExt.h>

namespace shv {
namespace {

using u128 = unsigned __int128;

constexpr uint32_t kM1 = 4294967087u, kM2 = 4294944443u;
constexpr uint32_t kC[2] = {209u, 22853u};
constexpr uint32_t kMod[2] = {kM1, kM2};

thread_local std::string t_err;

// NVTX range around each ABI call (visible in nsys / ncu --nvtx; a no-op
// unless a tool is attached).
struct Range {
    explicit Range(const char* name) { nvtxRangePushA(name); }
    ~Range() { nvtxRangePop(); }
};

shv_status fail(shv_status s, const char* fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    t_err = buf;
    return s;
}

// ---------------------------------------------------------------- H1: jump math

struct Mat {
    uint32_t v[9];
};

inline uint32_t fold(uint64_t x, int comp)
{
    const uint64_t c = kC[comp], m = kMod[comp];
    x = (x >> 32) * c + (uint32_t)x;
    x = (x >> 32) * c + (uint32_t)x;
    return (uint32_t)(x >= m ? x - m : x);
}

Mat mul(const Mat& A, const Mat& B, int comp)
{
    Mat R;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            uint64_t s = 0;
            for (int k = 0; k < 3; ++k) s += fold((uint64_t)A.v[3 * r + k] * B.v[3 * k + c], comp);
            R.v[3 * r + c] = fold(s, comp);
        }
    return R;
}

const Mat kIdentity = {{1, 0, 0, 0, 1, 0, 0, 0, 1}};

struct PowTable {
    Mat p[2][192];  // p[comp][b] = A_comp^(2^b)
    PowTable()
    {
        // Companion matrices of x1,n = a12 x1,n-2 - a13n x1,n-3 and
        // x2,n = a21 x2,n-1 - a23n x2,n-3 on (x_{n-3}, x_{n-2}, x_{n-1}) (R3).
        const Mat A1 = {{0, 1, 0, 0, 0, 1, kM1 - 810728u, 1403580u, 0}};
        const Mat A2 = {{0, 1, 0, 0, 0, 1, kM2 - 1370589u, 0, 527612u}};
        p[0][0] = A1;
        p[1][0] = A2;
        for (int c = 0; c < 2; ++c)
            for (int b = 1; b < 192; ++b) p[c][b] = mul(p[c][b - 1], p[c][b - 1], c);
    }
};

const PowTable& pow_table()
{
    static const PowTable t;
    return t;
}

// A^(e * 2^shift), e < 2^128, shift + bitlen(e) <= 192.
Mat mpow(u128 e, int shift, int comp)
{
    const PowTable& T = pow_table();
    Mat R = kIdentity;
    for (int b = 0; e; ++b, e >>= 1)
        if (e & 1) R = mul(R, T.p[comp][b + shift], comp);
    return R;
}

MatPair pair_pow(u128 e, int shift)
{
    MatPair P;
    const Mat a = mpow(e, shift, 0), b = mpow(e, shift, 1);
    memcpy(P.a, a.v, sizeof P.a);
    memcpy(P.b, b.v, sizeof P.b);
    return P;
}

MatPair pair_mul(const MatPair& X, const MatPair& Y)
{
    Mat xa, xb, ya, yb;
    memcpy(xa.v, X.a, 36);
    memcpy(xb.v, X.b, 36);
    memcpy(ya.v, Y.a, 36);
    memcpy(yb.v, Y.b, 36);
    const Mat a = mul(xa, ya, 0), b = mul(xb, yb, 1);
    MatPair R;
    memcpy(R.a, a.v, 36);
    memcpy(R.b, b.v, 36);
    return R;
}

void pair_apply(const MatPair& P, uint32_t s[6])
{
    for (int c = 0; c < 2; ++c) {
        const uint32_t* M = c ? P.b : P.a;
        uint32_t* v = s + 3 * c;
        uint32_t r[3];
        for (int k = 0; k < 3; ++k) {
            uint64_t acc = 0;
            for (int q = 0; q < 3; ++q) acc += fold((uint64_t)M[3 * k + q] * v[q], c);
            r[k] = fold(acc, c);
        }
        memcpy(v, r, sizeof r);
    }
}

// ---------------------------------------------------------------- registry

struct Handle {
    int gen = 0, spacing = 0, device = 0;
    uint32_t seed[6] = {};
    uint64_t first = 0, n = 0;
    u128 offset = 0;
    uint32_t* state = nullptr;
    bool own_state = false;
    uint32_t bps = 0, tpb = 256;
    uint64_t seg = 0;
    int sms = 0;
    // TinyMT32 (stateful; R15)
    uint32_t* params = nullptr;  // owned, (mat1, mat2, tmat) per group from group0
    uint64_t group0 = 0;
    uint32_t group_size = 0;
    uint64_t players = 0;         // Leap Frog: K (spacing SHV_SPACING_LEAPFROG)
};

TinyMtLaunch tm_launch(const Handle& h, uint64_t s0, uint64_t ns)
{
    TinyMtLaunch P{};
    P.state = h.state + s0;
    P.stride = h.n;
    P.ns = ns;
    P.params = h.params;
    P.first = h.first + s0;
    P.group0 = h.group0;
    P.group_size = h.group_size;
    return P;
}

MtgpLaunch mtgp_launch(const Handle& h, uint64_t s0, uint64_t ns)
{
    MtgpLaunch P{};
    P.state = h.state + kMtgpStateWords * s0;
    P.params = h.params + kMtgpParamWords * s0;
    P.ns = ns;
    P.first = h.first + s0;
    return P;
}

// One CTA per MTGP32 state (the generator's block-cooperative design); CTAs
// loop over states when there are more than fit at once.
unsigned mtgp_blocks(const Handle& h, uint64_t ns)
{
    const uint64_t cap = (uint64_t)(h.sms > 0 ? h.sms : 148) * 8;
    return (unsigned)(ns < cap ? (ns ? ns : 1) : cap);
}

std::mutex g_mu;
std::unordered_map<uint64_t, std::shared_ptr<Handle>> g_handles;
std::atomic<uint64_t> g_next_id{1};
bool g_tables_on[64] = {};

std::shared_ptr<Handle> lookup(shv_streams h)
{
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_handles.find(h);
    return it == g_handles.end() ? nullptr : it->second;
}

// Saves/restores the caller's current device around a call.
struct DeviceGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int dev)
    {
        err = cudaGetDevice(&prev);
        if (err == cudaSuccess && prev != dev) err = cudaSetDevice(dev);
    }
    ~DeviceGuard()
    {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

shv_status cuda_fail(cudaError_t e, const char* what)
{
    return fail(SHV_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

shv_status ensure_tables(int dev)
{
    std::lock_guard<std::mutex> lk(g_mu);
    if (dev < 0 || dev >= 64) return fail(SHV_ERR_INVALID_ARGUMENT, "device %d out of range", dev);
    if (g_tables_on[dev]) return SHV_OK;
    MatPair sub[51], str[64], drw[64];
    for (int b = 0; b < 51; ++b) sub[b] = pair_pow(1, 76 + b);
    for (int b = 0; b < 64; ++b) str[b] = pair_pow(1, 127 + b);
    for (int b = 0; b < 64; ++b) drw[b] = pair_pow(1, b);
    cudaError_t e = upload_jump_tables(sub, str, drw);
    if (e != cudaSuccess) return cuda_fail(e, "upload_jump_tables");
    g_tables_on[dev] = true;
    return SHV_OK;
}

// ---------------------------------------------------------------- H2: work split

// Occupancy (blocks per SM) of a kernel variant at a block size, cached per
// device: the query is host work on every launch otherwise.
int occupancy(int device, int kernel, int kind, bool fast, int tpb)
{
    static std::mutex mu;
    static std::unordered_map<uint64_t, int> cache;
    const uint64_t key = ((uint64_t)(device & 0xff) << 32) | ((uint64_t)kernel << 24) |
                         ((uint64_t)kind << 16) | ((uint64_t)fast << 12) | (uint64_t)tpb;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    int bps = 0;
    if (max_blocks_per_sm(kernel, kind, fast, tpb, &bps) != cudaSuccess || bps < 1) bps = 1;
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = bps;
    return bps;
}

unsigned blocks_for(const Handle& h, int kernel, int kind, bool fast, uint64_t items)
{
    int bps = (int)h.bps;
    if (bps == 0) bps = occupancy(h.device, kernel, kind, fast, (int)h.tpb);
    const uint64_t full = (uint64_t)h.sms * (uint64_t)bps;
    const uint64_t need = (items + h.tpb - 1) / h.tpb;
    uint64_t b = need < full ? need : full;
    return (unsigned)(b ? b : 1);
}

uint64_t resident_threads(const Handle& h, int kernel, int kind, bool fast)
{
    int bps = (int)h.bps;
    if (bps == 0) bps = occupancy(h.device, kernel, kind, fast, (int)h.tpb);
    return (uint64_t)h.sms * (uint64_t)bps * h.tpb;
}

// Split rows of `len` units into nseg segments of seg_len units (multiple of
// `align`, at least min_len unless the row is shorter), aiming at `waves` x
// resident threads work items; nseg < 2^kSegBits.
void split(const Handle& h, uint64_t ns, uint64_t len, uint64_t align, uint64_t waves,
           uint64_t resident, uint64_t cap, uint64_t* seg_len, uint32_t* nseg, uint64_t min_len = 256)
{
    uint64_t L;
    if (h.seg) {
        L = h.seg;
    } else {
        const uint64_t target = waves * resident;
        const uint64_t S = (target + ns - 1) / ns;
        L = (len + S - 1) / S;
        if (L < min_len) L = min_len;
    }
    L = (L + align - 1) / align * align;
    if (L > cap) L = cap / align * align;
    if (L == 0) L = align;
    uint64_t S = (len + L - 1) / L;
    while (S >= (1ull << kSegBits)) {  // user segment too short for 2^32 segments: grow it
        L *= 2;
        S = (len + L - 1) / L;
    }
    *seg_len = L;
    *nseg = (uint32_t)(S ? S : 1);
}

// TMA fill of MRG32k3a (mrg_fill_tma_kernel): a warp owns a tile of 32 rows
// x one segment, and tiles go round-robin over the resident warps, so the
// segment count decides the tail: pick the 64-value-aligned segment length
// that minimises rounds x (segment + start-jump cost), the start jump (state
// load, A^o and the per-bit segment jumps) costing about as much as 16 values.
void split_tiles(const Handle& h, uint64_t ns, uint64_t len, uint64_t resident_threads, uint64_t* seg_len,
                 uint32_t* nseg)
{
    if (h.seg) {
        split(h, ns, len, 64, 8, resident_threads, 1ull << 40, seg_len, nseg);
        return;
    }
    const uint64_t warps = resident_threads / 32 ? resident_threads / 32 : 1;
    const uint64_t G = (ns + 31) / 32;
    uint64_t bestL = (len + 63) / 64 * 64, bestS = 1;
    double best = -1.0;
    for (uint64_t S = 1; S <= 256; ++S) {
        const uint64_t L = ((len + S - 1) / S + 63) / 64 * 64;
        const uint64_t Sa = (len + L - 1) / L;
        if (Sa != S || (S > 1 && L < 256)) continue;
        const uint64_t tiles = G * S;
        const double rounds = (double)((tiles + warps - 1) / warps);
        const double cost = rounds * (double)(L + 16);
        if (best < 0 || cost < best) {
            best = cost;
            bestL = L;
            bestS = S;
        }
    }
    *seg_len = bestL;
    *nseg = (uint32_t)bestS;
}

// Row-tile segment length of the MRG32k3a u32/f32 fill: the first divisor of
// n in {128, 96, 160, 192, 64, 224, 256, ...}. S = 128 makes a warp tile one
// 16-KB region, the best store layout (6.1 vs 5.1 TB/s at S = 256 with a null
// generator). With the MrgIF step the C5 shape took S = 256 (half the lane
// starts: 3.38 vs 3.46 ms, lab42); with MrgSN / MrgMF the step is cheap enough that the
// S = 256 layout binds on its TMA stores (4.04 vs 3.17-3.25 ms, lab50).
// 0 if n has none.
uint64_t mrg_rows_seg_len(uint64_t n, int kind = kU32)
{
    // f64: half the values per segment (the same 512-B segments and 16-KB tiles in bytes;
    // rounds of 16 doubles): S = S_u32(2n) / 2
    if (kind == kF64) {
        if (n > (~0ull >> 1)) return 0;
        const uint64_t S2 = mrg_rows_seg_len(2 * n, kU32);
        return S2 % 32 == 0 ? S2 / 2 : 0;
    }
#ifdef SHV_MRG_ROWS_S  // lab knob: preferred segment length
    if (n % SHV_MRG_ROWS_S == 0) return SHV_MRG_ROWS_S;
#endif
    static const uint64_t pref[] = {128, 96, 160, 192, 64, 224, 256, 320, 384, 448, 512};
    for (uint64_t S : pref)
        if (n % S == 0) return S;
    return 0;
}

// The row-tile path takes 4-byte kinds at 16-B aligned outputs, no launch-config
// segment override, tensor dims < 2^31, and enough tiles (>= 2 per resident warp)
// that the stream-per-lane path's segment split would not balance better.
bool mrg_rows_fit(const Handle& h, int kind, bool aligned32, uint64_t ns, uint64_t n)
{
    if (!SHV_MRG_ROWS || !SHV_MRG_TMA || (kind == kF64 && !SHV_MRG_ROWS_F64) || !aligned32 || h.seg) return false;
    const uint64_t S = mrg_rows_seg_len(n, kind);
    if (!S || ns * (n / S) >= (1ull << 31)) return false;
    if (mrg_fill_rows_smem((int)h.tpb) > 227u * 1024u) return false;
    const uint64_t tiles = (ns * (n / S) + 31) / 32;
    return tiles >= 2 * resident_threads(h, kKMrgFillRows, kind, true) / 32;
}

// Leap Frog: the last base draw a call touches is (first+n-1) + K*(o+draws-1);
// it must exist in the base stream (R17).
shv_status check_leap_advance(const Handle& h, u128 draws)
{
    const u128 top = ~(u128)0;
    const u128 K = h.players;
    if (draws == 0) return SHV_OK;
    if (h.offset > top - draws || h.offset + draws > top / K)
        return fail(SHV_ERR_INVALID_ARGUMENT, "Leap Frog position would exceed 2^128 base draws");
    const u128 last = (u128)(h.first + h.n - 1) + K * (h.offset + draws - 1);
    const int lim = h.gen == SHV_GEN_PHILOX4X32_10 ? 66 : h.gen == SHV_GEN_THREEFRY4X64_20 ? 67 : 128;
    if (lim < 128 && last >= ((u128)1 << lim))
        return fail(SHV_ERR_INVALID_ARGUMENT, "Leap Frog base stream exhausted (2^%d draws)", lim);
    return SHV_OK;
}

shv_status check_advance(const Handle& h, u128 draws)
{
    if (h.spacing == SHV_SPACING_LEAPFROG) return check_leap_advance(h, draws);
    if (h.gen == SHV_GEN_THREEFRY4X64_20) {
        if (draws > ((u128)1 << 67) || h.offset > ((u128)1 << 67) - draws)
            return fail(SHV_ERR_INVALID_ARGUMENT, "Threefry stream exhausted (2^67 draws per stream)");
        return SHV_OK;
    }
    if (h.gen == SHV_GEN_PHILOX4X32_10) {
        if (draws > ((u128)1 << 66) || h.offset > ((u128)1 << 66) - draws)
            return fail(SHV_ERR_INVALID_ARGUMENT, "Philox stream exhausted (2^66 draws per stream)");
    } else if (h.offset + draws < h.offset) {
        return fail(SHV_ERR_INVALID_ARGUMENT, "offset would exceed 2^128 draws");
    }
    return SHV_OK;
}

// cuTensorMapEncodeTiled from the driver (no libcuda link); nullptr if absent.
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// 2D map of `ns` rows x `n` values of `elem` bytes at `out` (row-major), box
// 128 B x 32 rows with the 128-byte swizzle (mrg_fill_tma_kernel).
// Transposed fills write their boxes unswizzled: lane l stores word l of a box row, so the
// 32 lanes of one st.shared cover one 128-B row (conflict-free) at base + row * 128 + 4 l.
bool encode_rows_map(CUtensorMap* m, void* out, uint64_t n, uint64_t ns, int elem, uint32_t box_rows = 32,
                     bool swizzle = true, uint32_t row_bytes = 128)
{
    const auto enc = tensor_map_encoder();
    if (!enc) return false;
    const cuuint64_t dims[2] = {n, ns};
    const cuuint64_t strides[1] = {n * (uint64_t)elem};
    const cuuint32_t box[2] = {row_bytes / (cuuint32_t)elem, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return enc(m, elem == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, out, dims, strides,
               box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Segment jumps of a MRG launch: seg0 = A^o, segpow[b] = (A^(L*dpu))^(2^b)
// for the bits b that segment indices < nseg use.
void fill_mrg_segments(const Handle& h, uint64_t units_per_seg, uint64_t draws_per_unit, uint32_t nseg,
                       MrgLaunch* P)
{
    // shv::dev::MrgFpK: 1.5*2^52, RN(1/m1), RU(1/m2), m1, m2, a23n*m2 (include/shv_device.cuh)
    const double fpk[6] = {6755399441055744.0, 1.0 / 4294967087.0, 0x1.000059451f212p-32,
                           4294967087.0, 4294944443.0, 5886603609186927.0};
    memcpy(P->fpk, fpk, sizeof fpk);
    P->imul[0] = 1403580u;  // a12
    P->imul[1] = 810728u;   // a13n
    // shv::dev::MrgFpK::sn_*: D(202682 m1), D(a23n m2), 4 RN(1/m1) 2^1010, RU(1/m2) 2^1010, 1.5 2^-12
    const double snk[5] = {0x0.317b9fd79a126p-1022, 0x1.4e9d5b50f226fp-1022, 0x1.000000d10000bp+980,
                           0x1.000059451f212p+978, 0x1.8p-12};
    memcpy(P->snk, snk, sizeof snk);
    P->seg0 = pair_pow(h.offset, 0);
    P->segpow[0] = pair_pow((u128)units_per_seg * draws_per_unit, 0);
    for (int b = 1; b < kSegBits && ((uint64_t)nseg - 1) >> b; ++b)
        P->segpow[b] = pair_mul(P->segpow[b - 1], P->segpow[b - 1]);
}

// Warp tasks of the counter-based fast fills: (row, 32*R chunks of 32 B). R
// starts at ceil(chunks_per_row / 32) <= 16 and halves until there are >= 4
// tasks per resident warp (load balance); a launch-config segment overrides it.
// Rows of at most 16 runs per lane are grouped: *rpt_out whole rows per task,
// about 16 runs per lane, still >= 4 tasks per resident warp.
void counter_tasks(const Handle& h, uint64_t ns, uint64_t cpr, uint64_t resident, uint32_t* R_out,
                   uint64_t* tasks_out, uint32_t* rpt_out = nullptr)
{
    const uint64_t rwarps = resident / 32;
    uint64_t R = (cpr + 31) / 32;
    if (R > 16) R = 16;
    if (h.seg) R = h.seg / 8 < 1 ? 1 : (h.seg / 8 > 64 ? 64 : h.seg / 8);
    auto tasks = [&](uint64_t r) { return ns * ((cpr + 32 * r - 1) / (32 * r)); };
    while (!h.seg && R > 1 && tasks(R) < 4 * rwarps) R /= 2;
    *R_out = (uint32_t)R;
    *tasks_out = tasks(R);
    if (!rpt_out) return;
    *rpt_out = 1;
    if (h.seg || 32 * R < cpr) return;  // rows span several tasks
    uint64_t rpt = 16 / R;
    while (rpt > 1 && (ns + rpt - 1) / rpt < 4 * rwarps) rpt /= 2;
    if (rpt > 1) {
        *rpt_out = (uint32_t)rpt;
        *tasks_out = (ns + rpt - 1) / rpt;
    }
}

// ---------------------------------------------------------------- Leap Frog (R17)

uint32_t mulmod(uint64_t a, uint64_t b, uint64_t m) { return (uint32_t)((u128)a * b % m); }

// Coefficients of u_{t+3} = cp[2] u_{t+2} + cp[1] u_{t+1} + cp[0] u_t for the
// order-3 recurrence B's characteristic polynomial gives (Cayley-Hamilton:
// B^3 = tr B^2 - M2 B + det I; M2 = sum of the principal 2x2 minors).
void charpoly(const uint32_t* B, int comp, uint32_t cp[3])
{
    const uint64_t m = kMod[comp];
    auto e = [&](int r, int c) -> uint64_t { return B[3 * r + c]; };
    auto minor = [&](int a, int b) -> uint64_t {  // B[a][a] B[b][b] - B[a][b] B[b][a] (mod m)
        return (mulmod(e(a, a), e(b, b), m) + m - mulmod(e(a, b), e(b, a), m)) % m;
    };
    const uint64_t tr = (e(0, 0) + e(1, 1) + e(2, 2)) % m;
    const uint64_t m2 = (minor(0, 1) + minor(0, 2) + minor(1, 2)) % m;
    const uint64_t c0 = (mulmod(e(1, 1), e(2, 2), m) + m - mulmod(e(1, 2), e(2, 1), m)) % m;
    const uint64_t c1 = (mulmod(e(1, 0), e(2, 2), m) + m - mulmod(e(1, 2), e(2, 0), m)) % m;
    const uint64_t c2 = (mulmod(e(1, 0), e(2, 1), m) + m - mulmod(e(1, 1), e(2, 0), m)) % m;
    const uint64_t det = (mulmod(e(0, 0), c0, m) + m - mulmod(e(0, 1), c1, m) + mulmod(e(0, 2), c2, m)) % m;
    cp[2] = (uint32_t)tr;
    cp[1] = (uint32_t)((m - m2) % m);
    cp[0] = (uint32_t)det;
}

int leap_gen(int gen) { return gen == SHV_GEN_MRG32K3A ? kLeapMrg : gen == SHV_GEN_PHILOX4X32_10 ? kLeapPhilox : kLeapThreefry; }

// A Leap Frog launch over handle rows [s0, s0+ns): len units per row (values
// or samples), dpv player draws per unit. Segments of >= 64 units (a MRG
// segment start costs up to 35 mat-vecs), enough work items for 8 waves.
// Philox Leap Frog players share counter blocks four at a time when K % 4 == 0
// (grouped kernels, kernels_leapfrog.cu).
bool leap_grouped(const Handle& h) { return h.gen == SHV_GEN_PHILOX4X32_10 && h.players % 4 == 0; }

std::unique_ptr<LeapLaunch> leap_launch(const Handle& h, uint64_t s0, uint64_t ns, uint64_t len, uint64_t dpv,
                                        uint64_t align, uint64_t resident)
{
    auto P = std::make_unique<LeapLaunch>();
    const bool grouped = leap_grouped(h);
    const uint64_t first = h.first + s0;
    const uint64_t nrow_items = grouped ? ((first + ns - 1) >> 2) - (first >> 2) + 1 : ns;
    uint64_t L;
    if (h.seg) {
        L = h.seg;
    } else {
        const uint64_t target = 8 * resident;
        const uint64_t S = (target + nrow_items - 1) / nrow_items;
        L = (len + S - 1) / S;
        if (L < 64) L = 64;
    }
    L = (L + align - 1) / align * align;
    if (L > (1ull << 31)) L = (1ull << 31) / align * align;  // MC: per-item counts fit in u32
    const uint64_t nseg = (len + L - 1) / L;
    P->players = h.players;
    P->first = h.first + s0;
    P->ns = ns;
    P->o_lo = (uint64_t)h.offset;
    P->o_hi = (uint64_t)(h.offset >> 64);
    P->seg_len = L;
    P->seg_draws = L * dpv;
    P->n = len;
    P->items = nrow_items * nseg;
    if (grouped) {
        P->g0 = first >> 2;
        P->ngroups = nrow_items;
    }
    if (h.gen == SHV_GEN_PHILOX4X32_10) {
        P->k0 = h.seed[0];
        P->k1 = h.seed[1];
    } else if (h.gen == SHV_GEN_THREEFRY4X64_20) {
        P->k0 = (uint64_t)h.seed[0] | ((uint64_t)h.seed[1] << 32);
        P->k1 = (uint64_t)h.seed[2] | ((uint64_t)h.seed[3] << 32);
    } else {
        P->state = h.state;
        P->stride = h.n;
        P->stream_begin = s0;
        P->B = pair_pow(h.players, 0);
        charpoly(P->B.a, 0, P->cp1);
        charpoly(P->B.b, 1, P->cp2);
        P->start = pair_pow(1 + (u128)h.players * h.offset, 0);
        P->segpow[0] = pair_pow((u128)h.players * P->seg_draws, 0);
        for (int b = 1; b < kSegBits && (nseg - 1) >> b; ++b) P->segpow[b] = pair_mul(P->segpow[b - 1], P->segpow[b - 1]);
    }
    return P;
}

template <typename T>
shv_status generate(shv_streams hid, T* out, uint64_t n, void* stream, int kind, bool host_out)
{
    Range nvtx_range(host_out ? "shv_generate_u32_host" : kind == kU32 ? "shv_generate_u32" : kind == kF32 ? "shv_generate_f32" : "shv_generate_f64");
    auto hp = lookup(hid);
    if (!hp) return fail(SHV_ERR_LIFECYCLE, "unknown or destroyed handle %llu", (unsigned long long)hid);
    Handle& h = *hp;
    if (!out && n) return fail(SHV_ERR_INVALID_ARGUMENT, "NULL output pointer");
    if ((uintptr_t)out % sizeof(T)) return fail(SHV_ERR_MISALIGNED, "output not %zu-byte aligned", sizeof(T));
    if (n == 0) return SHV_OK;
    if (h.n > UINT64_MAX / n / sizeof(T)) return fail(SHV_ERR_INVALID_ARGUMENT, "size overflow");
    const uint64_t dpv = (h.gen != SHV_GEN_MRG32K3A && kind == kF64) ? 2 : 1;
    shv_status st = check_advance(h, (u128)n * dpv);
    if (st) return st;
    DeviceGuard dg(h.device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    cudaStream_t s = (cudaStream_t)stream;

    // Host output: generate stream slices into device staging buffers and
    // copy them back on a second stream, two slices in flight.
    uint64_t slice = h.n;
    T* stage[2] = {nullptr, nullptr};
    cudaStream_t cs = nullptr;
    cudaEvent_t gen_done[2] = {}, copy_done[2] = {};
    const uint64_t row_bytes = n * sizeof(T);
    if (host_out) {
        const uint64_t target = 256ull << 20;
        slice = target / row_bytes;
        if (slice < 1) slice = 1;
        if (slice > h.n) slice = h.n;
        cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
        for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
            e = cudaMallocAsync((void**)&stage[b], slice * row_bytes, s);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&gen_done[b], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&copy_done[b], cudaEventDisableTiming);
        }
        if (e != cudaSuccess) {
            for (int b = 0; b < 2; ++b) {
                if (stage[b]) cudaFreeAsync(stage[b], s);
                if (gen_done[b]) cudaEventDestroy(gen_done[b]);
                if (copy_done[b]) cudaEventDestroy(copy_done[b]);
            }
            if (cs) cudaStreamDestroy(cs);
            return cuda_fail(e, "staging setup");
        }
    }

    cudaError_t err = cudaSuccess;
    const bool aligned32 = !host_out ? ((uintptr_t)out % 32 == 0) : true;
    for (uint64_t s0 = 0, k = 0; s0 < h.n && err == cudaSuccess; s0 += slice, ++k) {
        const uint64_t ns = (h.n - s0) < slice ? (h.n - s0) : slice;
        T* dst = host_out ? stage[k & 1] : out;
        if (host_out && k >= 2) err = cudaStreamWaitEvent(s, copy_done[k & 1], 0);
        if (err != cudaSuccess) break;
        CUtensorMap rows_tmap;  // MRG32k3a row-tile fill (encoded in its branch condition)
        if (h.spacing == SHV_SPACING_LEAPFROG && h.gen == SHV_GEN_TINYMT32) {
            TmLeapLaunch P{};
            P.buf = h.params;
            P.players = h.players;
            P.first = h.first + s0;
            P.ns = ns;
            P.o_lo = (uint64_t)h.offset;
            P.o_hi = (uint64_t)(h.offset >> 64);
            P.out = dst;
            P.n = n;
            CUtensorMap tmap;
            const bool tr = SHV_MRG_TMA && kind != kF64 && n % 4 == 0 && ((uintptr_t)dst % 16 == 0) &&
                            n < (1ull << 31) && ns < (1ull << 31) - 256 &&
                            encode_rows_map(&tmap, dst, n, ns, (int)sizeof(T), kTmTrRows);
            if (tr) {  // transpose of the base sequence, one TinyMT32 step per value (TMA boxes)
                int bps = 0;
                err = tm_leap_tr_blocks_per_sm(kind, &bps);
                P.tr_tb = (n + 31) / 32;
                const uint64_t warps = (uint64_t)h.sms * (uint64_t)(bps > 0 ? bps : 1) * 4;
                // items = tr_tb * tr_ps <= 4 waves of warps (rounding up made 4.04 waves at C5: a
                // fifth, nearly empty round)
                const uint64_t want_ps = (4 * warps) / P.tr_tb ? (4 * warps) / P.tr_tb : 1;
                uint64_t pl = (ns + want_ps - 1) / want_ps;
                if (pl < 4096) pl = 4096;  // long runs amortise the per-lane GF(2) jump
                P.tr_pl = (pl + kTmTrRows - 1) / kTmTrRows * kTmTrRows;
                P.tr_ps = (ns + P.tr_pl - 1) / P.tr_pl;
                const uint64_t items = P.tr_tb * P.tr_ps;
                const uint64_t cap = (uint64_t)h.sms * (uint64_t)(bps > 0 ? bps : 1);
                const uint64_t want = (items + 3) / 4;
                if (err == cudaSuccess) err = launch_tm_leap_tr(P, tmap, kind, (unsigned)(want < cap ? want : cap), s);
            } else {
                uint32_t nseg = 1;
                split(h, ns, n, 1, 8, (uint64_t)h.sms * 2048, 1ull << 40, &P.seg_len, &nseg, 64);
                P.seg_draws = P.seg_len * dpv;
                P.items = ns * nseg;
                Grid g{(unsigned)std::min<uint64_t>((P.items + 255) / 256, (uint64_t)h.sms * 8), 256};
                err = launch_tm_leap(P, kind, g, s);
            }
        } else if (h.spacing == SHV_SPACING_LEAPFROG) {
            const int lg = leap_gen(h.gen);
            bool vec = aligned32 && (n % 8 == 0);
            const int kid = leap_kernel_id(kKLeapFill, lg);
            // MRG32k3a, 4-byte values: fill by transposing the base sequence (TMA boxes)
            // Philox: K % 4 == 0 and a 4-aligned first player keep every lane's run
            // on whole counter blocks (leap_ctr_tr_kernel; Threefry: K % 8, 8-aligned)
            const bool trp = (h.gen == SHV_GEN_PHILOX4X32_10 && h.players % 4 == 0 && (h.first + s0) % 4 == 0) ||
                             (h.gen == SHV_GEN_THREEFRY4X64_20 && h.players % 8 == 0 && (h.first + s0) % 8 == 0);
            const uint32_t rows = leap_tr_rows();
            const uint32_t cols = trp ? leap_ctr_cols(lg) : 1u;  // 128-B box columns per lane
            CUtensorMap trmap;
            // an encode failure falls back to the per-player kernels below
            const bool tr = SHV_MRG_TMA && (h.gen == SHV_GEN_MRG32K3A || trp) && kind != kF64 && n % 4 == 0 &&
                            ((uintptr_t)dst % 16 == 0) && n < (1ull << 31) && ns < (1ull << 31) - 256 &&
                            encode_rows_map(&trmap, dst, n, ns, (int)sizeof(T), rows, false, 128u * cols);
            if (tr) {
                int bps = 0;
                err = trp ? leap_ctr_tr_blocks_per_sm(lg, kind, &bps) : leap_mrg_tr_blocks_per_sm(kind, &bps);
                auto P = std::make_unique<LeapLaunch>();
                P->players = h.players;
                P->first = h.first + s0;
                P->ns = ns;
                P->n = n;
                P->out = dst;
                P->o_lo = (uint64_t)h.offset;
                P->o_hi = (uint64_t)(h.offset >> 64);
                if (h.gen == SHV_GEN_THREEFRY4X64_20) {
                    P->k0 = (uint64_t)h.seed[0] | ((uint64_t)h.seed[1] << 32);
                    P->k1 = (uint64_t)h.seed[2] | ((uint64_t)h.seed[3] << 32);
                } else {
                    P->k0 = h.seed[0];
                    P->k1 = h.seed[1];
                }
                if (!trp) {
                    uint32_t s6[6];
                    memcpy(s6, h.seed, sizeof s6);
                    pair_apply(pair_pow((u128)P->first + (u128)h.players * h.offset, 0), s6);
                    memcpy(P->tr_s0, s6, sizeof s6);
                    P->segpow[0] = pair_pow(h.players, 0);  // (A^K)^(2^b): t offsets
                    for (int b = 1; b < kSegBits && ((n - 1) >> b); ++b)
                        P->segpow[b] = pair_mul(P->segpow[b - 1], P->segpow[b - 1]);
                }
                P->tr_tb = (n + 32 * cols - 1) / (32 * cols);
                const uint64_t wpb = leap_tr_warps(!trp);  // warps per block
                const uint64_t warps = (uint64_t)h.sms * (uint64_t)(bps > 0 ? bps : 1) * wpb;
                const uint64_t want_ps = (4 * warps) / P->tr_tb ? (4 * warps) / P->tr_tb : 1;
                uint64_t pl = (ns + want_ps - 1) / want_ps;
                if (pl < 1024) pl = 1024;  // runs long enough to amortise the start jump
                pl = (pl + rows - 1) / rows * rows;
                P->tr_pl = pl;
                P->tr_ps = (ns + pl - 1) / pl;
                P->tr_ppow[0] = pair_pow(pl, 0);
                for (int b = 1; b < kSegBits && ((P->tr_ps - 1) >> b); ++b)
                    P->tr_ppow[b] = pair_mul(P->tr_ppow[b - 1], P->tr_ppow[b - 1]);
                const double fpk[6] = {6755399441055744.0, 1.0 / 4294967087.0, 0x1.000059451f212p-32,
                                       4294967087.0, 4294944443.0, 1370589.0 * 4294944443.0};
                memcpy(P->fpk, fpk, sizeof fpk);
                P->imul[0] = 1403580u;  // a12
                P->imul[1] = 810728u;   // a13n
                const uint64_t items = P->tr_tb * P->tr_ps;
                const uint64_t cap = (uint64_t)h.sms * (uint64_t)(bps > 0 ? bps : 1);
                const uint64_t want = (items + wpb - 1) / wpb;
                if (err == cudaSuccess)
                    err = trp ? launch_leap_ctr_tr(*P, trmap, leap_gen(h.gen), kind, (unsigned)(want < cap ? want : cap), s)
                              : launch_leap_mrg_tr(*P, trmap, kind, (unsigned)(want < cap ? want : cap), s);
            } else {
            // grouped Philox, 4-byte values: TMA boxes of 32 values x 128 rows
            bool tma = SHV_MRG_TMA && vec && leap_grouped(h) && kind != kF64 && n % 32 == 0 &&
                       n < (1ull << 31) && ns < (1ull << 31) - 8;
            auto P = leap_launch(h, s0, ns, n, dpv, tma ? 32 : vec ? 8 : 1, resident_threads(h, kid, kind, vec));
            if (vec && P->seg_len % 8) vec = false;
            if (tma && P->seg_len % 32) tma = false;
            P->out = dst;
            CUtensorMap tmap;
            if (tma && !encode_rows_map(&tmap, dst, n, ns, (int)sizeof(T), 128)) tma = false;
            if (tma) {
                int bps = 0;
                err = leap_tma_blocks_per_sm(kind, &bps);
                const uint64_t tiles = (P->ngroups + 31) / 32 * (P->items / P->ngroups);
                const uint64_t cap = (uint64_t)h.sms * (uint64_t)(bps > 0 ? bps : 1);
                const uint64_t want = (tiles + 3) / 4;
                Grid g{(unsigned)(want < cap ? (want ? want : 1) : cap), 128};
                if (err == cudaSuccess) err = launch_leap_fill_tma(*P, tmap, kind, g, s);
            } else {
                Grid g{blocks_for(h, kid, kind, vec, P->items), h.tpb};
                err = launch_leap_fill(*P, lg, kind, vec, g, s);
            }
            }
        } else if (h.gen == SHV_GEN_THREEFRY4X64_20) {
            const uint64_t E = kind == kF64 ? 4 : 8;
            const bool fast = aligned32 && (n % E == 0) && ((uint32_t)h.offset & 7) == 0;
            ThreefryLaunch P{};
            P.k0 = (uint64_t)h.seed[0] | ((uint64_t)h.seed[1] << 32);
            P.k1 = (uint64_t)h.seed[2] | ((uint64_t)h.seed[3] << 32);
            P.g0 = h.first + s0;
            P.ns = ns;
            P.o_blk = (uint64_t)(h.offset >> 3);
            P.o_word = (uint32_t)(h.offset & 7);
            P.out = dst;
            P.n = n;
            Grid g{};
            if (fast) {
                counter_tasks(h, ns, n / E, resident_threads(h, kKThreefryFill, kind, true), &P.nseg, &P.items);
                g = Grid{blocks_for(h, kKThreefryFill, kind, true, P.items * 32), h.tpb};
            } else {
                P.items = (ns * n + 7) / 8;
                g = Grid{blocks_for(h, kKThreefryFill, kind, false, P.items), h.tpb};
            }
            err = launch_threefry_fill(P, kind, fast, g, s);
        } else if (h.gen == SHV_GEN_MTGP32) {
            MtgpLaunch P = mtgp_launch(h, s0, ns);
            P.out = dst;
            P.n = n;
            err = launch_mtgp(P, kind, mtgp_blocks(h, ns), s);
        } else if (h.gen == SHV_GEN_TINYMT32) {
            const bool vec = aligned32 && (n % 8 == 0) && n <= 0xFFFFFFFFull;
            TinyMtLaunch P = tm_launch(h, s0, ns);
            P.out = dst;
            P.n = n;
            const unsigned full = (unsigned)((ns + h.tpb - 1) / h.tpb);
            Grid g{vec ? blocks_for(h, kKTinyFill, kind, true, ns) : full, h.tpb};
            err = launch_tinymt_fill(P, kind, vec, g, s);
        } else if (h.gen == SHV_GEN_MRG32K3A && mrg_rows_fit(h, kind, aligned32, ns, n) &&
                   encode_rows_map(&rows_tmap, dst, mrg_rows_seg_len(n, kind), ns * (n / mrg_rows_seg_len(n, kind)),
                                   (int)sizeof(T))) {
            // row tiles: a warp writes 32 consecutive segments of S values (C5: two 16-KB rows);
            // an encode failure falls through to the stream-per-lane paths below
            const uint64_t S = mrg_rows_seg_len(n, kind);
            auto R = std::make_unique<MrgRowsLaunch>();
            MrgLaunch* P = &R->m;
            P->state = h.state;
            P->stride = h.n;
            P->stream_begin = s0;
            P->ns = ns;
            P->out = dst;
            P->n = n;
            P->seg_len = S;
            P->nseg = (uint32_t)(n / S);
            P->items = ns * P->nseg;
            P->seg_fastest = 1;
            fill_mrg_segments(h, 32 * S, 1, (P->nseg + 31) / 32, P);  // segpow: (A^(32 S))^(2^b)
            const MatPair AS = pair_pow(S, 0);
            R->lanetab[0] = P->seg0;  // A^o
            for (uint32_t k = 1; k < 32 && k < P->nseg; ++k) R->lanetab[k] = pair_mul(R->lanetab[k - 1], AS);
            // item / nseg for items < 2^31: l = ceil(log2 nseg), m = ceil(2^(31+l) / nseg) < 2^32,
            // floor(it / nseg) = (it * m) >> (31 + l) = umulhi(it, m) >> (l - 1)
            if (P->nseg > 1) {
                uint32_t l = 0;
                while ((1ull << l) < P->nseg) ++l;
                R->div_m = (uint32_t)(((1ull << (31 + l)) + P->nseg - 1) / P->nseg);
                R->div_s = l - 1;
            } else {
                R->div_m = 0;
                R->div_s = 0;
            }
            // run mode for rows of several tiles: runs of consecutive tiles per warp, about
            // four runs per resident warp (balance) and as long as possible (the first tile
            // of a run pays the per-bit jumps)
            R->nh = R->run = R->rpr = 0;
            if (P->nseg % 32 == 0 && P->nseg >= 64) {
                R->nh = P->nseg / 32;
                const uint64_t warps = resident_threads(h, kKMrgFillRows, kind, true) / 32;
                const uint64_t tiles = ns * R->nh;
                uint64_t run = tiles / (4 * (warps ? warps : 1));
                run = run < 1 ? 1 : run > R->nh ? R->nh : run;
                R->rpr = (uint32_t)((R->nh + run - 1) / run);
                R->run = (R->nh + R->rpr - 1) / R->rpr;  // equal runs (the last one at most rpr - 1 shorter)
                R->step31 = pair_pow((u128)31 * S, 0);
            }
            const uint64_t work = R->nh ? ns * R->rpr * 32 : (P->items + 31) / 32 * 32;
            Grid g{blocks_for(h, kKMrgFillRows, kind, true, work), h.tpb};
            err = launch_mrg_fill_rows(*R, rows_tmap, kind, g, s);
        } else if (h.gen == SHV_GEN_MRG32K3A) {
            bool vec = aligned32 && (n % 8 == 0);
            auto P = std::make_unique<MrgLaunch>();
            P->state = h.state;
            P->stride = h.n;
            P->stream_begin = s0;
            P->ns = ns;
            P->out = dst;
            P->n = n;
            // TMA path for 4-byte values: 128-B boxes of 32 rows (16-B aligned rows, int32 box
            // coordinates). f64 keeps the staged 256-B warp stores, faster there.
            bool tma = SHV_MRG_TMA && vec && kind != kF64 && n < (1ull << 31) && ns < (1ull << 31) &&
                       mrg_fill_tma_fits((int)h.tpb);
            const int kid = tma ? kKMrgFillTma : kKMrgFill;
            // vector paths: segments in whole 256-byte rounds (64 values; 2 or 4 TMA boxes)
            if (tma)
                split_tiles(h, ns, n, resident_threads(h, kid, kind, vec), &P->seg_len, &P->nseg);
            else
                split(h, ns, n, vec ? 64 : 1, 8, resident_threads(h, kid, kind, vec), 1ull << 40,
                      &P->seg_len, &P->nseg);
            if (vec && P->seg_len % 64) vec = tma = false;  // user segment length: per-lane paths
            P->items = ns * P->nseg;
            P->seg_fastest = SHV_MRG_ORDER ? SHV_MRG_ORDER == 2 : row_bytes > (512u << 10);
            fill_mrg_segments(h, P->seg_len, 1, P->nseg, P.get());
            CUtensorMap tmap;
            if (tma && !encode_rows_map(&tmap, dst, n, ns, (int)sizeof(T))) tma = false;
            if (tma) {
                Grid g{blocks_for(h, kKMrgFillTma, kind, true, P->items), h.tpb};
                err = launch_mrg_fill_tma(*P, tmap, kind, g, s);
            } else {
                Grid g{blocks_for(h, kKMrgFill, kind, vec, P->items), h.tpb};
                err = launch_mrg_fill(*P, kind, vec, g, s);
            }
        } else {
            const uint64_t E = kind == kF64 ? 4 : 8;
            const bool fast = aligned32 && (n % E == 0) && ((uint32_t)h.offset & 3) == 0;
            PhiloxLaunch P{};
            P.rpt = 1;
            P.keyed = h.spacing == SHV_SPACING_KEYED;
            P.k0 = h.seed[0];
            P.k1 = P.keyed ? h.seed[0] : h.seed[1];
            P.g0 = h.first + s0;
            P.ns = ns;
            P.o_blk = (uint64_t)(h.offset >> 2);
            P.o_lane = (uint32_t)(h.offset & 3);
            P.out = dst;
            P.n = n;
            Grid g{};
            if (fast) {
                const int kid = P.keyed ? kKPhiloxFillKeyed : kKPhiloxFill;
                counter_tasks(h, ns, n / E, resident_threads(h, kid, kind, true), &P.nseg, &P.items, &P.rpt);
                g = Grid{blocks_for(h, kid, kind, true, P.items * 32), h.tpb};
            } else {
                P.items = (ns * n + 7) / 8;
                g = Grid{blocks_for(h, P.keyed ? kKPhiloxFillKeyed : kKPhiloxFill, kind, false, P.items), h.tpb};
            }
            err = launch_philox_fill(P, kind, fast, g, s);
        }
        if (err != cudaSuccess) break;
        if (host_out) {
            err = cudaEventRecord(gen_done[k & 1], s);
            if (err == cudaSuccess) err = cudaStreamWaitEvent(cs, gen_done[k & 1], 0);
            if (err == cudaSuccess)
                err = cudaMemcpyAsync(reinterpret_cast<char*>(out) + s0 * row_bytes, dst, ns * row_bytes,
                                      cudaMemcpyDeviceToHost, cs);
            if (err == cudaSuccess) err = cudaEventRecord(copy_done[k & 1], cs);
        }
    }
    if (host_out) {
        // Completion is ordered on the caller's stream.
        for (int b = 0; b < 2; ++b) {
            if (err == cudaSuccess && h.n > (uint64_t)b * slice) err = cudaStreamWaitEvent(s, copy_done[b], 0);
            if (stage[b]) cudaFreeAsync(stage[b], s);
        }
        for (int b = 0; b < 2; ++b) {
            if (gen_done[b]) cudaEventDestroy(gen_done[b]);
            if (copy_done[b]) cudaEventDestroy(copy_done[b]);
        }
        if (cs) cudaStreamDestroy(cs);
    }
    if (err != cudaSuccess) return cuda_fail(err, "generate launch");
    h.offset += (u128)n * dpv;
    return SHV_OK;
}

shv_status validate_seed(int gen, const uint32_t* seed, size_t words, uint32_t out[6])
{
    memset(out, 0, 24);
    if (!seed) return fail(SHV_ERR_INVALID_ARGUMENT, "NULL seed");
    if (gen == SHV_GEN_MRG32K3A) {
        if (words == 1) {
            for (int k = 0; k < 6; ++k) out[k] = seed[0];
        } else if (words == 6) {
            memcpy(out, seed, 24);
        } else {
            return fail(SHV_ERR_INVALID_ARGUMENT, "MRG32k3a takes 1 or 6 seed words, got %zu", words);
        }
        for (int k = 0; k < 3; ++k)
            if (out[k] >= kM1 || out[3 + k] >= kM2)
                return fail(SHV_ERR_INVALID_SEED, "seed residue out of range (s1 < m1, s2 < m2)");
        if (!(out[0] | out[1] | out[2]) || !(out[3] | out[4] | out[5]))
            return fail(SHV_ERR_INVALID_SEED, "an all-zero MRG32k3a component never leaves zero");
        return SHV_OK;
    }
    if (gen == SHV_GEN_PHILOX4X32_10) {
        if (words != 1 && words != 2)
            return fail(SHV_ERR_INVALID_ARGUMENT, "Philox4x32-10 takes 1 or 2 key words, got %zu", words);
        out[0] = seed[0];
        out[1] = words == 2 ? seed[1] : 0;
        return SHV_OK;
    }
    if (gen == SHV_GEN_THREEFRY4X64_20) {
        if (words < 1 || words > 4)
            return fail(SHV_ERR_INVALID_ARGUMENT, "Threefry4x64-20 takes 1 to 4 key words, got %zu", words);
        for (size_t k = 0; k < words; ++k) out[k] = seed[k];
        return SHV_OK;
    }
    if (gen == SHV_GEN_TINYMT32)
        return fail(SHV_ERR_MISSING_PARAMETERS, "TinyMT32 handles come from shv_streams_create_tinymt32");
    if (gen == SHV_GEN_MTGP32)
        return fail(SHV_ERR_MISSING_PARAMETERS, "MTGP32 handles come from shv_streams_create_mtgp32");
    return fail(SHV_ERR_INVALID_ARGUMENT, "unknown generator %d", gen);
}

}  // namespace
}  // namespace shv

using namespace shv;

extern "C" {

size_t shv_state_bytes(int gen, uint64_t n_streams)
{
    const uint64_t per = gen == SHV_GEN_MRG32K3A ? 24 : gen == SHV_GEN_TINYMT32 ? 16
                       : gen == SHV_GEN_MTGP32 ? 4 * kMtgpStateWords : 0;
    if (!per || n_streams > SIZE_MAX / per) return 0;
    return (size_t)(per * n_streams);
}

shv_status shv_streams_create_tinymt32(shv_streams* out, const uint32_t* params, size_t n_params, uint32_t seed,
                                       uint32_t group_size, uint64_t first_stream, uint64_t n_streams, void* d_state,
                                       size_t state_bytes, int device, void* cuda_stream)
{
    Range nvtx_range("shv_streams_create_tinymt32");
    if (!out) return fail(SHV_ERR_INVALID_ARGUMENT, "NULL out handle");
    *out = 0;
    if (!params || n_params == 0)
        return fail(SHV_ERR_MISSING_PARAMETERS, "TinyMT32 needs Dynamic Creator parameter sets (P L304-306)");
    if (n_streams == 0) return fail(SHV_ERR_INVALID_ARGUMENT, "n_streams must be >= 1");
    if (group_size == 0 || (group_size & (group_size - 1)) || group_size > (1u << 16))
        return fail(SHV_ERR_INVALID_ARGUMENT, "group_size must be a power of two <= 2^16");
    const u128 end = (u128)first_stream + n_streams;
    if (end > ((u128)1 << 64)) return fail(SHV_ERR_INSUFFICIENT_STREAMS, "streams end at 2^64");
    const uint64_t g0 = first_stream / group_size, g1 = (uint64_t)((end - 1) / group_size);
    if (g1 >= n_params)
        return fail(SHV_ERR_INSUFFICIENT_STREAMS, "streams need %llu parameter sets, %zu given (one per group)",
                    (unsigned long long)(g1 + 1), n_params);
    const size_t need = shv_state_bytes(SHV_GEN_TINYMT32, n_streams);
    if (need == 0) return fail(SHV_ERR_INVALID_ARGUMENT, "state size overflow");
    if (d_state && state_bytes < need) return fail(SHV_ERR_INVALID_ARGUMENT, "state buffer %zu B < %zu B", state_bytes, need);
    if (d_state && ((uintptr_t)d_state & 3)) return fail(SHV_ERR_MISALIGNED, "state not 4-byte aligned");
    int dev = device;
    if (dev < 0) {
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    }
    DeviceGuard dg(dev);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    auto h = std::make_shared<Handle>();
    h->gen = SHV_GEN_TINYMT32;
    h->spacing = SHV_SPACING_STREAM;
    h->device = dev;
    h->seed[0] = seed;
    h->seed[1] = group_size;
    h->first = first_stream;
    h->n = n_streams;
    h->group0 = g0;
    h->group_size = group_size;
    cudaStream_t s = (cudaStream_t)cuda_stream;
    cudaError_t e = cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    const uint64_t ng = g1 - g0 + 1;
    e = cudaMalloc((void**)&h->params, 12 * ng);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(params)");
    e = cudaMemcpyAsync(h->params, params + 3 * g0, 12 * ng, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && d_state) {
        h->state = (uint32_t*)d_state;
    } else if (e == cudaSuccess) {
        e = cudaMalloc((void**)&h->state, need);
        h->own_state = e == cudaSuccess;
    }
    int log2_gs = 0;
    while ((1u << log2_gs) < group_size) ++log2_gs;
    uint32_t* tables = nullptr;
    if (e == cudaSuccess && log2_gs > 0) e = cudaMallocAsync((void**)&tables, (size_t)ng * log2_gs * 2048, s);
    if (e == cudaSuccess) e = launch_tinymt_prep(h->params, ng, log2_gs, tables, s);
    if (e == cudaSuccess) {
        TinyMtLaunch P = tm_launch(*h, 0, n_streams);
        e = launch_tinymt_seed(P, seed, tables, log2_gs, Grid{(unsigned)((n_streams + 255) / 256), 256}, s);
    }
    if (tables) cudaFreeAsync(tables, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // the host params copy must complete
    if (e != cudaSuccess) {
        if (h->own_state) cudaFree(h->state);
        cudaFree(h->params);
        return cuda_fail(e, "tinymt32 create");
    }
    const uint64_t id = g_next_id.fetch_add(1);
    {
        std::lock_guard<std::mutex> lk(g_mu);
        g_handles[id] = h;
    }
    *out = id;
    return SHV_OK;
}

shv_status shv_streams_create_mtgp32(shv_streams* out, const uint32_t* params, size_t n_params, uint64_t seed,
                                     uint64_t first_stream, uint64_t n_streams, void* d_state, size_t state_bytes,
                                     int device, void* cuda_stream)
{
    Range nvtx_range("shv_streams_create_mtgp32");
    if (!out) return fail(SHV_ERR_INVALID_ARGUMENT, "NULL out handle");
    *out = 0;
    if (!params || n_params == 0)
        return fail(SHV_ERR_MISSING_PARAMETERS, "MTGP32 needs Dynamic Creator parameter sets (P L74-76)");
    if (n_streams == 0) return fail(SHV_ERR_INVALID_ARGUMENT, "n_streams must be >= 1");
    if (first_stream >= n_params || n_streams > n_params - first_stream)
        return fail(SHV_ERR_INSUFFICIENT_STREAMS, "streams [%llu, %llu) need as many parameter sets, %zu given",
                    (unsigned long long)first_stream, (unsigned long long)(first_stream + n_streams), n_params);
    for (uint64_t g = first_stream; g < first_stream + n_streams; ++g) {
        const uint32_t* r = params + kMtgpParamWords * g;
        if (r[0] < 3 || r[0] > kMtgpN - 2 || r[1] > 31 || r[2] > 31)
            return fail(SHV_ERR_INVALID_ARGUMENT, "parameter set %llu: pos %u sh1 %u sh2 %u out of range",
                        (unsigned long long)g, r[0], r[1], r[2]);
    }
    const size_t need = shv_state_bytes(SHV_GEN_MTGP32, n_streams);
    if (need == 0) return fail(SHV_ERR_INVALID_ARGUMENT, "state size overflow");
    if (d_state && state_bytes < need) return fail(SHV_ERR_INVALID_ARGUMENT, "state buffer %zu B < %zu B", state_bytes, need);
    if (d_state && ((uintptr_t)d_state & 15)) return fail(SHV_ERR_MISALIGNED, "state not 16-byte aligned");
    int dev = device;
    if (dev < 0) {
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    }
    DeviceGuard dg(dev);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    auto h = std::make_shared<Handle>();
    h->gen = SHV_GEN_MTGP32;
    h->spacing = SHV_SPACING_STREAM;
    h->device = dev;
    h->seed[0] = (uint32_t)seed;
    h->seed[1] = (uint32_t)(seed >> 32);
    h->first = first_stream;
    h->n = n_streams;
    cudaStream_t s = (cudaStream_t)cuda_stream;
    cudaError_t e = cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    const size_t pbytes = 4 * kMtgpParamWords * n_streams;
    e = cudaMalloc((void**)&h->params, pbytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(params)");
    e = cudaMemcpyAsync(h->params, params + kMtgpParamWords * first_stream, pbytes, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && d_state) {
        h->state = (uint32_t*)d_state;
    } else if (e == cudaSuccess) {
        e = cudaMalloc((void**)&h->state, need);
        h->own_state = e == cudaSuccess;
    }
    if (e == cudaSuccess) e = launch_mtgp_seed(mtgp_launch(*h, 0, n_streams), (uint32_t)(seed ^ (seed >> 32)), s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // the host params copy must complete
    if (e != cudaSuccess) {
        if (h->own_state) cudaFree(h->state);
        cudaFree(h->params);
        return cuda_fail(e, "mtgp32 create");
    }
    const uint64_t id = g_next_id.fetch_add(1);
    {
        std::lock_guard<std::mutex> lk(g_mu);
        g_handles[id] = h;
    }
    *out = id;
    return SHV_OK;
}

shv_status shv_streams_create_ex(shv_streams* out, int gen, const uint32_t* seed, size_t seed_words,
                                 uint64_t first_stream, uint64_t n_streams, int spacing, void* d_state,
                                 size_t state_bytes, int device, void* cuda_stream)
{
    Range nvtx_range("shv_streams_create_ex");
    if (!out) return fail(SHV_ERR_INVALID_ARGUMENT, "NULL out handle");
    *out = 0;
    uint32_t s6[6];
    shv_status st = validate_seed(gen, seed, seed_words, s6);
    if (st) return st;
    if (n_streams == 0) return fail(SHV_ERR_INVALID_ARGUMENT, "n_streams must be >= 1");
    if (spacing != SHV_SPACING_STREAM && spacing != SHV_SPACING_SUBSTREAM && spacing != SHV_SPACING_KEYED)
        return fail(SHV_ERR_INVALID_ARGUMENT, "unknown spacing %d", spacing);
    if (gen == SHV_GEN_PHILOX4X32_10 && spacing == SHV_SPACING_SUBSTREAM)
        return fail(SHV_ERR_UNSUPPORTED, "Philox4x32-10 has no substreams");
    if (gen == SHV_GEN_THREEFRY4X64_20 && spacing != SHV_SPACING_STREAM)
        return fail(SHV_ERR_UNSUPPORTED, "Threefry4x64-20 supports counter-stream spacing only");
    if (gen == SHV_GEN_MRG32K3A && spacing == SHV_SPACING_KEYED)
        return fail(SHV_ERR_UNSUPPORTED, "MRG32k3a has no keys (use STREAM or SUBSTREAM spacing)");
    if (spacing == SHV_SPACING_KEYED && seed_words != 1)
        return fail(SHV_ERR_INVALID_ARGUMENT, "keyed Philox takes one seed word (the experiment tag)");
    const u128 end = (u128)first_stream + n_streams;
    if (spacing == SHV_SPACING_KEYED && end > ((u128)1 << 32))
        return fail(SHV_ERR_INSUFFICIENT_STREAMS, "key space exhausted: stream ids end at 2^32");
    if (gen == SHV_GEN_MRG32K3A && spacing == SHV_SPACING_SUBSTREAM && end > ((u128)1 << 51))
        return fail(SHV_ERR_INSUFFICIENT_STREAMS, "substreams end at 2^51 per stream");
    if (end > ((u128)1 << 64)) return fail(SHV_ERR_INSUFFICIENT_STREAMS, "streams end at 2^64");
    const size_t need = shv_state_bytes(gen, n_streams);
    if (gen == SHV_GEN_MRG32K3A) {
        if (need == 0) return fail(SHV_ERR_INVALID_ARGUMENT, "state size overflow");
        if (d_state && state_bytes < need)
            return fail(SHV_ERR_INVALID_ARGUMENT, "state buffer %zu B < %zu B", state_bytes, need);
        if (d_state && ((uintptr_t)d_state & 3)) return fail(SHV_ERR_MISALIGNED, "state not 4-byte aligned");
    }
    int dev = device;
    if (dev < 0) {
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    }
    DeviceGuard dg(dev);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");

    auto h = std::make_shared<Handle>();
    h->gen = gen;
    h->spacing = spacing;
    h->device = dev;
    memcpy(h->seed, s6, sizeof s6);
    h->first = first_stream;
    h->n = n_streams;
    cudaError_t e = cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");

    if (gen == SHV_GEN_MRG32K3A) {
        st = ensure_tables(dev);
        if (st) return st;
        if (d_state) {
            h->state = (uint32_t*)d_state;
        } else {
            e = cudaMalloc((void**)&h->state, need);
            if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(state)");
            h->own_state = true;
        }
        // Rank/handle base: seed jumped to stream (or substream) first_stream.
        uint32_t base[6];
        memcpy(base, s6, sizeof base);
        const MatPair B = pair_pow(first_stream, spacing == SHV_SPACING_STREAM ? 127 : 76);
        pair_apply(B, base);
        const int table = spacing == SHV_SPACING_STREAM ? 1 : 0;
        // 2^16 seeding threads (fewer for small n), each walking its streams
        // by the jump A^(T * spacing).
        const uint64_t T = n_streams < (1u << 16) ? (n_streams + 255) / 256 * 256 : (1u << 16);
        Grid g{(unsigned)(T / 256), 256};
        const MatPair step = pair_pow(T, spacing == SHV_SPACING_STREAM ? 127 : 76);
        e = launch_mrg_seed(h->state, n_streams, base, table, step, g, (cudaStream_t)cuda_stream);
        if (e != cudaSuccess) {
            if (h->own_state) cudaFree(h->state);
            return cuda_fail(e, "seed launch");
        }
    }
    const uint64_t id = g_next_id.fetch_add(1);
    {
        std::lock_guard<std::mutex> lk(g_mu);
        g_handles[id] = h;
    }
    *out = id;
    return SHV_OK;
}

shv_status shv_streams_create(shv_streams* out, int gen, const uint32_t* seed, size_t seed_words,
                              uint64_t n_streams)
{
    return shv_streams_create_ex(out, gen, seed, seed_words, 0, n_streams, SHV_SPACING_STREAM, nullptr, 0,
                                 -1, nullptr);
}

shv_status shv_streams_create_leapfrog(shv_streams* out, int gen, const uint32_t* seed, size_t seed_words,
                                       uint64_t players, uint64_t first_player, uint64_t n_players, void* d_state,
                                       size_t state_bytes, int device, void* cuda_stream)
{
    Range nvtx_range("shv_streams_create_leapfrog");
    if (!out) return fail(SHV_ERR_INVALID_ARGUMENT, "NULL out handle");
    *out = 0;
    if (gen == SHV_GEN_MTGP32) return fail(SHV_ERR_UNSUPPORTED, "MTGP32 has no Leap Frog layout (R18)");
    uint32_t s6[6] = {};
    shv_status st = SHV_OK;
    if (gen == SHV_GEN_TINYMT32) {  // R19: seed = {seed, mat1, mat2, tmat}
        if (!seed || seed_words != 4)
            return fail(SHV_ERR_MISSING_PARAMETERS, "TinyMT32 Leap Frog takes {seed, mat1, mat2, tmat}");
        memcpy(s6, seed, 16);
    } else {
        st = validate_seed(gen, seed, seed_words, s6);
        if (st) return st;
    }
    if (players == 0) return fail(SHV_ERR_INVALID_ARGUMENT, "players must be >= 1");
    if (n_players == 0) return fail(SHV_ERR_INVALID_ARGUMENT, "n_players must be >= 1");
    if ((u128)first_player + n_players > players)
        return fail(SHV_ERR_INSUFFICIENT_STREAMS, "players [%llu, %llu) beyond K = %llu",
                    (unsigned long long)first_player, (unsigned long long)(first_player + n_players),
                    (unsigned long long)players);
    const size_t need = shv_state_bytes(SHV_GEN_MRG32K3A, n_players);
    if (gen == SHV_GEN_MRG32K3A) {
        if (need == 0) return fail(SHV_ERR_INVALID_ARGUMENT, "state size overflow");
        if (d_state && state_bytes < need)
            return fail(SHV_ERR_INVALID_ARGUMENT, "state buffer %zu B < %zu B", state_bytes, need);
        if (d_state && ((uintptr_t)d_state & 3)) return fail(SHV_ERR_MISALIGNED, "state not 4-byte aligned");
    }
    int dev = device;
    if (dev < 0) {
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    }
    DeviceGuard dg(dev);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    auto h = std::make_shared<Handle>();
    h->gen = gen;
    h->spacing = SHV_SPACING_LEAPFROG;
    h->device = dev;
    memcpy(h->seed, s6, sizeof s6);
    h->first = first_player;
    h->n = n_players;
    h->players = players;
    cudaError_t e = cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    if (gen == SHV_GEN_TINYMT32) {
        e = cudaMalloc((void**)&h->params, kTmLeapBufWords * 4);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(tinymt leap tables)");
        e = cudaMemcpyAsync(h->params, s6 + 1, 12, cudaMemcpyHostToDevice, (cudaStream_t)cuda_stream);
        if (e == cudaSuccess) e = launch_tm_leap_prep(h->params, players, s6[0], (cudaStream_t)cuda_stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)cuda_stream);  // host params copy
        if (e != cudaSuccess) {
            cudaFree(h->params);
            return cuda_fail(e, "tinymt leap prep");
        }
    }
    if (gen == SHV_GEN_MRG32K3A) {
        st = ensure_tables(dev);
        if (st) return st;
        if (d_state) {
            h->state = (uint32_t*)d_state;
        } else {
            e = cudaMalloc((void**)&h->state, need);
            if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(state)");
            h->own_state = true;
        }
        // Player p's base state A^p * seed: base A^first * seed, then per-bit
        // single-draw tables (table 2) and the stride jump A^T.
        uint32_t base[6];
        memcpy(base, s6, sizeof base);
        pair_apply(pair_pow(first_player, 0), base);
        const uint64_t T = n_players < (1u << 16) ? (n_players + 255) / 256 * 256 : (1u << 16);
        e = launch_mrg_seed(h->state, n_players, base, 2, pair_pow(T, 0), Grid{(unsigned)(T / 256), 256},
                            (cudaStream_t)cuda_stream);
        if (e != cudaSuccess) {
            if (h->own_state) cudaFree(h->state);
            return cuda_fail(e, "seed launch");
        }
    }
    const uint64_t id = g_next_id.fetch_add(1);
    {
        std::lock_guard<std::mutex> lk(g_mu);
        g_handles[id] = h;
    }
    *out = id;
    return SHV_OK;
}

// TinyMT32 jumps of at most this many draws step the generator (cheaper
// than the <= 128-step polynomial jump plus its per-group setup).
constexpr uint64_t kTinyStepJumpMax = 256;

shv_status shv_jump(shv_streams hid, int kind, uint64_t n, void* stream)
{
    Range nvtx_range("shv_jump");
    auto hp = lookup(hid);
    if (!hp) return fail(SHV_ERR_LIFECYCLE, "unknown or destroyed handle");
    Handle& h = *hp;
    u128 d;
    if (h.gen == SHV_GEN_MTGP32) {
        // sequential advance on the device (no jump polynomial), on the caller's stream
        if (kind != SHV_JUMP_DRAWS) return fail(SHV_ERR_UNSUPPORTED, "MTGP32 jumps by draws only");
        if (n == 0) return SHV_OK;
        shv_status st = check_advance(h, n);
        if (st) return st;
        DeviceGuard dg(h.device);
        if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
        MtgpLaunch P = mtgp_launch(h, 0, h.n);
        P.n = n;
        cudaError_t e = launch_mtgp(P, 4, mtgp_blocks(h, h.n), (cudaStream_t)stream);
        if (e != cudaSuccess) return cuda_fail(e, "mtgp32 advance");
        h.offset += n;
        return SHV_OK;
    }
    if (h.gen == SHV_GEN_TINYMT32 && h.spacing != SHV_SPACING_LEAPFROG) {
        // stateful: the state buffer advances on the caller's stream; short
        // jumps step (S L355), longer ones apply the jump polynomial x^n mod
        // the minimal polynomial of each parameter set's orbit (deg <= 128)
        if (kind != SHV_JUMP_DRAWS) return fail(SHV_ERR_UNSUPPORTED, "TinyMT32 jumps by draws only");
        if (n == 0) return SHV_OK;
        shv_status st = check_advance(h, n);
        if (st) return st;
        DeviceGuard dg(h.device);
        if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
        TinyMtLaunch P = tm_launch(h, 0, h.n);
        cudaStream_t s = (cudaStream_t)stream;
        cudaError_t e;
        if (n <= kTinyStepJumpMax) {
            P.steps = n;
            e = launch_tinymt_advance(P, Grid{(unsigned)((h.n + 255) / 256), 256}, s);
        } else {
            const uint64_t ngroups = (h.first + h.n - 1) / h.group_size - h.first / h.group_size + 1;
            uint32_t* poly = nullptr;
            e = cudaMallocAsync((void**)&poly, 16 * ngroups, s);
            if (e == cudaSuccess) e = launch_tinymt_jump(P, n, poly, s);
            if (poly) {
                const cudaError_t ef = cudaFreeAsync(poly, s);
                if (e == cudaSuccess) e = ef;
            }
        }
        if (e != cudaSuccess) return cuda_fail(e, "tinymt jump");
        h.offset += n;
        return SHV_OK;
    }
    if (kind == SHV_JUMP_DRAWS) {
        d = n;
    } else if (kind == SHV_JUMP_SUBSTREAMS || kind == SHV_JUMP_STREAMS) {
        if (h.spacing == SHV_SPACING_LEAPFROG) return fail(SHV_ERR_UNSUPPORTED, "Leap Frog players jump by draws only");
        if (h.gen != SHV_GEN_MRG32K3A) return fail(SHV_ERR_UNSUPPORTED, "counter-based generators jump by draws only");
        const int sh = kind == SHV_JUMP_SUBSTREAMS ? 76 : 127;
        if (n >> (128 - sh)) return fail(SHV_ERR_INVALID_ARGUMENT, "jump exceeds 2^128 draws");
        d = (u128)n << sh;
    } else {
        return fail(SHV_ERR_INVALID_ARGUMENT, "unknown jump kind %d", kind);
    }
    shv_status st = check_advance(h, d);
    if (st) return st;
    h.offset += d;
    return SHV_OK;
}

shv_status shv_generate_u32(shv_streams h, uint32_t* d_out, uint64_t n, void* s)
{
    return generate<uint32_t>(h, d_out, n, s, kU32, false);
}
shv_status shv_generate_f32(shv_streams h, float* d_out, uint64_t n, void* s)
{
    return generate<float>(h, d_out, n, s, kF32, false);
}
shv_status shv_generate_f64(shv_streams h, double* d_out, uint64_t n, void* s)
{
    return generate<double>(h, d_out, n, s, kF64, false);
}
shv_status shv_generate_u32_host(shv_streams h, uint32_t* h_out, uint64_t n, void* s)
{
    return generate<uint32_t>(h, h_out, n, s, kU32, true);
}
shv_status shv_mc_pi_ex(shv_streams hid, uint64_t samples, uint64_t* d_hits, uint64_t* d_counts,
                        void* stream)
{
    Range nvtx_range("shv_mc_pi_ex");
    auto hp = lookup(hid);
    if (!hp) return fail(SHV_ERR_LIFECYCLE, "unknown or destroyed handle");
    Handle& h = *hp;
    if (samples == 0) return fail(SHV_ERR_EMPTY_EXPERIMENT, "zero samples per stream");
    if (!d_hits) return fail(SHV_ERR_INVALID_ARGUMENT, "NULL d_hits");
    if (((uintptr_t)d_hits & 7) || ((uintptr_t)d_counts & 7)) return fail(SHV_ERR_MISALIGNED, "counters not 8-byte aligned");
    if (samples > (UINT64_MAX >> 2)) return fail(SHV_ERR_INVALID_ARGUMENT, "samples too large");
    shv_status st = check_advance(h, (u128)samples * 2);
    if (st) return st;
    DeviceGuard dg(h.device);
    if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t err;
    const uint64_t cap = 1ull << 31;  // per-item count fits in u32
    if (h.spacing == SHV_SPACING_LEAPFROG && h.gen == SHV_GEN_TINYMT32) {
        TmLeapLaunch P{};
        P.buf = h.params;
        P.players = h.players;
        P.first = h.first;
        P.ns = h.n;
        P.o_lo = (uint64_t)h.offset;
        P.o_hi = (uint64_t)(h.offset >> 64);
        P.n = samples;
        P.hits = (unsigned long long*)d_hits;
        P.counts = (unsigned long long*)d_counts;
        uint32_t nseg = 1;
        split(h, h.n, samples, 1, 8, (uint64_t)h.sms * 2048, cap, &P.seg_len, &nseg, 64);
        P.seg_draws = P.seg_len * 2;
        P.items = h.n * nseg;
        Grid g{(unsigned)std::min<uint64_t>((P.items + 255) / 256, (uint64_t)h.sms * 8), 256};
        err = launch_tm_leap(P, 3, g, s);
    } else if (h.spacing == SHV_SPACING_LEAPFROG) {
        const int lg = leap_gen(h.gen);
        const int kid = leap_kernel_id(kKLeapMc, lg);
        auto P = leap_launch(h, 0, h.n, samples, 2, 1, resident_threads(h, kid, 0, true));
        P->hits = (unsigned long long*)d_hits;
        P->counts = (unsigned long long*)d_counts;
        Grid g{blocks_for(h, kid, 0, true, P->items), h.tpb};
        err = launch_leap_mc(*P, lg, g, s);
    } else if (h.gen == SHV_GEN_THREEFRY4X64_20) {
        const bool fast = ((uint32_t)h.offset & 7) == 0;
        ThreefryLaunch P{};
        P.k0 = (uint64_t)h.seed[0] | ((uint64_t)h.seed[1] << 32);
        P.k1 = (uint64_t)h.seed[2] | ((uint64_t)h.seed[3] << 32);
        P.g0 = h.first;
        P.ns = h.n;
        P.o_blk = (uint64_t)(h.offset >> 3);
        P.o_word = (uint32_t)(h.offset & 7);
        P.n = samples;
        P.hits = (unsigned long long*)d_hits;
        P.counts = (unsigned long long*)d_counts;
        split(h, h.n, samples, 4, 32, resident_threads(h, kKThreefryMc, 0, fast), cap, &P.seg_len, &P.nseg);
        P.items = h.n * P.nseg;
        Grid g{blocks_for(h, kKThreefryMc, 0, fast, P.items), h.tpb};
        err = launch_threefry_mc(P, fast, g, s);
    } else if (h.gen == SHV_GEN_MTGP32) {
        MtgpLaunch P = mtgp_launch(h, 0, h.n);
        P.n = samples;
        P.hits = (unsigned long long*)d_hits;
        P.counts = (unsigned long long*)d_counts;
        err = launch_mtgp(P, 3, mtgp_blocks(h, h.n), s);
    } else if (h.gen == SHV_GEN_TINYMT32) {
        TinyMtLaunch P = tm_launch(h, 0, h.n);
        P.n = samples;
        P.hits = (unsigned long long*)d_hits;
        P.counts = (unsigned long long*)d_counts;
        Grid g{(unsigned)((h.n + h.tpb - 1) / h.tpb), h.tpb};
        err = launch_tinymt_mc(P, g, s);
    } else if (h.gen == SHV_GEN_MRG32K3A) {
        auto P = std::make_unique<MrgLaunch>();
        P->state = h.state;
        P->stride = h.n;
        P->stream_begin = 0;
        P->ns = h.n;
        P->out = nullptr;
        P->n = samples;
        P->hits = (unsigned long long*)d_hits;
        P->counts = (unsigned long long*)d_counts;
        split(h, h.n, samples, 2, 32, resident_threads(h, kKMrgMc, 0, true), cap, &P->seg_len, &P->nseg);
        P->items = h.n * P->nseg;
        fill_mrg_segments(h, P->seg_len, 2, P->nseg, P.get());
        Grid g{blocks_for(h, kKMrgMc, 0, true, P->items), h.tpb};
        err = launch_mrg_mc(*P, g, s);
    } else {
        const bool fast = ((uint32_t)h.offset & 3) == 0;
        PhiloxLaunch P{};
        P.keyed = h.spacing == SHV_SPACING_KEYED;
        P.k0 = h.seed[0];
        P.k1 = P.keyed ? h.seed[0] : h.seed[1];
        P.g0 = h.first;
        P.ns = h.n;
        P.o_blk = (uint64_t)(h.offset >> 2);
        P.o_lane = (uint32_t)(h.offset & 3);
        P.n = samples;
        P.hits = (unsigned long long*)d_hits;
        P.counts = (unsigned long long*)d_counts;
        const int kid = P.keyed ? kKPhiloxMcKeyed : kKPhiloxMc;
        split(h, h.n, samples, 2, 32, resident_threads(h, kid, 0, fast), cap, &P.seg_len, &P.nseg);
        P.items = h.n * P.nseg;
        Grid g{blocks_for(h, kid, 0, fast, P.items), h.tpb};
        err = launch_philox_mc(P, fast, g, s);
    }
    if (err != cudaSuccess) return cuda_fail(err, "mc_pi launch");
    h.offset += (u128)samples * 2;
    return SHV_OK;
}

shv_status shv_mc_pi(shv_streams h, uint64_t samples, uint64_t* d_hits, void* s)
{
    return shv_mc_pi_ex(h, samples, d_hits, nullptr, s);
}

shv_status shv_get_position(shv_streams hid, shv_position* out)
{
    auto hp = lookup(hid);
    if (!hp) return fail(SHV_ERR_LIFECYCLE, "unknown or destroyed handle");
    if (!out) return fail(SHV_ERR_INVALID_ARGUMENT, "NULL out");
    const Handle& h = *hp;
    out->gen = (uint32_t)h.gen;
    out->spacing = (uint32_t)h.spacing;
    memcpy(out->seed, h.seed, sizeof out->seed);
    out->first_stream = h.first;
    out->n_streams = h.n;
    out->offset_lo = (uint64_t)h.offset;
    out->offset_hi = (uint64_t)(h.offset >> 64);
    out->players = h.players;
    return SHV_OK;
}

shv_status shv_get_device_view(shv_streams hid, shv_device_view* out)
{
    Range nvtx_range("shv_get_device_view");
    auto hp = lookup(hid);
    if (!hp) return fail(SHV_ERR_LIFECYCLE, "unknown or destroyed handle");
    if (!out) return fail(SHV_ERR_INVALID_ARGUMENT, "NULL out");
    const Handle& h = *hp;
    if (h.spacing == SHV_SPACING_LEAPFROG) return fail(SHV_ERR_UNSUPPORTED, "no device view for Leap Frog handles");
    if (h.gen == SHV_GEN_MTGP32)
        return fail(SHV_ERR_UNSUPPORTED, "no per-thread device view for MTGP32 (block-cooperative generator)");
    memset(out, 0, sizeof *out);
    out->gen = (uint32_t)h.gen;
    out->spacing = (uint32_t)h.spacing;
    out->key0 = h.seed[0];
    out->key1 = h.spacing == SHV_SPACING_KEYED ? h.seed[0] : h.seed[1];
    out->key2 = h.seed[2];
    out->key3 = h.seed[3];
    out->first_stream = h.first;
    out->n_streams = h.n;
    out->offset_lo = (uint64_t)h.offset;
    out->offset_hi = (uint64_t)(h.offset >> 64);
    if (h.gen == SHV_GEN_TINYMT32) {
        out->state = h.state;  // current states (stateful handle)
        out->params = h.params;
        out->group0 = h.group0;
        out->group_size = h.group_size;
    } else if (h.gen == SHV_GEN_MRG32K3A) {
        out->state = h.state;
        const MatPair J = pair_pow(h.offset, 0);
        memcpy(out->jump, J.a, 36);
        memcpy(out->jump + 9, J.b, 36);
    }
    return SHV_OK;
}

shv_status shv_streams_destroy(shv_streams hid)
{
    Range nvtx_range("shv_streams_destroy");
    std::shared_ptr<Handle> h;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_handles.find(hid);
        if (it == g_handles.end()) return fail(SHV_ERR_LIFECYCLE, "unknown or already destroyed handle");
        h = it->second;
        g_handles.erase(it);
    }
    if ((h->own_state && h->state) || h->params) {
        DeviceGuard dg(h->device);
        if (h->own_state && h->state) cudaFree(h->state);
        if (h->params) cudaFree(h->params);
    }
    return SHV_OK;
}

shv_status shv_set_launch_config(shv_streams hid, uint32_t bps, uint32_t tpb, uint64_t seg)
{
    auto hp = lookup(hid);
    if (!hp) return fail(SHV_ERR_LIFECYCLE, "unknown or destroyed handle");
    if (tpb == 0) tpb = 256;
    if (tpb % 32 || tpb > 256) return fail(SHV_ERR_INVALID_ARGUMENT, "threads_per_block must be 32..256, multiple of 32");
    if (seg % 8) return fail(SHV_ERR_INVALID_ARGUMENT, "segment must be a multiple of 8");
    if (bps > 64) return fail(SHV_ERR_INVALID_ARGUMENT, "blocks_per_sm too large");
    hp->bps = bps;
    hp->tpb = tpb;
    hp->seg = seg;
    return SHV_OK;
}

static uint64_t audit_windows(uint64_t n_pe, uint64_t horizon)
{
    return horizon < 4 ? 0 : n_pe * (horizon - 3);
}

size_t shv_verify_disjoint_workspace_bytes(uint64_t n_pe, uint64_t horizon)
{
    if (n_pe && horizon > (((uint64_t)1 << 40) - 2) / n_pe) return 0;
    const uint64_t w = audit_windows(n_pe, horizon);
    return w ? (size_t)8 * audit_workspace_words(w) : 0;
}

shv_status shv_verify_disjoint(const uint32_t* d_rows, uint64_t n_pe, uint64_t horizon, void* d_ws,
                               size_t ws_bytes, shv_disjoint_report* d_report, void* stream)
{
    Range nvtx_range("shv_verify_disjoint");
    if (!d_report) return fail(SHV_ERR_INVALID_ARGUMENT, "NULL d_report");
    if ((uintptr_t)d_report & 7) return fail(SHV_ERR_MISALIGNED, "d_report not 8-byte aligned");
    if (n_pe && horizon > (((uint64_t)1 << 40) - 2) / n_pe)
        return fail(SHV_ERR_INVALID_ARGUMENT, "n_pe * horizon must be below 2^40 - 1");
    AuditLaunch P{};
    P.rows = d_rows;
    P.horizon = horizon;
    P.wpr = horizon < 4 ? 0 : horizon - 3;
    P.windows = audit_windows(n_pe, horizon);
    P.report = d_report;
    if (P.windows) {
        if (!d_rows || !d_ws) return fail(SHV_ERR_INVALID_ARGUMENT, "NULL d_rows or d_workspace");
        if ((uintptr_t)d_ws & 7) return fail(SHV_ERR_MISALIGNED, "d_workspace not 8-byte aligned");
        const uint64_t words = audit_workspace_words(P.windows);
        if (ws_bytes / 8 < words)
            return fail(SHV_ERR_INVALID_ARGUMENT, "workspace of %zu bytes; %llu windows need %llu",
                        ws_bytes, (unsigned long long)P.windows, (unsigned long long)(8 * words));
        P.lgb = audit_lg_buckets(P.windows);
        P.nb = 1u << P.lgb;
        unsigned long long* w = (unsigned long long*)d_ws;
        P.scratch = w;
        P.count = w + 6;
        P.rec_off = P.count + P.nb;
        P.cursor = P.rec_off + P.nb;
        P.tab_off = P.cursor + P.nb;
        P.rec = P.tab_off + P.nb;
        P.slots = P.rec + 2 * P.windows;
        P.cand = P.slots + 2 * P.windows + P.nb;
    }
    int dev = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_fail(e, "device query");
    const uint64_t want = (P.windows + 255) / 256;
    const unsigned blocks = (unsigned)(want < (uint64_t)sms * 8 ? (want ? want : 1) : (uint64_t)sms * 8);
    e = launch_audit(P, blocks, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "verify_disjoint launch");
    return SHV_OK;
}

const char* shv_status_string(shv_status s)
{
    switch (s) {
    case SHV_OK: return "SHV_OK";
    case SHV_ERR_INVALID_ARGUMENT: return "SHV_ERR_INVALID_ARGUMENT";
    case SHV_ERR_INVALID_SEED: return "SHV_ERR_INVALID_SEED";
    case SHV_ERR_INSUFFICIENT_STREAMS: return "SHV_ERR_INSUFFICIENT_STREAMS";
    case SHV_ERR_UNSUPPORTED: return "SHV_ERR_UNSUPPORTED";
    case SHV_ERR_LIFECYCLE: return "SHV_ERR_LIFECYCLE";
    case SHV_ERR_MISALIGNED: return "SHV_ERR_MISALIGNED";
    case SHV_ERR_EMPTY_EXPERIMENT: return "SHV_ERR_EMPTY_EXPERIMENT";
    case SHV_ERR_MISSING_PARAMETERS: return "SHV_ERR_MISSING_PARAMETERS";
    case SHV_ERR_CUDA: return "SHV_ERR_CUDA";
    }
    return "SHV_ERR_UNKNOWN";
}

const char* shv_last_error_message(void) { return t_err.c_str(); }

shv_status shv_partition(uint64_t total, int rank, int world, uint64_t* first, uint64_t* count)
{
    if (!first || !count) return fail(SHV_ERR_INVALID_ARGUMENT, "NULL out");
    if (world < 1 || rank < 0 || rank >= world) return fail(SHV_ERR_INVALID_ARGUMENT, "bad rank/world");
    const uint64_t lo = (uint64_t)(((u128)total * (uint64_t)rank) / (uint64_t)world);
    const uint64_t hi = (uint64_t)(((u128)total * (uint64_t)(rank + 1)) / (uint64_t)world);
    *first = lo;
    *count = hi - lo;
    return SHV_OK;
}

shv_status shv_jump_matrix(uint64_t e_lo, uint64_t e_hi, uint32_t out[18])
{
    if (!out) return fail(SHV_ERR_INVALID_ARGUMENT, "NULL out");
    const MatPair P = pair_pow(((u128)e_hi << 64) | e_lo, 0);
    memcpy(out, P.a, 36);
    memcpy(out + 9, P.b, 36);
    return SHV_OK;
}

const char* shv_build_info(void) { return "shv 0.1 sm_100a"; }

}  // extern "C"
