// shv_internal.h — launch records shared by the ABI layer (shv_api.cpp) and the
// sm_100a kernels (kernels_*.cu). Not installed; the public ABI is include/shv.h.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>  // CUtensorMap (types only; the encoder comes from cudaGetDriverEntryPoint)
#include <cuda_runtime.h>

#include "../../include/shv.h"  // shv_disjoint_report

namespace shv {

// Intra-stream Sequence Splitting (P L109-112 [§2.3]): a launch splits each
// row into up to 2^kSegBits segments; segment j starts j segment lengths
// later, reached through per-bit jump tables in the kernel parameter block
// (72 B per entry).
constexpr int kSegBits = 32;

// Output kinds.
enum Kind : int { kU32 = 0, kF32 = 1, kF64 = 2 };

// A 3x3 jump matrix pair, row-major: a = A1^e mod m1, b = A2^e mod m2.
struct MatPair {
    uint32_t a[9];
    uint32_t b[9];
};

// MRG32k3a bulk fill / Monte Carlo launch. Work item it in [0, items):
// segment j = it / ns, stream i = it % ns (streams fastest so a warp shares
// one segment matrix), or i = it / nseg, j = it % nseg with seg_fastest. Segment j covers values [j*seg_len, min(n,(j+1)*seg_len))
// of the row and starts from (prod over set bits b of j of segpow[b]) * seg0 * state_i.
struct MrgLaunch {
    const uint32_t* state;   // SoA: word k of stream s at state[k*stride + s]
    uint64_t stride;         // handle n_streams
    uint64_t stream_begin;   // first handle stream of this launch (host slices)
    uint64_t ns;             // streams in this launch
    void* out;               // fill: row i at out + i*n (elements); MC: unused
    uint64_t n;              // fill: values per row; MC: samples per stream
    uint64_t seg_len;        // values (fill) or samples (MC) per segment
    uint64_t items;          // ns * nseg
    unsigned long long* hits;    // MC only
    unsigned long long* counts;  // MC only, optional (indexed by launch stream)
    uint32_t nseg;
    uint32_t seg_fastest;    // 1: work item it -> (i = it / nseg, j = it % nseg)
    MatPair seg0;                 // A^o (o = handle offset)
    MatPair segpow[kSegBits];     // (A^(seg_len * draws per unit))^(2^b)
    double fpk[6];                // FP64 step constants (shv::dev::MrgFpK order), set by
                                  // fill_mrg_segments: read from the parameter block so
                                  // ptxas keeps them in registers
    uint32_t imul[2];             // a12, a13n (MrgFpK::a12/a13n): runtime values, so ptxas
                                  // emits plain IMAD.WIDE for the integer half-step
    double snk[5];                // subnormal-state step constants (MrgFpK::sn_c1q .. sn_M)
};

// Philox4x32-10 bulk fill / Monte Carlo launch. Draw d of handle stream i
// (d counted from the handle offset o = 4*o_blk + o_lane) is lane
// (o_lane + d) & 3 of counter block o_blk + ((o_lane + d) >> 2) with
// ctr = (blk_lo, blk_hi, g_lo, g_hi), g = g0 + i, key = (k0, k1) (R6); with
// keyed = 1 instead key = (g0 + i, k1) and ctr = (blk_lo, blk_hi, 0, 0).
struct PhiloxLaunch {
    uint32_t k0, k1;
    uint64_t g0;             // family stream of launch stream 0
    uint64_t ns;             // streams in this launch
    uint64_t o_blk;          // offset / 4
    uint32_t o_lane;         // offset % 4
    void* out;
    uint64_t n;              // fill: values per row; MC: samples per stream
    uint64_t seg_len;        // MC: samples per work item
    uint64_t items;          // fill: warp tasks; MC: ns * nseg
    uint32_t nseg;           // fill fast path: chunks per lane per row (R); MC: segments
    uint32_t rpt;            // fill fast path: whole rows per warp task (>= 1)
    unsigned long long* hits;
    unsigned long long* counts;
    uint32_t keyed;          // 1: key = (g0 + i, k1), ctr[2..3] = 0 (SHV_SPACING_KEYED)
};

// Threefry4x64-20 launch (NEXT-2; R16). Draw d of launch stream i is word
// (o_word + d) & 7 of block o_blk + ((o_word + d) >> 3), ctr = (blk, g0 + i, 0, 0),
// key = (k0, k1, 0, 0); words are (lo, hi) of the four 64-bit lanes.
struct ThreefryLaunch {
    uint64_t k0, k1;
    uint64_t g0;
    uint64_t ns;
    uint64_t o_blk;
    uint32_t o_word;
    uint32_t nseg;            // fill fast path: chunks per lane per task (R); MC: segments
    void* out;
    uint64_t n;
    uint64_t seg_len;         // MC: samples per work item
    uint64_t items;
    unsigned long long* hits;
    unsigned long long* counts;
};

// TinyMT32 launch (NEXT-3; R15). Stateful: the SoA state buffer holds every
// stream's current state and each launch writes it back. Family stream
// g = first + i belongs to group g / group_size, whose parameter set is
// params[3 * (g / group_size - group0) ..].
struct TinyMtLaunch {
    uint32_t* state;          // SoA: word k of stream i at state[k*stride + i]
    uint64_t stride;          // handle n_streams
    uint64_t ns;              // streams in this launch (from stream 0)
    const uint32_t* params;   // (mat1, mat2, tmat) per group from group0
    uint64_t first;
    uint64_t group0;
    uint32_t group_size;
    void* out;                // fill: row i at out + i*n elements
    uint64_t n;               // values per row (fill) or samples (MC)
    uint64_t steps;           // advance kernel: draws to skip
    unsigned long long* hits;
    unsigned long long* counts;
};

// Leap Frog launch (NEXT-4; R17). Work item it in [0, items): segment
// j = it / ns, row i = it % ns (player p = first + i). Segment j covers values
// [j*seg_len, min(n, (j+1)*seg_len)) of the row, i.e. player draws from
// o + j*seg_len*dpv (dpv = draws per value, 2 for counter-based f64 and MC).
enum LeapGen : int { kLeapMrg = 0, kLeapPhilox = 1, kLeapThreefry = 2 };
struct LeapLaunch {
    uint64_t players;            // K
    uint64_t first;              // player id of launch row 0
    uint64_t ns;                 // rows in this launch
    uint64_t o_lo, o_hi;         // counter-based: player draw offset o (u128)
    uint64_t seg_draws;          // counter-based: player draws per segment
    void* out;
    uint64_t n;                  // fill: values per row; MC: samples per row
    uint64_t seg_len;            // values (fill) or samples (MC) per segment
    uint64_t items;              // ns * nseg
    unsigned long long* hits;    // MC only
    unsigned long long* counts;  // MC only, optional (indexed by launch row)
    uint64_t k0, k1;             // Philox: key (k0, k1) (32-bit); Threefry: key lanes 0, 1
    // Philox grouped mode (K % 4 == 0; ngroups != 0): work item = (group g0+g,
    // segment j), g fastest; group G holds players 4G .. 4G+3.
    uint64_t g0, ngroups;
    // MRG32k3a: state[k*stride + stream_begin + i] = word k of A^p * seed.
    const uint32_t* state;
    uint64_t stride;
    uint64_t stream_begin;
    uint32_t cp1[3], cp2[3];     // u_{t+3} = cp[2] u_{t+2} + cp[1] u_{t+1} + cp[0] u_t (mod m1 / m2)
    MatPair B;                   // A^K
    MatPair start;               // A^(1 + K*o)
    MatPair segpow[kSegBits];  // (A^(K*seg_draws))^(2^b); transposed mode: (A^K)^(2^b)
    // MRG32k3a transposed mode (u32/f32): out[p][t] = base draw (first+p) + K*(o+t)
    // is the transpose of the base sequence laid out as [t][p]; a lane steps
    // one t-row through consecutive players (leap_mrg_tr_kernel).
    uint32_t tr_s0[6];           // A^(first + K*o) seed
    uint64_t tr_tb, tr_ps, tr_pl;  // t-blocks of 32, player segments, players per segment (% 128 == 0)
    MatPair tr_ppow[kSegBits];   // (A^tr_pl)^(2^b)
    double fpk[6];               // FP64 step constants (shv::dev::MrgFpK order)
    uint32_t imul[2];            // a12, a13n (as MrgLaunch::imul)
};

struct Grid {
    unsigned blocks;
    unsigned threads;
};


// ---- launchers (kernels_mrg.cu, kernels_philox.cu, kernels_threefry.cu, kernels_tinymt32.cu,
//      kernels_leapfrog.cu) ----
// TinyMT32: tables[g][b] = (T_g^(2^64))^(2^b), 128 columns x 4 words each.
cudaError_t launch_threefry_fill(const ThreefryLaunch& p, int kind, bool fast, Grid g, cudaStream_t s);
cudaError_t launch_threefry_mc(const ThreefryLaunch& p, bool fast, Grid g, cudaStream_t s);
cudaError_t launch_tinymt_prep(const uint32_t* params, uint64_t n_groups, int log2_gs, uint32_t* tables,
                               cudaStream_t s);
cudaError_t launch_tinymt_seed(const TinyMtLaunch& p, uint32_t seed, const uint32_t* tables, int log2_gs,
                               Grid g, cudaStream_t s);
cudaError_t launch_tinymt_fill(const TinyMtLaunch& p, int kind, bool vec, Grid g, cudaStream_t s);
cudaError_t launch_tinymt_advance(const TinyMtLaunch& p, Grid g, cudaStream_t s);
// Jump every stream of p (p.ns from stream 0) by n draws with the jump
// polynomial x^n mod (minimal polynomial of the group's orbit); d_poly:
// 16 bytes of device scratch per parameter set the launch touches.
cudaError_t launch_tinymt_jump(const TinyMtLaunch& p, uint64_t n, uint32_t* d_poly, cudaStream_t s);
cudaError_t launch_tinymt_mc(const TinyMtLaunch& p, Grid g, cudaStream_t s);
cudaError_t upload_jump_tables(const MatPair* sub51, const MatPair* str64, const MatPair* draw64);
// T = g.blocks * g.threads seeding threads; step = A^(T * spacing); table 0
// substreams, 1 streams, 2 single draws (Leap Frog players).
cudaError_t launch_mrg_seed(uint32_t* state, uint64_t n, const uint32_t base[6], int table,
                            const MatPair& step, Grid g, cudaStream_t s);
cudaError_t launch_mrg_fill(const MrgLaunch& p, int kind, bool vec, Grid g, cudaStream_t s);
// MRG32k3a fill with TMA stores: `tmap` is a 2D map of the launch's rows
// (dim0 = n values, dim1 = ns rows, box 128 B x 32 rows, 128-B swizzle);
// needs seg_len % (128 / value bytes) == 0, n and ns < 2^31.
cudaError_t launch_mrg_fill_tma(const MrgLaunch& p, const CUtensorMap& tmap, int kind, Grid g, cudaStream_t s);
size_t mrg_fill_tma_smem(int threads);
bool mrg_fill_tma_fits(int threads);  // dynamic shared memory of a block within the 227-KB limit
cudaError_t launch_mrg_mc(const MrgLaunch& p, Grid g, cudaStream_t s);
// MRG32k3a fill in row tiles (u32/f32): m.seg_len = S, m.nseg = n / S (S * nseg = n,
// S % 4 == 0), items = ns * nseg; lanetab[k] = A^(o + k S) for k < min(32, nseg),
// m.segpow[b] = (A^(32 S))^(2^b) (per-bit tables of the tile index within a row). `tmap`: 2D map of [ns * nseg][S] values, box
// 128 B x 32 rows, 128-B swizzle.
struct MrgRowsLaunch {
    MrgLaunch m;
    MatPair lanetab[32];
    uint32_t div_m, div_s;  // item / nseg = umulhi(item, div_m) >> div_s for items < 2^31 (div_m = 0: nseg = 1)
    // run mode (nseg = 32 nh, nh >= 2; nh = 0 otherwise): work item = run of `run` consecutive
    // tiles of one row (rpr runs per row); lanes step between tiles by step31 = A^(31 S)
    uint32_t nh, run, rpr;
    MatPair step31;
};
cudaError_t launch_mrg_fill_rows(const MrgRowsLaunch& p, const CUtensorMap& tmap, int kind, Grid g, cudaStream_t s);
size_t mrg_fill_rows_smem(int threads);
cudaError_t launch_philox_fill(const PhiloxLaunch& p, int kind, bool fast, Grid g, cudaStream_t s);
cudaError_t launch_philox_mc(const PhiloxLaunch& p, bool fast, Grid g, cudaStream_t s);
// TinyMT32 Leap Frog launch (kernels_tinymt32.cu; R19): buf = the handle's
// device buffer (params, base state, skip matrix T^(K-1), tables T^(2^b)).
constexpr size_t kTmLeapBufWords = 520 + 128 * 512;
// Player rows per TMA box of the transposed TinyMT32 Leap Frog fill (128-B rows, 128-B swizzle).
#ifndef SHV_TM_TR_ROWS
#define SHV_TM_TR_ROWS 128
#endif
constexpr uint32_t kTmTrRows = SHV_TM_TR_ROWS;
struct TmLeapLaunch {
    const uint32_t* buf;
    uint64_t players, first, ns;
    uint64_t o_lo, o_hi;       // player draw offset o (u128)
    uint64_t seg_len, seg_draws, n, items;  // item it: segment it / ns, row it % ns
    void* out;
    unsigned long long* hits;
    unsigned long long* counts;
    uint64_t tr_tb, tr_ps, tr_pl;  // transposed fill: t-blocks of 32, player segments, players per segment
};
// Transposed TinyMT32 Leap Frog fill (u32/f32, n % 4 == 0; tmap as for the
// MRG32k3a one: box 32 values x 128 rows, 128-B swizzle; tr_pl % 128 == 0).
cudaError_t launch_tm_leap_tr(const TmLeapLaunch& p, const CUtensorMap& tmap, int kind, unsigned blocks, cudaStream_t s);
cudaError_t tm_leap_tr_blocks_per_sm(int kind, int* out);
cudaError_t launch_tm_leap_prep(uint32_t* buf, uint64_t players, uint32_t seed, cudaStream_t s);
// mode: 0 u32, 1 f32, 2 f64 fill; 3 Monte Carlo
cudaError_t launch_tm_leap(const TmLeapLaunch& p, int mode, Grid g, cudaStream_t s);

// MTGP32-11213 launch (kernels_mtgp32.cu; R18): stream i of the launch has
// its parameter set at params + 36*i (pos, sh1, sh2, mask, tbl[16],
// tmp_tbl[16]) and its state at state + 352*i (the N = 351 current words,
// oldest first, one pad word).
constexpr uint32_t kMtgpN = 351, kMtgpStateWords = 352, kMtgpParamWords = 36;
struct MtgpLaunch {
    uint32_t* state;
    const uint32_t* params;
    uint64_t ns;
    uint64_t first;            // family index of launch stream 0 (seeding)
    void* out;                 // fill: row i at out + i*n elements
    uint64_t n;                // values per row (fill), samples (MC), draws (skip)
    unsigned long long* hits;
    unsigned long long* counts;
};
cudaError_t launch_mtgp_seed(const MtgpLaunch& p, uint32_t seed_base, cudaStream_t s);
// mode: 0 u32, 1 f32, 2 f64 fill; 3 Monte Carlo; 4 skip n draws
cudaError_t launch_mtgp(const MtgpLaunch& p, int mode, unsigned blocks, cudaStream_t s);

// Disjointness audit (kernels_audit.cu; S L407-415): rows = n_pe rows of
// `horizon` u32, windows = n_pe * wpr (wpr = horizon - 3). Workspace (u64
// words): scratch[6], count/rec_off/cursor/tab_off[nb] each, rec[2*windows]
// (hash, code), slots[2*windows + nb] (bucket b's table at tab_off[b],
// 2*count[b] + 1 slots), cand[2*windows] (slot, code); report on the device.
struct AuditLaunch {
    const uint32_t* rows;
    uint64_t horizon, wpr, windows;
    uint32_t lgb, nb;  // buckets: nb = 2^lgb (top hash bits)
    unsigned long long *scratch, *count, *rec_off, *cursor, *tab_off, *rec, *slots, *cand;
    shv_disjoint_report* report;
};
inline uint32_t audit_lg_buckets(uint64_t windows)
{
    uint32_t lg = 0;
    // >= ~2^16 windows per bucket, <= 2048 buckets: a scatter tile of 2^16 windows
    // then writes 32-record (512-B) runs per bucket, and a few bucket tables
    // (<= ~17 MB each at 2^30 windows) fit in L2 at a time
    while (lg < 11 && (windows >> (16 + lg)) > 0) ++lg;
    return lg;
}
inline uint64_t audit_workspace_words(uint64_t windows)
{
    const uint64_t nb = 1ull << audit_lg_buckets(windows);
    return 6 + 5 * nb + 6 * windows;
}
cudaError_t launch_audit(const AuditLaunch& p, unsigned blocks, cudaStream_t s);
// Leap Frog (kernels_leapfrog.cu): vec = 32-byte aligned rows, seg_len % 8 == 0.
cudaError_t launch_leap_fill(const LeapLaunch& p, int lgen, int kind, bool vec, Grid g, cudaStream_t s);
cudaError_t launch_leap_mc(const LeapLaunch& p, int lgen, Grid g, cudaStream_t s);
// Grouped Philox Leap Frog fill with TMA stores (u32/f32): `tmap` = 2D map of
// the launch rows (dim0 = n, dim1 = ns), box 32 values x 128 rows, 128-B
// swizzle; needs ngroups != 0, n % 32 == 0, seg_len % 32 == 0.
cudaError_t launch_leap_fill_tma(const LeapLaunch& p, const CUtensorMap& tmap, int kind, Grid g, cudaStream_t s);
cudaError_t leap_tma_blocks_per_sm(int kind, int* out);
// MRG32k3a Leap Frog fill by transposition (u32/f32): tmap as above (box 32
// values x 128 rows); needs n % 4 == 0, tr_pl % 128 == 0.
cudaError_t launch_leap_mrg_tr(const LeapLaunch& p, const CUtensorMap& tmap, int kind, unsigned blocks, cudaStream_t s);
cudaError_t leap_mrg_tr_blocks_per_sm(int kind, int* out);
cudaError_t leap_ctr_tr_blocks_per_sm(int lgen, int kind, int* out);
uint32_t leap_tr_warps(bool mrg);   // warps per block of leap_mrg_tr_kernel (mrg) / leap_ctr_tr_kernel
uint32_t leap_ctr_cols(int lgen);  // t-columns per lane (box row = 128 B per column) of leap_ctr_tr_kernel
uint32_t leap_tr_rows();  // players (box rows) per transposed TMA box; tr_pl is a multiple
// Counter-based Leap Frog fill by transposition (u32/f32): Philox with K % 4 == 0
// and first % 4 == 0, Threefry with K % 8 == 0 and first % 8 == 0.
cudaError_t launch_leap_ctr_tr(const LeapLaunch& p, const CUtensorMap& tmap, int lgen, int kind, unsigned blocks,
                               cudaStream_t s);

// Which kernel an occupancy query refers to.
enum KernelId : int {
    kKSeed = 0,
    kKMrgFill = 1,
    kKMrgMc = 2,
    kKPhiloxFill = 3,
    kKPhiloxMc = 4,
    kKPhiloxFillKeyed = 5,
    kKPhiloxMcKeyed = 6,
    kKTinyFill = 7,
    kKTinyMc = 8,
    kKThreefryFill = 9,
    kKThreefryMc = 10,
    kKLeapFill = 11,  // kind = output kind; `fast` = vector path; generator via leap_kernel_id
    kKLeapMc = 14,
    kKMrgFillTma = 17,  // after the leap ids 11..16
    kKMrgFillRows = 18,
};
// Leap kernels are keyed by (base id + generator): 11..13 fills, 14..16 MC.
constexpr int leap_kernel_id(int base, int lgen) { return base + lgen; }
// Occupancy of one kernel variant; each per-generator file answers for its own
// ids (cudaErrorInvalidValue otherwise).
cudaError_t mrg_occupancy(int kernel, int kind, bool fast, int threads, int* out);
cudaError_t philox_occupancy(int kernel, int kind, bool fast, int threads, int* out);
cudaError_t threefry_occupancy(int kernel, int kind, bool fast, int threads, int* out);
cudaError_t tinymt_occupancy(int kernel, int kind, bool fast, int threads, int* out);
cudaError_t leap_occupancy(int kernel, int kind, bool fast, int threads, int* out);
inline cudaError_t max_blocks_per_sm(int kernel, int kind, bool fast, int threads, int* out)
{
    switch (kernel) {
    case kKSeed: case kKMrgFill: case kKMrgMc: case kKMrgFillTma: case kKMrgFillRows:
        return mrg_occupancy(kernel, kind, fast, threads, out);
    case kKPhiloxFill: case kKPhiloxMc: case kKPhiloxFillKeyed: case kKPhiloxMcKeyed:
        return philox_occupancy(kernel, kind, fast, threads, out);
    case kKThreefryFill: case kKThreefryMc:
        return threefry_occupancy(kernel, kind, fast, threads, out);
    case kKTinyFill: case kKTinyMc:
        return tinymt_occupancy(kernel, kind, fast, threads, out);
    default:
        if (kernel >= kKLeapFill && kernel < kKLeapMc + 3) return leap_occupancy(kernel, kind, fast, threads, out);
    }
    return cudaErrorInvalidValue;
}
// Dynamic shared memory of the MRG vector-fill kernel at a block size.
size_t mrg_fill_smem(int threads, int kind);

}  // namespace shv
