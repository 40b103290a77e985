// kernels_mrg.cu — MRG32k3a kernels (arXiv 1412.8266 P L257-263 [§4.1]):
// per-stream seeding by jump matrices, bulk fills (u32 / f32 / f64) and the
// fused Monte Carlo pi kernel. Common pieces: kernels_common.cuh.
//
// The u32/f32 fills of shapes that split into row tiles run
// mrg_fill_rows_kernel (MrgMF step); other vector shapes run the
// stream-per-lane TMA kernel (u32/f32) or the staged vector kernel (f64), both
// on the MrgFF step; ragged shapes run the scalar kernel.
//
// Compile-time knobs (defaults = the product; tools/lab/build_knobs.sh builds
// variants for the labs, every variant gives bit-identical output):
//   SHV_MRG_STEP     step of the stream-per-lane / vector / scalar fills: 4 = MrgFF,
//                    3 = MrgIF, 5 = MrgSN, 7 = MrgMF
//   SHV_MRG_MC_STEP  step of the fused Monte Carlo kernel: 7 = MrgMF (385 ms for
//                    2^38 samples), 5 = MrgSN (405-409), 3 = MrgIF (464-474), 4 = MrgFF
//   SHV_MRG_MC_HIT   dartboard test: 0 = integer (MrgMF: 355 vs 387 ms), 1 = FP64 (MrgIF: 471 vs 474)
//   SHV_MRG_STAGE    staging of the vector fill: 1 = stage the f64 outputs only
//   SHV_MRG_MINB, SHV_MRG_TMA_MINB, SHV_MRG_ROWS_MINB: min-blocks hints
//   SHV_MRG_*_CKMASK which FP64 constants come from constant memory
//   SHV_LAB_GEN_HEADER / SHV_LAB_GEN: stand-in generator (tools/lab only)
#include "kernels_common.cuh"

#ifndef SHV_MRG_STEP
#define SHV_MRG_STEP 7  // stream-per-lane / vector fills: MrgMF (f64 vector 3.79 vs 3.88 ms, u32 TMA equal, lab77)
#endif
#ifndef SHV_MRG_MC_STEP
#define SHV_MRG_MC_STEP 7
#endif
#ifndef SHV_MRG_ROWS_STEP
#define SHV_MRG_ROWS_STEP 7  // step of the row-tile fill: 7 = MrgMF (2.75 vs 3.21 ms for MrgSN, lab65), 5 = MrgSN, 3 = MrgIF, 4 = MrgFF
#endif
#ifndef SHV_MRG_MC_HIT
#define SHV_MRG_MC_HIT 0  // dartboard test: 0 = integer (2 IMAD.WIDE; with MrgMF the FP64 pipe binds: 355 vs 387 ms, lab67), 1 = FP64 (hit_fp64)
#endif
#ifndef SHV_MRG_STAGE
#define SHV_MRG_STAGE 1
#endif
#ifndef SHV_MRG_MINB
#define SHV_MRG_MINB 4
#endif

namespace shv {

// Jump tables: [0][b] = A^(2^(76+b)) (substreams, b < 51),
//              [1][b] = A^(2^(127+b)) (streams, b < 64),
//              [2][b] = A^(2^b) (draws: Leap Frog players, b < 64).
__device__ MatPair g_jump_tab[3][64];

namespace {

// The six FP64 step constants (MrgFpK order) reach the DFMAs either from the
// launch parameters or from constant memory (bit i of MASK: c_mrg_fpk[i]).
// The mix decides which ptxas turns into uniform-register operands and which
// it keeps in registers; a DFMA reading three register pairs issues at 2/3
// rate (tools/lab/fp64_lab.cu: 82.6 vs 122 per SM per ns). Masks measured on
// B200 (tools/lab, all 64 compiled, the candidates timed): the TMA fill is
// fastest with 5 (3.49 ms vs 3.58 with no three-pair DFMA at all), the Monte
// Carlo kernel with 22 (no three-pair DFMA; 3 % faster than 0).
#ifndef SHV_MRG_FILL_CKMASK
#define SHV_MRG_FILL_CKMASK 5
#endif
#ifndef SHV_MRG_MC_CKMASK
#define SHV_MRG_MC_CKMASK 22
#endif
#ifndef SHV_MRG_ROWS_CKMASK
#define SHV_MRG_ROWS_CKMASK 21  // row-tile fill: magic, inv2, m2 from constant memory (MrgIF lab sweep: 3.43 vs 3.50 ms)
#endif
__constant__ double c_mrg_fpk[6] = {6755399441055744.0, 1.0 / 4294967087.0, 0x1.000059451f212p-32,
                                    4294967087.0, 4294944443.0, 5886603609186927.0};
// MrgSN constants (MrgFpK::sn_* order): bit i of SHV_MRG_SN_CKMASK takes
// c_mrg_snk[i] instead of the launch parameter; c_mrg_snk[5] = RN(1/m1) 2^1010
// (the lane starts reduce plain sums, not 4q).
#ifndef SHV_MRG_SN_CKMASK
#define SHV_MRG_SN_CKMASK 12  // c1s, c2s from constant memory: the DFMA.RM multiplicand as a uniform-register operand
#endif
__constant__ double c_mrg_snk[6] = {0x0.317b9fd79a126p-1022, 0x1.4e9d5b50f226fp-1022, 0x1.000000d10000bp+980,
                                    0x1.000059451f212p+978, 0x1.8p-12, 0x1.000000d10000bp+978};
#ifndef SHV_MRG_MF_LANE
#define SHV_MRG_MF_LANE 1  // MrgMF lane starts by magic-free split rows (split_row_mf)
#endif
#ifndef SHV_MRG_SN_LANE
#define SHV_MRG_SN_LANE 1  // MrgSN lane starts in the subnormal representation (split_row_sn)
#endif
template <int MASK>
__device__ __forceinline__ MrgFpK load_fpk(const MrgLaunch& P)
{
#define SHV_CKF(i) (((MASK >> (i)) & 1) ? c_mrg_fpk[i] : P.fpk[i])
    MrgFpK K{SHV_CKF(0), SHV_CKF(1), SHV_CKF(2), SHV_CKF(3), SHV_CKF(4), SHV_CKF(5), P.imul[0], P.imul[1]};
#undef SHV_CKF
#define SHV_CKS(i) (((SHV_MRG_SN_CKMASK >> (i)) & 1) ? c_mrg_snk[i] : P.snk[i])
    K.sn_c1q = SHV_CKS(0);
    K.sn_c2p = SHV_CKS(1);
    K.sn_c1s = SHV_CKS(2);
    K.sn_c2s = SHV_CKS(3);
    K.sn_M = SHV_CKS(4);
#undef SHV_CKS
    return K;
}

__device__ __forceinline__ void make_gen(const Mrg& s, MrgFF& g) { g = to_mrg_ff(s); }
__device__ __forceinline__ void make_gen(const Mrg& s, MrgIF& g) { g = to_mrg_if(s); }
__device__ __forceinline__ void make_gen(const Mrg& s, MrgSN& g) { g = to_mrg_sn(s); }
__device__ __forceinline__ void make_gen(const Mrg& s, MrgMF& g) { g = to_mrg_mf(s); }
// Step of a kernel by knob value: 3 = MrgIF, 4 = MrgFF, 5 = MrgSN, 7 = MrgMF.
template <int STEP>
using StepGen = typename std::conditional<
    STEP == 4, MrgFF,
    typename std::conditional<STEP == 5, MrgSN, typename std::conditional<STEP == 7, MrgMF, MrgIF>::type>::type>::type;
#ifdef SHV_LAB_GEN_HEADER  // tools/lab builds only: stand-in generators (never in libshv.so)
#include SHV_LAB_GEN_HEADER
using GenFill = SHV_LAB_GEN;
#else
using GenFill = StepGen<SHV_MRG_STEP>;
#endif
using GenMc = StepGen<SHV_MRG_MC_STEP>;
#ifndef SHV_MRG_SCALAR_STEP
#define SHV_MRG_SCALAR_STEP 4  // step of the scalar (ragged) fill: MrgFF (MrgMF: 9.71 vs 8.82 ms, lab77)
#endif
using GenScalar = StepGen<SHV_MRG_SCALAR_STEP>;


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

// Work item -> (launch stream i, segment j): streams fastest (a warp = 32
// rows, one segment), or segments fastest when rows are long (P.seg_fastest,
// set by the host for rows > 512 KB: a stream-fastest warp would scatter its
// 32 stores over 16+ different 2-MB pages).
template <bool SEG_FASTEST>
__device__ __forceinline__ void item_ij(const MrgLaunch& P, uint64_t it, uint64_t& i, uint64_t& j)
{
    if (SEG_FASTEST) {
        i = it / P.nseg;
        j = it - i * P.nseg;
    } else {
        j = it / P.ns;
        i = it - j * P.ns;
    }
}

// Start state of work item (stream i of the launch, segment j).
template <class Gen = GenFill>
__device__ __forceinline__ Gen item_state(const MrgLaunch& P, uint64_t i, uint64_t j)
{
    Mrg s = load_state(P.state, P.stride, P.stream_begin + i);
    apply(P.seg0.a, P.seg0.b, s);
    for (int b = 0; j; ++b, j >>= 1)
        if (j & 1) apply(P.segpow[b].a, P.segpow[b].b, s);
    Gen g;
    make_gen(s, g);
    return g;
}

// 8 values -> staging pieces (u32/f32: 2 pieces; f64: 4 pieces).
template <int KIND>
__device__ __forceinline__ void stage8(uint4* wb, unsigned lane, unsigned q0, GenFill& s, const MrgFpK& K)
{
    uint32_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = mrg_next(s, K);
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

template <int KIND, bool SEG_FASTEST>
__global__ void __launch_bounds__(256, SHV_MRG_MINB) mrg_fill_vec_kernel(const __grid_constant__ MrgLaunch P)
{
    using T = OutT<KIND>;
    const MrgFpK K = load_fpk<SHV_MRG_MC_CKMASK>(P);
    const unsigned lane = threadIdx.x & 31, warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);  // warp-uniform loop (see the TMA fill)
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
        GenFill s{};
        if (it < P.items) {
            uint64_t i, j;
            item_ij<SEG_FASTEST>(P, it, i, j);
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
                for (unsigned g = 0; g < G / 8; ++g) stage8<KIND>(wb, lane, g * (KIND == kF64 ? 4 : 2), s, K);
            } else {
                for (unsigned g = 0; g < cnt / 8; ++g) stage8<KIND>(wb, lane, g * (KIND == kF64 ? 4 : 2), s, K);
            }
            write_round<T>(wb, lane, r, cnt, row);
        }
    }
    } else {
    (void)lane;
    (void)warp;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t it = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; it < P.items; it += nthr) {
        uint64_t i, j;
        item_ij<SEG_FASTEST>(P, it, i, j);
        GenFill s = item_state(P, i, j);
        const uint64_t c0 = j * P.seg_len;
        const uint64_t len = min(P.seg_len, P.n - c0);
        T* o = reinterpret_cast<T*>(P.out) + i * P.n + c0;
        for (uint64_t t = 0; t < len; t += 8) {
            uint32_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = mrg_next(s, K);
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

// MRG32k3a fill, TMA store path. A warp owns a tile of 32
// consecutive rows (streams 32g..32g+31 of the launch) x one segment; lane l
// generates row 32g+l. Each round the lanes write 128 B of their rows into the
// warp's 4-KB shared-memory box (128-B swizzle: 16-byte chunk q of row l sits
// at chunk q ^ (l & 7), so the eight lanes of a quarter-warp hit distinct
// banks), and one lane hands the 32 x 128-B box to the TMA engine
// (cp.async.bulk.tensor.2d shared -> global). The SM's load/store unit never
// sees the scattered 32-byte row pieces that cap per-lane STG.256 stores at
// ~4.5 TB/s (tools/lab, null generator); boxes that run past the row end or
// past the launch's last row are clipped by the tensor map bounds.
#ifndef SHV_MRG_NBUF
#define SHV_MRG_NBUF 1
#endif
#ifndef SHV_MRG_TMA_MINB
#define SHV_MRG_TMA_MINB (SHV_MRG_STEP == 4 ? 4 : 2)  // lab sweep: FF 4 blocks, IF 2 blocks per SM
#endif
#ifndef SHV_MRG_PIN
#define SHV_MRG_PIN 1  // state through an empty volatile asm after every SHV_MRG_PIN-th 4-value store (0: never)
#endif
// An empty volatile asm the state passes through: volatile asms keep their
// order, so ptxas cannot run the serial component-2 chain of later groups
// ahead of the current group's store (it did, holding up to 32 finished
// words live and spilling at the 48-register bound).
__device__ __forceinline__ void pin_state(MrgSN& g)
{
    asm volatile("" : "+r"(g.x0), "+r"(g.x1), "+r"(g.x2), "+r"(g.y0), "+r"(g.y1), "+r"(g.y2));
}
__device__ __forceinline__ void pin_state(MrgMF& g)
{
    asm volatile("" : "+d"(g.x0), "+d"(g.x1), "+d"(g.x2), "+d"(g.y0), "+d"(g.y1), "+d"(g.y2));
}
__device__ __forceinline__ void pin_state(MrgIF& g)
{
    asm volatile("" : "+r"(g.x0), "+r"(g.x1), "+r"(g.x2), "+d"(g.y0), "+d"(g.y1), "+d"(g.y2));
}
__device__ __forceinline__ void pin_state(MrgFF& g)
{
    asm volatile("" : "+d"(g.x0), "+d"(g.x1), "+d"(g.x2), "+d"(g.y0), "+d"(g.y1), "+d"(g.y2));
}
#ifndef SHV_MRG_STS4
#define SHV_MRG_STS4 1  // u32/f32 boxes: one shared store per 4 values (0: per 8)
#endif
constexpr uint32_t kTmaBufs = SHV_MRG_NBUF;  // boxes per warp in flight (2: double buffering)

// Generates `len` values per lane from g (lane l: box row l) in rounds of 128 B
// and hands each 32-row x 128-B box to the TMA engine at tensor coordinates
// (col0 + r, row0). bsel (the warp's current box buffer) carries across calls.
template <int KIND, class Gen>
__device__ __forceinline__ void mrg_tma_rounds(const CUtensorMap* tmap, const MrgFpK& K, unsigned lane, uint32_t box0,
                                               uint32_t& bsel, Gen& s, uint32_t len, uint64_t col0, uint64_t row0)
{
    constexpr uint32_t W = 128 / sizeof(OutT<KIND>);  // values per row per box
    for (uint32_t r = 0; r < len; r += W) {
        const uint32_t box = box0 + bsel * 4096u;
        const uint32_t rowsw = box + lane * 128u + ((lane & 7u) << 4);  // ^ (q << 4) = chunk q
        if constexpr (KIND != kF64 && SHV_MRG_STS4) {
            // 4 values per shared store: fewer live registers (48-register bound)
#pragma unroll
            for (unsigned q = 0; q < W / 4; ++q) {
                uint32_t v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = mrg_next(s, K);
                if (q == 0) {  // this buffer's previous box must have left shared memory
                    if (lane == 0) {
                        if (kTmaBufs == 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                        else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    }
                    __syncwarp();
                }
                const uint4 a = pack4<KIND>(v[0], v[1], v[2], v[3]);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowsw ^ (q << 4)), "r"(a.x), "r"(a.y),
                             "r"(a.z), "r"(a.w)
                             : "memory");
                if (SHV_MRG_PIN && q % SHV_MRG_PIN == SHV_MRG_PIN - 1) pin_state(s);
            }
        } else {
#pragma unroll
        for (unsigned q8 = 0; q8 < W / 8; ++q8) {
            uint32_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = mrg_next(s, K);
            if (q8 == 0) {  // this buffer's previous box must have left shared memory
                if (lane == 0) {
                    if (kTmaBufs == 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                }
                __syncwarp();
            }
            if (KIND == kF64) {
#pragma unroll
                for (unsigned k = 0; k < 4; ++k) {
                    const double a = mrg_f64(v[2 * k]), b = mrg_f64(v[2 * k + 1]);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowsw ^ ((4 * q8 + k) << 4)),
                                 "r"(__double2loint(a)), "r"(__double2hiint(a)), "r"(__double2loint(b)),
                                 "r"(__double2hiint(b))
                                 : "memory");
                }
            } else {
                const uint4 a = pack4<KIND>(v[0], v[1], v[2], v[3]), b = pack4<KIND>(v[4], v[5], v[6], v[7]);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowsw ^ ((2 * q8) << 4)), "r"(a.x),
                             "r"(a.y), "r"(a.z), "r"(a.w)
                             : "memory");
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowsw ^ ((2 * q8 + 1) << 4)),
                             "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                             : "memory");
            }
        }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // st.shared -> async proxy
        __syncwarp();
        if (lane == 0) {
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tmap),
                         "r"(box), "r"((int)(col0 + r)), "r"((int)row0)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        bsel = kTmaBufs == 1 ? 0u : bsel ^ 1u;
    }
}

// One TMA tile: rows 32g..32g+31 of the launch x segment j; lane l generates
// row 32g + l.
template <int KIND>
__device__ __forceinline__ void mrg_tma_tile(const MrgLaunch& P, const CUtensorMap* tmap, const MrgFpK& K,
                                             unsigned lane, uint32_t box0, uint32_t& bsel, uint64_t g, uint64_t j)
{
    const uint64_t i = 32 * g + lane;
    // rows past the launch's last stream compute a clipped, discarded row
    GenFill s = item_state(P, i < P.ns ? i : P.ns - 1, j);
    const uint64_t c0 = j * P.seg_len;
    const uint32_t len = (uint32_t)min(P.seg_len, P.n - c0);  // warp-uniform
    mrg_tma_rounds<KIND>(tmap, K, lane, box0, bsel, s, len, c0, 32 * g);
}

template <int KIND, bool SEG_FASTEST>
__global__ void __launch_bounds__(256, SHV_MRG_TMA_MINB)
    mrg_fill_tma_kernel(const __grid_constant__ MrgLaunch P, const __grid_constant__ CUtensorMap tmap)
{
    extern __shared__ uint8_t tma_smem[];
    const MrgFpK K = load_fpk<SHV_MRG_FILL_CKMASK>(P);
    // warp index through a shuffle from lane 0: ptxas then sees the tile loop as
    // warp-uniform and keeps loop-invariant FP64 constants in uniform registers
    // (DFMA operands at full rate); 3.73 -> 3.50 ms for the C5 MRG fill (tools/lab)
    const unsigned lane = threadIdx.x & 31, warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
    // 1024-byte aligned boxes (128-B swizzle); the launch adds 1 KB of slack
    const uint32_t base = ((uint32_t)__cvta_generic_to_shared(tma_smem) + 1023u) & ~1023u;
    const uint32_t box0 = base + warp * (4096u * kTmaBufs);
    uint32_t bsel = 0;  // buffer of the box being generated
    const uint64_t G = (P.ns + 31) / 32, ntiles = G * P.nseg;
    const uint64_t wstride = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t t = (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp; t < ntiles; t += wstride) {
        uint64_t g, j;
        if (SEG_FASTEST) {
            g = t / P.nseg;
            j = t - g * P.nseg;
        } else {
            j = t / G;
            g = t - j * G;
        }
        mrg_tma_tile<KIND>(P, &tmap, K, lane, box0, bsel, g, j);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// The lane table in shared memory, FP64-split for the start jump: entry e of
// lane matrix j at ltab[e * 32 + j] (lanes read consecutive 8-byte words),
// e = (component c, row r, column q, half h) -> ((c * 3 + r) * 3 + q) * 2 + h,
// half 0 = M >> 16, half 1 = M & 0xffff (exact doubles; lanes index the table
// divergently, so it lives in shared memory, not the parameter block).
// (double2 entries with LDS.128 spill at the 48-register bound: lab26.)
constexpr uint32_t kLaneTabEntries = 36;

// Row r of one component: (M v) mod m for canonical v (doubles) and the split
// row (Mh, Ml): Ah = sum Mh_q v_q and Al = sum Ml_q v_q are exact (< 3 * 2^48),
// Ah mod m by a floor reduction (Ah * delta * m < 0.1 for inv = RN / RU(1/m),
// DESIGN.md §4.2), X = (Ah mod m) * 2^16 + Al < 2^50 exact, X mod m likewise.
// 13 FP64 operations, no IMAD.WIDE (which the start jump's integer matvec
// spends 37 of per apply, ~6 issue cycles each on B200; tools/lab/pipe_mix2_lab.cu).
__device__ __forceinline__ double split_row_mod(const double* __restrict__ lt, uint32_t stride, uint32_t e0, double v0,
                                                double v1, double v2, double inv, double m, double magic)
{
    const double h0 = lt[(e0 + 0) * stride], l0 = lt[(e0 + 1) * stride];
    const double h1 = lt[(e0 + 2) * stride], l1 = lt[(e0 + 3) * stride];
    const double h2 = lt[(e0 + 4) * stride], l2 = lt[(e0 + 5) * stride];
    const double ah = __fma_rn(h2, v2, __fma_rn(h1, v1, __dmul_rn(h0, v0)));
    const double al = __fma_rn(l2, v2, __fma_rn(l1, v1, __dmul_rn(l0, v0)));
    const double kh = __dadd_rn(__fma_rd(ah, inv, magic), -magic);
    const double rh = __fma_rn(-kh, m, ah);
    const double x = __fma_rn(rh, 65536.0, al);
    const double kx = __dadd_rn(__fma_rd(x, inv, magic), -magic);
    return __fma_rn(-kx, m, x);
}

// M * (x, y) on the FP64 pipe for a split matrix at `tab` (entries `stride`
// doubles apart: the lane table with stride 32 at lane jl, or the run-step
// matrix with stride 1), returned as the generator state of the row tiles.
__device__ __forceinline__ void set_state(MrgIF& g, const double r[6], const MrgFpK& K)
{
    g.x0 = (uint32_t)__double2loint(__dadd_rn(r[0], K.magic));
    g.x1 = (uint32_t)__double2loint(__dadd_rn(r[1], K.magic));
    g.x2 = (uint32_t)__double2loint(__dadd_rn(r[2], K.magic));
    g.y0 = r[3];
    g.y1 = r[4];
    g.y2 = r[5];
}
__device__ __forceinline__ void set_state(MrgSN& g, const double r[6], const MrgFpK& K)
{
    g.x0 = (uint32_t)__double2loint(__dadd_rn(r[0], K.magic));
    g.x1 = (uint32_t)__double2loint(__dadd_rn(r[1], K.magic));
    g.x2 = (uint32_t)__double2loint(__dadd_rn(r[2], K.magic));
    g.y0 = (uint32_t)__double2loint(__dadd_rn(r[3], K.magic));
    g.y1 = (uint32_t)__double2loint(__dadd_rn(r[4], K.magic));
    g.y2 = (uint32_t)__double2loint(__dadd_rn(r[5], K.magic));
}
#if SHV_MRG_ROWS_STEP == 4
__device__ __forceinline__ void set_state(MrgFF& g, const double r[6], const MrgFpK&)
{
    g = MrgFF{r[0], r[1], r[2], r[3], r[4], r[5]};
}
#endif
__device__ __forceinline__ double x_of(double x) { return x; }
__device__ __forceinline__ double x_of(uint32_t x) { return __uint2double_rn(x); }

template <class Gen>
__device__ __forceinline__ Gen apply_split(const double* __restrict__ tab, uint32_t stride, double x0, double x1,
                                           double x2, double y0, double y1, double y2, const MrgFpK& K)
{
    double r[6];
    r[0] = split_row_mod(tab, stride, 0, x0, x1, x2, K.inv1, K.m1, K.magic);
    r[1] = split_row_mod(tab, stride, 6, x0, x1, x2, K.inv1, K.m1, K.magic);
    r[2] = split_row_mod(tab, stride, 12, x0, x1, x2, K.inv1, K.m1, K.magic);
    r[3] = split_row_mod(tab, stride, 18, y0, y1, y2, K.inv2, K.m2, K.magic);
    r[4] = split_row_mod(tab, stride, 24, y0, y1, y2, K.inv2, K.m2, K.magic);
    r[5] = split_row_mod(tab, stride, 30, y0, y1, y2, K.inv2, K.m2, K.magic);
    Gen g;
    set_state(g, r, K);
    return g;
}

// Row r of one component in the subnormal representation (MrgSN, DESIGN.md
// §4.2): v as the pairs D(v) = {v, 0}; Ah = sum Mh_q v_q and Al = sum Ml_q v_q
// are exact (< 3 * 2^48 units) and their bit patterns are the integers, so
// rh = Ah mod m = lo(Ah) + c floor(Ah / m) (one DFMA.RM and one IMAD), then
// X = rh 2^16 + Al < 2^50 the same way. 9 FP64 + 2 IMAD, canonical u32 out.
__device__ __forceinline__ uint32_t split_row_sn(const double* __restrict__ lt, uint32_t stride, uint32_t e0,
                                                 double v0, double v1, double v2, double cinv, double M, uint32_t c)
{
    const double h0 = lt[(e0 + 0) * stride], l0 = lt[(e0 + 1) * stride];
    const double h1 = lt[(e0 + 2) * stride], l1 = lt[(e0 + 3) * stride];
    const double h2 = lt[(e0 + 4) * stride], l2 = lt[(e0 + 5) * stride];
    const double ah = __fma_rn(h2, v2, __fma_rn(h1, v1, __dmul_rn(h0, v0)));
    const double al = __fma_rn(l2, v2, __fma_rn(l1, v1, __dmul_rn(l0, v0)));
    const uint32_t rh = (uint32_t)__double2loint(ah) + c * (uint32_t)__double2loint(__fma_rd(ah, cinv, M));
    const double x = __fma_rn(65536.0, mrg_sn(rh), al);
    return (uint32_t)__double2loint(x) + c * (uint32_t)__double2loint(__fma_rd(x, cinv, M));
}

__device__ __forceinline__ MrgSN apply_split_sn(const double* __restrict__ tab, uint32_t stride, const uint32_t w[6],
                                                const MrgFpK& K)
{
    const double c1 = c_mrg_snk[5];  // RN(1/m1) 2^1010 (the plain, not the 4x, inverse)
    const double x0 = mrg_sn(w[0]), x1 = mrg_sn(w[1]), x2 = mrg_sn(w[2]);
    const double y0 = mrg_sn(w[3]), y1 = mrg_sn(w[4]), y2 = mrg_sn(w[5]);
    MrgSN g;
    g.x0 = split_row_sn(tab, stride, 0, x0, x1, x2, c1, K.sn_M, kC1);
    g.x1 = split_row_sn(tab, stride, 6, x0, x1, x2, c1, K.sn_M, kC1);
    g.x2 = split_row_sn(tab, stride, 12, x0, x1, x2, c1, K.sn_M, kC1);
    g.y0 = split_row_sn(tab, stride, 18, y0, y1, y2, K.sn_c2s, K.sn_M, kC2);
    g.y1 = split_row_sn(tab, stride, 24, y0, y1, y2, K.sn_c2s, K.sn_M, kC2);
    g.y2 = split_row_sn(tab, stride, 30, y0, y1, y2, K.sn_c2s, K.sn_M, kC2);
    return g;
}

// Row r in the subnormal representation with magic-free quotients (MrgMF):
// Ah, Al as in split_row_sn, kh = mul.rm(Ah, inv) = D(floor(Ah / m)), D(rh) =
// fma(-kh, m, Ah), X = 2^16 D(rh) + Al, then the same for X: 11 FP64, no
// integer or move instructions, the result already the state pair D(r).
__device__ __forceinline__ double split_row_mf(const double* __restrict__ lt, uint32_t stride, uint32_t e0,
                                               double v0, double v1, double v2, double inv, double m)
{
    const double h0 = lt[(e0 + 0) * stride], l0 = lt[(e0 + 1) * stride];
    const double h1 = lt[(e0 + 2) * stride], l1 = lt[(e0 + 3) * stride];
    const double h2 = lt[(e0 + 4) * stride], l2 = lt[(e0 + 5) * stride];
    const double ah = __fma_rn(h2, v2, __fma_rn(h1, v1, __dmul_rn(h0, v0)));
    const double al = __fma_rn(l2, v2, __fma_rn(l1, v1, __dmul_rn(l0, v0)));
    const double rh = __fma_rn(-__dmul_rd(ah, inv), m, ah);
    const double x = __fma_rn(65536.0, rh, al);
    return __fma_rn(-__dmul_rd(x, inv), m, x);
}

__device__ __forceinline__ MrgMF apply_split_mf(const double* __restrict__ tab, uint32_t stride, double x0, double x1,
                                                double x2, double y0, double y1, double y2, const MrgFpK& K)
{
    MrgMF g;
    g.x0 = split_row_mf(tab, stride, 0, x0, x1, x2, K.inv1, K.m1);
    g.x1 = split_row_mf(tab, stride, 6, x0, x1, x2, K.inv1, K.m1);
    g.x2 = split_row_mf(tab, stride, 12, x0, x1, x2, K.inv1, K.m1);
    g.y0 = split_row_mf(tab, stride, 18, y0, y1, y2, K.inv2, K.m2);
    g.y1 = split_row_mf(tab, stride, 24, y0, y1, y2, K.inv2, K.m2);
    g.y2 = split_row_mf(tab, stride, 30, y0, y1, y2, K.inv2, K.m2);
    return g;
}

__device__ __forceinline__ MrgMF mf_of(const MrgSN& g)
{
    return MrgMF{mrg_sn(g.x0), mrg_sn(g.x1), mrg_sn(g.x2), mrg_sn(g.y0), mrg_sn(g.y1), mrg_sn(g.y2)};
}

// Start state of a row-tile lane: lanetab[jl] * (x, y).
template <class Gen>
__device__ __forceinline__ Gen lane_start(const double* __restrict__ lt, uint32_t jl, const uint32_t w[6], const MrgFpK& K)
{
    if constexpr (std::is_same<Gen, MrgMF>::value) {
        if (SHV_MRG_MF_LANE)
            return apply_split_mf(lt + jl, 32, mrg_sn(w[0]), mrg_sn(w[1]), mrg_sn(w[2]), mrg_sn(w[3]), mrg_sn(w[4]),
                                  mrg_sn(w[5]), K);
        return mf_of(apply_split_sn(lt + jl, 32, w, K));
    } else if constexpr (std::is_same<Gen, MrgSN>::value && SHV_MRG_SN_LANE) {
        return apply_split_sn(lt + jl, 32, w, K);
    } else {
        return apply_split<Gen>(lt + jl, 32, __uint2double_rn(w[0]), __uint2double_rn(w[1]), __uint2double_rn(w[2]),
                                __uint2double_rn(w[3]), __uint2double_rn(w[4]), __uint2double_rn(w[5]), K);
    }
}

// A lane that ended segment j of a tile (at offset (j + 1) S) continues with
// segment j + 32 of the next tile of its row: A^(31 S) * state (run mode).
template <class Gen>
__device__ __forceinline__ Gen lane_advance(const double* __restrict__ st31, const Gen& g, const MrgFpK& K)
{
    if constexpr (std::is_same<Gen, MrgMF>::value) {
        if (SHV_MRG_MF_LANE) return apply_split_mf(st31, 1, g.x0, g.x1, g.x2, g.y0, g.y1, g.y2, K);
        const uint32_t w[6] = {(uint32_t)__double2loint(g.x0), (uint32_t)__double2loint(g.x1),
                               (uint32_t)__double2loint(g.x2), (uint32_t)__double2loint(g.y0),
                               (uint32_t)__double2loint(g.y1), (uint32_t)__double2loint(g.y2)};
        return mf_of(apply_split_sn(st31, 1, w, K));
    } else if constexpr (std::is_same<Gen, MrgSN>::value && SHV_MRG_SN_LANE) {
        const uint32_t w[6] = {g.x0, g.x1, g.x2, g.y0, g.y1, g.y2};
        return apply_split_sn(st31, 1, w, K);
    } else {
        return apply_split<Gen>(st31, 1, x_of(g.x0), x_of(g.x1), x_of(g.x2), x_of(g.y0), x_of(g.y1), x_of(g.y2), K);
    }
}

#if defined(SHV_LAB_GEN_HEADER) && SHV_MRG_ROWS_STEP == 9
using GenRows = MrgNullRows;  // tools/lab builds only: the store-path ceiling of the row tiles
#else
using GenRows = StepGen<SHV_MRG_ROWS_STEP>;
#endif

__device__ __forceinline__ void prefetch_words(const MrgLaunch& P, uint32_t i)
{
    const uint32_t* st = P.state + P.stream_begin + i;
#pragma unroll
    for (int k = 0; k < 6; ++k) asm volatile("prefetch.global.L2 [%0];" ::"l"(st + k * P.stride));
}

__device__ __forceinline__ void load_words(const MrgLaunch& P, uint32_t i, uint32_t w[6])
{
    const uint32_t* st = P.state + P.stream_begin + i;
#pragma unroll
    for (int k = 0; k < 6; ++k) w[k] = __ldg(st + k * P.stride);
}

// MRG32k3a fill, row tiles (TMA). The output is viewed as
// [ns * nseg][S] (row i = segments i*nseg .. i*nseg + nseg - 1 of S = seg_len
// values, contiguous since S * nseg = n), and a warp tile is 32 consecutive
// segments — for the C5 shape (S = 256, nseg = 16) two whole 16-KB stream rows.
// Lane l owns segment j of row i (32t + l = i*nseg + j) and starts from
// (A^(32 S))^(j / 32) * lanetab[j % 32] * state_i, lanetab[k] = A^(o + k S)
// (host-built, FP64-split into shared memory). Each round the warp's box
// covers 32 segments x 128 B, 4 KB of one DRAM-local region, so a row's pages
// are complete within a few rounds; stream-per-lane tiles
// (mrg_fill_tma_kernel) scatter each round over 32 rows 16 KB apart and cap
// the store path at ~4.6 TB/s (tools/lab/tma_layout_lab.cu: 6.1 vs 4.7 TB/s
// with a null generator). The next tile's state words are loaded while the
// current tile generates.
#ifndef SHV_MRG_ROWS_TPB
#define SHV_MRG_ROWS_TPB 256  // launch bound (threads per block) of the row-tile fill
#endif
#ifndef SHV_MRG_ROWS_PREF
#define SHV_MRG_ROWS_PREF 0  // next tile's state words: 0 = registers, 1 = L2 prefetch hint (more spills), 2 = none
#endif
#ifndef SHV_MRG_ROWS_MINB
#define SHV_MRG_ROWS_MINB 5  // <= 48 registers: 5 blocks of 256 per SM (lab: 3.50 vs 3.56 ms at 4)
#endif
template <int KIND, bool RUN>
__global__ void __launch_bounds__(SHV_MRG_ROWS_TPB, SHV_MRG_ROWS_MINB)
    mrg_fill_rows_kernel(const __grid_constant__ MrgRowsLaunch R, const __grid_constant__ CUtensorMap tmap)
{
    extern __shared__ uint8_t tma_smem[];
    const MrgLaunch& P = R.m;
    const MrgFpK K = load_fpk<SHV_MRG_ROWS_CKMASK>(P);
    const unsigned lane = threadIdx.x & 31, warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(tma_smem);
    const uint32_t base = (sbase + 1023u) & ~1023u;
    const uint32_t nwarps = blockDim.x >> 5;
    double* lt = reinterpret_cast<double*>(tma_smem + (base - sbase) + nwarps * 4096u * kTmaBufs);
    double* st31 = lt + 32 * kLaneTabEntries;  // run-step matrix A^(31 S), same split layout, stride 1
    for (uint32_t k = threadIdx.x; k < 33 * kLaneTabEntries; k += blockDim.x) {
        const bool step = k >= 32 * kLaneTabEntries;
        const uint32_t j = step ? 0 : (k & 31), e = step ? k - 32 * kLaneTabEntries : k >> 5;
        const uint32_t c = e / 18, rq = (e % 18) >> 1, h = e & 1;
        const MatPair& mp = step ? R.step31 : R.lanetab[j];
        const uint32_t M = c ? mp.b[rq] : mp.a[rq];
        lt[k] = (double)(h ? (M & 0xffffu) : (M >> 16));
    }
    __syncthreads();
    const uint32_t box0 = base + warp * (4096u * kTmaBufs);
    uint32_t bsel = 0;
    if constexpr (RUN) {
        // Run mode (rows of nh = nseg / 32 >= 2 tiles): a warp owns a run of up to R.run
        // consecutive tiles of one row; the first starts by the per-bit jumps of its tile
        // index and the lane table, each next one by one A^(31 S) step per lane (the
        // per-tile jump would cost popcount(jh) integer mat-vecs per lane).
        const uint32_t len = (uint32_t)P.seg_len;
        const uint64_t nruns = P.ns * (uint64_t)R.rpr;
        const uint64_t wstride = (uint64_t)gridDim.x * nwarps;
        for (uint64_t run = (uint64_t)blockIdx.x * nwarps + warp; run < nruns; run += wstride) {
            const uint64_t i = run / R.rpr;
            const uint32_t jh0 = (uint32_t)(run - i * R.rpr) * R.run;
            const uint32_t cnt = min(R.run, R.nh - jh0);
            uint32_t w[6];
            load_words(P, (uint32_t)i, w);
            Mrg s{w[0], w[1], w[2], w[3], w[4], w[5]};
            for (uint32_t jh = jh0, bit = 0; jh; ++bit, jh >>= 1)
                if (jh & 1) apply(P.segpow[bit].a, P.segpow[bit].b, s);
            const uint32_t v[6] = {s.x0, s.x1, s.x2, s.y0, s.y1, s.y2};
            GenRows g = lane_start<GenRows>(lt, lane, v, K);
            for (uint32_t k = 0; k < cnt; ++k) {
                if (k) g = lane_advance<GenRows>(st31, g, K);
                mrg_tma_rounds<KIND>(&tmap, K, lane, box0, bsel, g, len, 0, i * P.nseg + 32ull * (jh0 + k));
            }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        return;
    } else {
    const uint64_t ntiles = (P.items + 31) / 32;
    const uint64_t wstride = (uint64_t)gridDim.x * nwarps;
    const uint32_t len = (uint32_t)P.seg_len, items = (uint32_t)P.items, nseg = P.nseg;  // items < 2^31 (host check)
    uint64_t t = (uint64_t)blockIdx.x * nwarps + warp;
    auto item = [&](uint64_t tt) {
        uint32_t it = (uint32_t)(32 * tt) + lane;
        return it < items ? it : items - 1;  // past the last segment: a clipped, discarded row
    };
    // it / nseg by the host's multiply-shift (Granlund-Montgomery, 31-bit numerators)
    auto row = [&](uint32_t it) { return R.div_m ? __umulhi(it, R.div_m) >> R.div_s : it; };
#if SHV_MRG_ROWS_PREF == 0
    uint32_t w[6];
    if (t < ntiles) load_words(P, row(item(t)), w);
#else
    if (t < ntiles) prefetch_words(P, row(item(t)));
#endif
    for (; t < ntiles; t += wstride) {
        const uint32_t it = item(t);
        const uint32_t i = row(it), j = it - i * nseg;
        uint32_t cur[6];
#if SHV_MRG_ROWS_PREF == 0
#pragma unroll
        for (int k = 0; k < 6; ++k) cur[k] = w[k];
        if (t + wstride < ntiles) load_words(P, row(item(t + wstride)), w);  // prefetch
#else
        // the next tile's words go to L2 by a prefetch hint: no registers held
        // across the tile's rounds (the register copy spilled at 48 registers)
        load_words(P, i, cur);
        if (SHV_MRG_ROWS_PREF == 1 && t + wstride < ntiles) prefetch_words(P, row(item(t + wstride)));
#endif
        GenRows g;
        if (j < 32) {
            g = lane_start<GenRows>(lt, j, cur, K);
        } else {  // rows of more than 32 segments: (A^(32 S))^(j / 32) first
            Mrg s{cur[0], cur[1], cur[2], cur[3], cur[4], cur[5]};
            for (uint32_t jh = j >> 5, bit = 0; jh; ++bit, jh >>= 1)
                if (jh & 1) apply(P.segpow[bit].a, P.segpow[bit].b, s);
            const uint32_t v[6] = {s.x0, s.x1, s.x2, s.y0, s.y1, s.y2};
            g = lane_start<GenRows>(lt, j & 31, v, K);
        }
        mrg_tma_rounds<KIND>(&tmap, K, lane, box0, bsel, g, len, 0, 32 * t);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

// MRG32k3a fill, scalar path (any row length / element-aligned pointer).
template <int KIND>
__global__ void __launch_bounds__(256) mrg_fill_scalar_kernel(const __grid_constant__ MrgLaunch P)
{
    using T = OutT<KIND>;
    const MrgFpK K = load_fpk<SHV_MRG_MC_CKMASK>(P);
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t it = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; it < P.items; it += nthr) {
        uint64_t i, j;
        item_ij<false>(P, it, i, j);
        GenScalar s = item_state<GenScalar>(P, i, j);
        const uint64_t c0 = j * P.seg_len;
        const uint64_t len = min(P.seg_len, P.n - c0);
        T* o = reinterpret_cast<T*>(P.out) + i * P.n + c0;
        for (uint64_t t = 0; t < len; ++t) {
            const uint32_t z = mrg_next(s, K);
            if (KIND == kU32) o[t] = (T)z;
            else if (KIND == kF32) o[t] = (T)to_f32(z);
            else o[t] = (T)mrg_f64(z);
        }
    }
}

#ifndef SHV_MRG_MC_UNROLL
#define SHV_MRG_MC_UNROLL 12  // samples per unrolled iteration of the MC loop
#endif
constexpr uint32_t kMcU = SHV_MRG_MC_UNROLL;
__global__ void __launch_bounds__(256) mrg_mc_kernel(const __grid_constant__ MrgLaunch P)
{
    const MrgFpK K = load_fpk<SHV_MRG_MC_CKMASK>(P);
    // Warp-uniform loops (warp index via shuffle, trip counts via warp max) so
    // ptxas keeps the FP64 constants in uniform registers, as in the fills.
    // Lanes past their segment's end keep stepping but count no hits.
    const unsigned lane = threadIdx.x & 31;
    const uint64_t wstride = (uint64_t)gridDim.x * (blockDim.x >> 5) * 32;
    uint64_t total = 0;
    for (uint64_t base = ((uint64_t)blockIdx.x * (blockDim.x >> 5) + __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0)) * 32;
         base < P.items; base += wstride) {
        const uint64_t it = base + lane;
        uint64_t i, j;
        item_ij<false>(P, it < P.items ? it : P.items - 1, i, j);
        GenMc s = item_state<GenMc>(P, i, j);
        const uint64_t c0 = j * P.seg_len;
        const uint32_t len = it < P.items ? (uint32_t)min(P.seg_len, P.n - c0) : 0u;
        const uint32_t wlen = __reduce_max_sync(0xffffffffu, len);
        const uint32_t wmin = __reduce_min_sync(0xffffffffu, len);
        uint32_t h = 0;
        uint32_t k = 0;
        for (; k + kMcU <= wmin; k += kMcU) {  // every lane inside its segment: no per-sample mask
#pragma unroll
            for (int u = 0; u < (int)kMcU; ++u) {
                const uint32_t w0 = mrg_next(s, K);
                const uint32_t w1 = mrg_next(s, K);
                h += SHV_MRG_MC_HIT ? hit_fp64(w0, w1) : hit(w0, w1);
            }
        }
        for (; k + kMcU <= wlen; k += kMcU) {
#pragma unroll
            for (int u = 0; u < (int)kMcU; ++u) {
                const uint32_t w0 = mrg_next(s, K);
                const uint32_t w1 = mrg_next(s, K);
                h += (SHV_MRG_MC_HIT ? hit_fp64(w0, w1) : hit(w0, w1)) & (k + u < len ? 1u : 0u);
            }
        }
        for (; k < wlen; ++k) {
            const uint32_t w0 = mrg_next(s, K);
            const uint32_t w1 = mrg_next(s, K);
            h += (SHV_MRG_MC_HIT ? hit_fp64(w0, w1) : hit(w0, w1)) & (k < len ? 1u : 0u);
        }
        total += h;
        if (P.counts && it < P.items) atomicAdd(P.counts + i, (unsigned long long)h);
    }
    block_reduce_add(total, P.hits);
}

template <int KIND>
cudaError_t ensure_smem_attr()
{
    static std::atomic<uint64_t> done{0};
    cudaError_t e = ensure_dyn_smem(mrg_fill_vec_kernel<KIND, false>, mrg_fill_smem(256, KIND), done);
    static std::atomic<uint64_t> done_sf{0};
    if (e == cudaSuccess) e = ensure_dyn_smem(mrg_fill_vec_kernel<KIND, true>, mrg_fill_smem(256, KIND), done_sf);
    return e;
}

template <int KIND>
cudaError_t launch_vec(const MrgLaunch& p, Grid g, cudaStream_t s)
{
    const cudaError_t e = ensure_smem_attr<KIND>();
    if (e != cudaSuccess) return e;
    if (p.seg_fastest) mrg_fill_vec_kernel<KIND, true><<<g.blocks, g.threads, mrg_fill_smem((int)g.threads, KIND), s>>>(p);
    else mrg_fill_vec_kernel<KIND, false><<<g.blocks, g.threads, mrg_fill_smem((int)g.threads, KIND), s>>>(p);
    return cudaGetLastError();
}

}  // namespace

size_t mrg_fill_tma_smem(int threads) { return (size_t)(threads / 32) * 4096 * kTmaBufs + 1024; }

namespace {
// Opt the TMA fills into their dynamic shared memory (> 48 KB with two
// boxes per warp) once per device.
cudaError_t ensure_tma_smem(int threads)
{
    const size_t sm = mrg_fill_tma_smem(threads);
    static std::atomic<uint64_t> d[6];
    cudaError_t e = ensure_dyn_smem(mrg_fill_tma_kernel<kU32, false>, sm, d[0]);
    if (e == cudaSuccess) e = ensure_dyn_smem(mrg_fill_tma_kernel<kU32, true>, sm, d[1]);
    if (e == cudaSuccess) e = ensure_dyn_smem(mrg_fill_tma_kernel<kF32, false>, sm, d[2]);
    if (e == cudaSuccess) e = ensure_dyn_smem(mrg_fill_tma_kernel<kF32, true>, sm, d[3]);
    if (e == cudaSuccess) e = ensure_dyn_smem(mrg_fill_tma_kernel<kF64, false>, sm, d[4]);
    if (e == cudaSuccess) e = ensure_dyn_smem(mrg_fill_tma_kernel<kF64, true>, sm, d[5]);
    return e;
}
}  // namespace

bool mrg_fill_tma_fits(int threads) { return mrg_fill_tma_smem(threads) <= 227u * 1024u; }

cudaError_t launch_mrg_fill_tma(const MrgLaunch& p, const CUtensorMap& tmap, int kind, Grid g, cudaStream_t s)
{
    const size_t sm = mrg_fill_tma_smem((int)g.threads);
    const cudaError_t e = ensure_tma_smem((int)g.threads);
    if (e != cudaSuccess) return e;
    if (kind == kF64) {
        if (p.seg_fastest) mrg_fill_tma_kernel<kF64, true><<<g.blocks, g.threads, sm, s>>>(p, tmap);
        else mrg_fill_tma_kernel<kF64, false><<<g.blocks, g.threads, sm, s>>>(p, tmap);
    } else if (kind == kF32) {
        if (p.seg_fastest) mrg_fill_tma_kernel<kF32, true><<<g.blocks, g.threads, sm, s>>>(p, tmap);
        else mrg_fill_tma_kernel<kF32, false><<<g.blocks, g.threads, sm, s>>>(p, tmap);
    } else {
        if (p.seg_fastest) mrg_fill_tma_kernel<kU32, true><<<g.blocks, g.threads, sm, s>>>(p, tmap);
        else mrg_fill_tma_kernel<kU32, false><<<g.blocks, g.threads, sm, s>>>(p, tmap);
    }
    return cudaGetLastError();
}


size_t mrg_fill_rows_smem(int threads) { return mrg_fill_tma_smem(threads) + 33 * kLaneTabEntries * 8; }

namespace {
cudaError_t ensure_rows_smem(int threads)
{
    const size_t sm = mrg_fill_rows_smem(threads);
    static std::atomic<uint64_t> d[6];
    cudaError_t e = ensure_dyn_smem(mrg_fill_rows_kernel<kU32, false>, sm, d[0]);
    if (e == cudaSuccess) e = ensure_dyn_smem(mrg_fill_rows_kernel<kF32, false>, sm, d[1]);
    if (e == cudaSuccess) e = ensure_dyn_smem(mrg_fill_rows_kernel<kU32, true>, sm, d[2]);
    if (e == cudaSuccess) e = ensure_dyn_smem(mrg_fill_rows_kernel<kF32, true>, sm, d[3]);
    if (e == cudaSuccess) e = ensure_dyn_smem(mrg_fill_rows_kernel<kF64, false>, sm, d[4]);
    if (e == cudaSuccess) e = ensure_dyn_smem(mrg_fill_rows_kernel<kF64, true>, sm, d[5]);
    return e;
}
}  // namespace

cudaError_t launch_mrg_fill_rows(const MrgRowsLaunch& p, const CUtensorMap& tmap, int kind, Grid g, cudaStream_t s)
{
    const size_t sm = mrg_fill_rows_smem((int)g.threads);
    const cudaError_t e = ensure_rows_smem((int)g.threads);
    if (e != cudaSuccess) return e;
    if (p.nh) {
        if (kind == kF64) mrg_fill_rows_kernel<kF64, true><<<g.blocks, g.threads, sm, s>>>(p, tmap);
        else if (kind == kF32) mrg_fill_rows_kernel<kF32, true><<<g.blocks, g.threads, sm, s>>>(p, tmap);
        else mrg_fill_rows_kernel<kU32, true><<<g.blocks, g.threads, sm, s>>>(p, tmap);
    } else {
        if (kind == kF64) mrg_fill_rows_kernel<kF64, false><<<g.blocks, g.threads, sm, s>>>(p, tmap);
        else if (kind == kF32) mrg_fill_rows_kernel<kF32, false><<<g.blocks, g.threads, sm, s>>>(p, tmap);
        else mrg_fill_rows_kernel<kU32, false><<<g.blocks, g.threads, sm, s>>>(p, tmap);
    }
    return cudaGetLastError();
}

size_t mrg_fill_smem(int threads, int kind)
{
    const bool staged = kind == kU32 ? mrg_staged<kU32>() : kind == kF32 ? mrg_staged<kF32>() : mrg_staged<kF64>();
    return staged ? staged_smem(threads) : 0;
}

cudaError_t upload_jump_tables(const MatPair* sub51, const MatPair* str64, const MatPair* draw64)
{
    MatPair h[3][64] = {};
    for (int b = 0; b < 51; ++b) h[0][b] = sub51[b];
    for (int b = 0; b < 64; ++b) h[1][b] = str64[b];
    for (int b = 0; b < 64; ++b) h[2][b] = draw64[b];
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

cudaError_t mrg_occupancy(int kernel, int kind, bool fast, int threads, int* out)
{
    switch (kernel) {
    case kKSeed:
        return occ(mrg_seed_kernel, threads, 0, out);
    case kKMrgFill: {
        const size_t sm = fast ? mrg_fill_smem(threads, kind) : 0;
        if (fast) {
            const cudaError_t e = kind == kU32 ? ensure_smem_attr<kU32>()
                                : kind == kF32 ? ensure_smem_attr<kF32>() : ensure_smem_attr<kF64>();
            if (e != cudaSuccess) return e;
        }
        if (kind == kU32) return fast ? occ(mrg_fill_vec_kernel<kU32, false>, threads, sm, out)
                                      : occ(mrg_fill_scalar_kernel<kU32>, threads, 0, out);
        if (kind == kF32) return fast ? occ(mrg_fill_vec_kernel<kF32, false>, threads, sm, out)
                                      : occ(mrg_fill_scalar_kernel<kF32>, threads, 0, out);
        return fast ? occ(mrg_fill_vec_kernel<kF64, false>, threads, sm, out)
                    : occ(mrg_fill_scalar_kernel<kF64>, threads, 0, out);
    }
    case kKMrgMc:
        return occ(mrg_mc_kernel, threads, 0, out);
    case kKMrgFillRows: {
        const size_t sm = mrg_fill_rows_smem(threads);
        if (sm > 227u * 1024u) {
            *out = 0;
            return cudaSuccess;
        }
        if (const cudaError_t e = ensure_rows_smem(threads); e != cudaSuccess) return e;
        return kind == kF64   ? occ(mrg_fill_rows_kernel<kF64, false>, threads, sm, out)
               : kind == kF32 ? occ(mrg_fill_rows_kernel<kF32, false>, threads, sm, out)
                              : occ(mrg_fill_rows_kernel<kU32, false>, threads, sm, out);
    }
    case kKMrgFillTma: {
        const size_t sm = mrg_fill_tma_smem(threads);
        if (!mrg_fill_tma_fits(threads)) {
            *out = 0;
            return cudaSuccess;
        }
        if (const cudaError_t e = ensure_tma_smem(threads); e != cudaSuccess) return e;
        if (kind == kU32) return occ(mrg_fill_tma_kernel<kU32, false>, threads, sm, out);
        if (kind == kF32) return occ(mrg_fill_tma_kernel<kF32, false>, threads, sm, out);
        return occ(mrg_fill_tma_kernel<kF64, false>, threads, sm, out);
    }
    }
    return cudaErrorInvalidValue;
}

}  // namespace shv
