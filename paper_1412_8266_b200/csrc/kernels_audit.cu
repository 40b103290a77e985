// kernels_audit.cu — disjointness audit of generated rows on the GPU
// (SPEC verify_disjoint, S L407-415, L425-426): every
// window of 4 consecutive draws of every PE row is hashed; a window value held
// by two different PEs is a collision.
//
// Radix-partitioned hash aggregation, so that the hash
// tables stay L2-resident instead of turning every probe into a random HBM
// access:
//   count    hash every window (64-bit mix of its 4 words); bucket = top
//            log2(P) bits; per-CTA shared-memory histogram, one global add
//            per CTA and bucket;
//   scan     bucket offsets for the records and the tables (bucket b's table
//            has 2*count_b + 1 slots: load <= 1/2);
//   scatter  per CTA tile of 8192 windows: histogram again, reserve a run in
//            each bucket with one global atomicAdd, stage the tile's 16-byte
//            records (hash, code) in shared memory sorted by bucket, and write
//            each run with coalesced stores;
//   insert   records in bucket order, so the few tables in use at any time
//            sit in L2: open addressing, linear probing inside the bucket's
//            table; slot word = (23-bit fingerprint << 40) | code, code =
//            pe*horizon + pos, whose numeric order is (pe, pos) order; CAS on
//            empty slots, atomicMin among equal windows (the slot ends with
//            the smallest occurrence of its value);
//   second   each record finds its slot again; an occurrence whose PE differs
//            from the slot minimum's flags the slot (bit 63; first setter
//            counts a colliding value), lowers the global minimum first
//            occurrence a, and appends (slot, code) to a candidate list;
//   cand     over the candidates of a's slot: the smallest code b;
//   final    one thread writes the report.
// Window data are read only to hash (sequentially) and to confirm a
// fingerprint match (true duplicates; rare otherwise). The result is defined
// by the rows alone, not by the order in which threads meet (S L429).
#include <cstdint>
#include <cuda_runtime.h>

#include "shv_internal.h"

namespace shv {
namespace {

constexpr unsigned long long kEmpty = ~0ull;
constexpr unsigned long long kCodeMask = (1ull << 40) - 1;
constexpr unsigned long long kFlag = 1ull << 63;
constexpr unsigned long long kFpMask = 0x7FFFFFull << 40;  // bits 40..62
constexpr unsigned kThreads = 256;

struct Win {
    uint32_t w[4];
};

__device__ __forceinline__ Win load_win(const uint32_t* __restrict__ rows, uint64_t c)
{
    const uint32_t* p = rows + c;
    return Win{{__ldg(p), __ldg(p + 1), __ldg(p + 2), __ldg(p + 3)}};
}

__device__ __forceinline__ bool same(const Win& a, const Win& b)
{
    return a.w[0] == b.w[0] && a.w[1] == b.w[1] && a.w[2] == b.w[2] && a.w[3] == b.w[3];
}

// 64-bit mix of the window (multiply-xorshift, as in SplitMix64's finalizer).
__device__ __forceinline__ uint64_t mix(const Win& v)
{
    uint64_t a = ((uint64_t)v.w[1] << 32 | v.w[0]) * 0x9E3779B97F4A7C15ull;
    uint64_t b = ((uint64_t)v.w[3] << 32 | v.w[2]) * 0xC2B2AE3D27D4EB4Full;
    uint64_t x = a ^ ((b << 31) | (b >> 33));
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

__device__ __forceinline__ uint32_t bucket_of(uint64_t x, uint32_t lg) { return lg ? (uint32_t)(x >> (64 - lg)) : 0u; }
__device__ __forceinline__ uint64_t fp_of(uint64_t x) { return (x << 40) & kFpMask; }
// home slot inside a bucket table of cap slots: the hash bits below the bucket bits
__device__ __forceinline__ uint64_t home(uint64_t x, uint32_t lg, uint64_t cap) { return __umul64hi(x << lg, cap); }

__device__ __forceinline__ unsigned long long ld_slot(const unsigned long long* p)
{
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

// Window w (w < n_pe * wpr) -> occurrence code pe*horizon + pos.
__device__ __forceinline__ uint64_t code_of(uint64_t w, uint64_t wpr, uint64_t horizon)
{
    const uint64_t pe = w / wpr;
    return pe * horizon + (w - pe * wpr);
}

// Walks windows w0, w0 + step, ... as (pe, pos) without a 64-bit division per
// window (one at the start, then carries).
struct WinWalk {
    uint64_t pe, pos;
    __device__ __forceinline__ WinWalk(uint64_t w0, uint64_t wpr) : pe(w0 / wpr), pos(w0 - (w0 / wpr) * wpr) {}
    __device__ __forceinline__ uint64_t code(uint64_t horizon) const { return pe * horizon + pos; }
    __device__ __forceinline__ void advance(uint64_t step, uint64_t wpr)
    {
        pos += step;
        while (pos >= wpr) {
            pos -= wpr;
            ++pe;
        }
    }
};

__global__ void __launch_bounds__(kThreads) audit_count_kernel(AuditLaunch p)
{
    extern __shared__ uint32_t hist[];
    for (uint32_t b = threadIdx.x; b < p.nb; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < p.windows; w += stride)
        atomicAdd(&hist[bucket_of(mix(load_win(p.rows, code_of(w, p.wpr, p.horizon))), p.lgb)], 1u);
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < p.nb; b += blockDim.x)
        if (hist[b]) atomicAdd(p.count + b, (unsigned long long)hist[b]);
}

// One block: exclusive scans of the bucket counts (records, tables).
__global__ void __launch_bounds__(1024) audit_scan_kernel(AuditLaunch p)
{
    __shared__ unsigned long long part[1024];
    const uint32_t per = (p.nb + blockDim.x - 1) / blockDim.x;
    const uint32_t b0 = threadIdx.x * per, b1 = min(p.nb, b0 + per);
    unsigned long long s = 0;
    for (uint32_t b = b0; b < b1; ++b) s += p.count[b];
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long acc = 0;
        for (uint32_t t = 0; t < blockDim.x; ++t) {
            const unsigned long long v = part[t];
            part[t] = acc;
            acc += v;
        }
    }
    __syncthreads();
    unsigned long long r = part[threadIdx.x];
    for (uint32_t b = b0; b < b1; ++b) {
        p.rec_off[b] = r;
        p.cursor[b] = r;
        p.tab_off[b] = 2 * r + b;  // 2*count + 1 slots per bucket
        r += p.count[b];
    }
}

// Scatter: one CTA tile of kSTile windows at a time, staged in shared memory
// sorted by bucket so that each bucket's run leaves as one coalesced write
// (scattering records straight from the hashing threads left ~2.4M partially
// written sectors open in L2 and doubled the DRAM traffic by read-modify-write).
#ifndef SHV_AUDIT_STILE
#define SHV_AUDIT_STILE 8192  // 4096 / 2048 (two / four CTAs per SM) measured no faster
#endif
constexpr uint32_t kSTile = SHV_AUDIT_STILE;
constexpr unsigned kSThreads = 512;

// Exclusive scan of v[0..n) in shared memory (n <= 4 * blockDim.x), into out.
__device__ __forceinline__ void block_exclusive_scan(const uint32_t* v, uint32_t* out, uint32_t n)
{
    __shared__ uint32_t warp_tot[32];
    const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
    const uint32_t b0 = threadIdx.x * per;
    uint32_t loc = 0;
    for (uint32_t k = 0; k < per; ++k)
        if (b0 + k < n) loc += v[b0 + k];
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t incl = loc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= (unsigned)d) incl += o;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const unsigned nw = blockDim.x >> 5;
        uint32_t t = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, t, d);
            if (lane >= (unsigned)d) t += o;
        }
        if (lane < nw) warp_tot[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    uint32_t run = incl - loc + (wid ? warp_tot[wid - 1] : 0);
    for (uint32_t k = 0; k < per; ++k)
        if (b0 + k < n) {
            out[b0 + k] = run;
            run += v[b0 + k];
        }
    __syncthreads();
}

__global__ void __launch_bounds__(kSThreads) audit_scatter_kernel(AuditLaunch p)
{
    extern __shared__ unsigned long long sm64[];
    unsigned long long* srec = sm64;                              // 2 * kSTile: (hash, code), bucket order
    unsigned long long* base = srec + 2 * kSTile;                 // nb: global run start per bucket
    uint32_t* hist = reinterpret_cast<uint32_t*>(base + p.nb);    // nb: counts, then ranks
    uint32_t* loff = hist + p.nb;                                 // nb: local exclusive offsets
    const uint64_t ntiles = (p.windows + kSTile - 1) / kSTile;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t w0 = tile * kSTile, w1 = min(p.windows, w0 + kSTile);
        const uint32_t cnt = (uint32_t)(w1 - w0);
        for (uint32_t b = threadIdx.x; b < p.nb; b += blockDim.x) hist[b] = 0;
        __syncthreads();
        const WinWalk start(w0 + threadIdx.x, p.wpr);
        WinWalk ww = start;
        for (uint64_t w = w0 + threadIdx.x; w < w1; w += blockDim.x, ww.advance(blockDim.x, p.wpr))
            atomicAdd(&hist[bucket_of(mix(load_win(p.rows, ww.code(p.horizon))), p.lgb)], 1u);
        __syncthreads();
        block_exclusive_scan(hist, loff, p.nb);
        for (uint32_t b = threadIdx.x; b < p.nb; b += blockDim.x) {
            const uint32_t c = hist[b];
            base[b] = c ? atomicAdd(p.cursor + b, (unsigned long long)c) : 0ull;
            hist[b] = 0;
        }
        __syncthreads();
        ww = start;
        for (uint64_t w = w0 + threadIdx.x; w < w1; w += blockDim.x, ww.advance(blockDim.x, p.wpr)) {
            const uint64_t c = ww.code(p.horizon);
            const uint64_t x = mix(load_win(p.rows, c));
            const uint32_t b = bucket_of(x, p.lgb);
            const uint32_t at = loff[b] + atomicAdd(&hist[b], 1u);
            srec[2 * at] = x;
            srec[2 * at + 1] = c;
        }
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
            const unsigned long long x = srec[2 * i];
            const uint32_t b = bucket_of(x, p.lgb);
            const uint64_t g = base[b] + (i - loff[b]);
            p.rec[2 * g] = x;
            p.rec[2 * g + 1] = srec[2 * i + 1];
        }
        __syncthreads();
    }
}

// Records are taken in chunks from a global queue in increasing order, so the
// records in flight (CTAs x kChunk) span only a few buckets and their tables
// stay in L2; a grid-stride loop lets CTAs drift apart over a long run.
constexpr uint32_t kChunk = 1024;

__device__ __forceinline__ bool next_chunk(unsigned long long* q, uint64_t windows, uint64_t& r0)
{
    __shared__ unsigned long long s_r0;
    if (threadIdx.x == 0) s_r0 = atomicAdd(q, (unsigned long long)kChunk);
    __syncthreads();
    r0 = s_r0;
    __syncthreads();
    return r0 < windows;
}

__global__ void __launch_bounds__(kThreads) audit_insert_kernel(AuditLaunch p)
{
    uint64_t r0;
    while (next_chunk(p.scratch + 3, p.windows, r0))
    for (uint64_t r = r0 + threadIdx.x; r < min(p.windows, r0 + kChunk); r += blockDim.x) {
        const uint64_t x = p.rec[2 * r], c = p.rec[2 * r + 1];
        const uint32_t b = bucket_of(x, p.lgb);
        unsigned long long* tab = p.slots + p.tab_off[b];
        const uint64_t cap = 2 * p.count[b] + 1;
        const unsigned long long mine = fp_of(x) | c;
        uint64_t i = home(x, p.lgb, cap);
        Win v{};
        bool have = false;
        for (;;) {
            unsigned long long cur = ld_slot(tab + i);
            if (cur == kEmpty) {
                cur = atomicCAS(tab + i, kEmpty, mine);
                if (cur == kEmpty) break;
            }
            if ((cur & kFpMask) == fp_of(x)) {
                if (!have) {
                    v = load_win(p.rows, c);
                    have = true;
                }
                if (same(load_win(p.rows, cur & kCodeMask), v)) {
                    if (mine < cur) atomicMin(tab + i, mine);
                    break;
                }
            }
            if (++i == cap) i = 0;
        }
    }
}

__global__ void __launch_bounds__(kThreads) audit_second_kernel(AuditLaunch p)
{
    uint64_t r0;
    while (next_chunk(p.scratch + 4, p.windows, r0))
    for (uint64_t r = r0 + threadIdx.x; r < min(p.windows, r0 + kChunk); r += blockDim.x) {
        const uint64_t x = p.rec[2 * r], c = p.rec[2 * r + 1];
        const uint32_t b = bucket_of(x, p.lgb);
        unsigned long long* tab = p.slots + p.tab_off[b];
        const uint64_t cap = 2 * p.count[b] + 1;
        uint64_t i = home(x, p.lgb, cap);
        for (;;) {
            const unsigned long long cur = ld_slot(tab + i);  // final after insert; bit 63 may be set now
            if ((cur & kFpMask) == fp_of(x)) {
                const uint64_t m1 = cur & kCodeMask;
                if (m1 == c) break;  // the value's smallest occurrence itself
                if (same(load_win(p.rows, m1), load_win(p.rows, c))) {
                    if (c / p.horizon != m1 / p.horizon) {
                        const unsigned long long old = atomicOr(tab + i, kFlag);
                        if (!(old & kFlag)) atomicAdd(reinterpret_cast<unsigned long long*>(&p.report->colliding), 1ull);
                        atomicMin(&p.scratch[0], (unsigned long long)m1);
                        const unsigned long long k = atomicAdd(&p.scratch[2], 1ull);
                        p.cand[2 * k] = (unsigned long long)(tab + i - p.slots);
                        p.cand[2 * k + 1] = c;
                    }
                    break;
                }
            }
            if (++i == cap) i = 0;
        }
    }
}

// Candidates of the first colliding value a: its smallest other-PE occurrence.
__global__ void __launch_bounds__(kThreads) audit_cand_kernel(AuditLaunch p)
{
    const unsigned long long a = p.scratch[0], n = p.scratch[2];
    if (a == kEmpty) return;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride)
        if ((p.slots[p.cand[2 * k]] & kCodeMask) == a) atomicMin(&p.scratch[1], p.cand[2 * k + 1]);
}

__global__ void audit_init_kernel(AuditLaunch p)
{
    shv_disjoint_report* r = p.report;
    r->disjoint = 1;
    r->windows = p.windows;
    r->colliding = 0;
    r->pe_a = r->pos_a = r->pe_b = r->pos_b = kEmpty;
    if (p.scratch) {
        p.scratch[0] = kEmpty;  // smallest first occurrence of a colliding value
        p.scratch[1] = kEmpty;  // its smallest other-PE occurrence
        p.scratch[2] = 0;       // candidates
        p.scratch[3] = 0;       // insert queue
        p.scratch[4] = 0;       // second queue
    }
}

__global__ void audit_final_kernel(AuditLaunch p)
{
    const unsigned long long a = p.scratch[0], b = p.scratch[1];
    if (a == kEmpty) return;
    shv_disjoint_report* r = p.report;
    r->disjoint = 0;
    r->pe_a = a / p.horizon;
    r->pos_a = a % p.horizon;
    r->pe_b = b / p.horizon;
    r->pos_b = b % p.horizon;
}

}  // namespace

size_t audit_scatter_smem(uint32_t nb) { return (size_t)kSTile * 16 + (size_t)nb * 16; }

cudaError_t launch_audit(const AuditLaunch& p, unsigned blocks, cudaStream_t s)
{
    audit_init_kernel<<<1, 1, 0, s>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || p.windows == 0) return e;
    e = cudaMemsetAsync(p.count, 0, (size_t)p.nb * 8, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(p.slots, 0xFF, (size_t)(2 * p.windows + p.nb) * 8, s);
    if (e != cudaSuccess) return e;
    const size_t ssm = audit_scatter_smem(p.nb);
    if (ssm > 48 * 1024) {
        e = cudaFuncSetAttribute(audit_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
        if (e != cudaSuccess) return e;
    }
    audit_count_kernel<<<blocks, kThreads, (size_t)p.nb * 4, s>>>(p);
    audit_scan_kernel<<<1, 1024, 0, s>>>(p);
    const uint64_t ntiles = (p.windows + kSTile - 1) / kSTile;
    int dev = 0, sms = 0;
    e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, audit_scatter_kernel, kSThreads, ssm) != cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    const uint64_t sgrid = (uint64_t)sms * (uint64_t)per_sm;
    audit_scatter_kernel<<<(unsigned)(ntiles < sgrid ? ntiles : sgrid), kSThreads, ssm, s>>>(p);
    audit_insert_kernel<<<blocks, kThreads, 0, s>>>(p);
    audit_second_kernel<<<blocks, kThreads, 0, s>>>(p);
    audit_cand_kernel<<<blocks, kThreads, 0, s>>>(p);
    audit_final_kernel<<<1, 1, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace shv
