// kernels_audit.cu — disjointness audit of generated rows on the GPU
// (SPEC verify_disjoint, S L407-415, L425-426): every
// window of 4 consecutive draws of every PE row is put in an open-addressing
// hash table in HBM; a window value held by two different PEs is a collision.
//
// The result is defined by the rows alone, not by the order in which threads
// reach the table (S "internally parallel with deterministic merge"):
//   pass 1 (insert)  one slot per distinct window value; the slot keeps the
//                    smallest occurrence code c = pe*horizon + pos (atomicMin),
//                    which orders occurrences as (pe, pos) lexicographically;
//   pass 2 (second)  every occurrence whose PE differs from the slot minimum's
//                    PE does atomicMin into the slot's second word: the
//                    smallest occurrence in the next-smallest PE;
//   pass 3 (reduce)  over slots with a second occurrence: count them and take
//                    the smallest first occurrence (unique per slot);
//   pass 4 (final)   one thread re-probes that window for its second word and
//                    writes the report.
// Slot word = (24-bit fingerprint << 40) | code, EMPTY = ~0: probes compare
// fingerprints and load the 16 bytes of a candidate window only on a
// fingerprint match. Occurrences of one value share the fingerprint, so
// atomicMin on the packed word is atomicMin on the code. Linear probing
// without deletion: a value's slot is reached before any empty slot.
//
// Roofline: random 32-byte sectors (one table probe + one row read per
// window per pass on average at load <= 1/2), not streaming bandwidth.
#include <cstdint>
#include <cuda_runtime.h>

#include "shv_internal.h"

namespace shv {
namespace {

constexpr unsigned long long kEmpty = ~0ull;
constexpr unsigned long long kCodeMask = (1ull << 40) - 1;

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

__device__ __forceinline__ uint64_t home(uint64_t x, uint64_t cap) { return __umul64hi(x, cap); }
__device__ __forceinline__ uint64_t fp_of(uint64_t x) { return (x & 0xFFFFFFull) << 40; }

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

__global__ void __launch_bounds__(256) audit_insert_kernel(AuditLaunch p)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < p.windows; w += stride) {
        const uint64_t c = code_of(w, p.wpr, p.horizon);
        const Win v = load_win(p.rows, c);
        const uint64_t x = mix(v);
        const unsigned long long mine = fp_of(x) | c;
        uint64_t i = home(x, p.cap);
        for (;;) {
            unsigned long long cur = ld_slot(p.slots + i);
            if (cur == kEmpty) {
                cur = atomicCAS(p.slots + i, kEmpty, mine);
                if (cur == kEmpty) break;
            }
            if ((cur & ~kCodeMask) == fp_of(x) && same(load_win(p.rows, cur & kCodeMask), v)) {
                if (mine < cur) atomicMin(p.slots + i, mine);
                break;
            }
            if (++i == p.cap) i = 0;
        }
    }
}

__global__ void __launch_bounds__(256) audit_second_kernel(AuditLaunch p)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < p.windows; w += stride) {
        const uint64_t c = code_of(w, p.wpr, p.horizon);
        const Win v = load_win(p.rows, c);
        const uint64_t x = mix(v);
        uint64_t i = home(x, p.cap);
        for (;;) {
            const unsigned long long cur = p.slots[i];  // final after pass 1
            if ((cur & ~kCodeMask) == fp_of(x)) {
                const uint64_t m1 = cur & kCodeMask;
                if (m1 == c) break;  // the value's smallest occurrence itself
                if (same(load_win(p.rows, m1), v)) {
                    if (c / p.horizon != m1 / p.horizon) atomicMin(p.second + i, (unsigned long long)c);
                    break;
                }
            }
            if (++i == p.cap) i = 0;
        }
    }
}

__device__ __forceinline__ unsigned long long warp_min(unsigned long long v)
{
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, v, d);
        v = o < v ? o : v;
    }
    return v;
}

__global__ void __launch_bounds__(256) audit_reduce_kernel(AuditLaunch p)
{
    __shared__ unsigned long long smin[8];
    __shared__ unsigned long long scnt[8];
    unsigned long long best = kEmpty, cnt = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.cap; i += stride) {
        if (p.second[i] != kEmpty) {
            const unsigned long long a = p.slots[i] & kCodeMask;
            best = a < best ? a : best;
            ++cnt;
        }
    }
    best = warp_min(best);
#pragma unroll
    for (int d = 16; d; d >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
    const unsigned wid = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (lane == 0) {
        smin[wid] = best;
        scnt[wid] = cnt;
    }
    __syncthreads();
    if (wid == 0) {
        best = lane < blockDim.x / 32 ? smin[lane] : kEmpty;
        cnt = lane < blockDim.x / 32 ? scnt[lane] : 0;
        best = warp_min(best);
#pragma unroll
        for (int d = 16; d; d >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
        if (lane == 0 && cnt) {
            atomicMin(reinterpret_cast<unsigned long long*>(&p.report->pe_a), best);  // holds the code until audit_final
            atomicAdd(reinterpret_cast<unsigned long long*>(&p.report->colliding), cnt);
        }
    }
}

__global__ void audit_init_kernel(AuditLaunch p)
{
    shv_disjoint_report* r = p.report;
    r->disjoint = 1;
    r->windows = p.windows;
    r->colliding = 0;
    r->pe_a = r->pos_a = r->pe_b = r->pos_b = kEmpty;
}

__global__ void audit_final_kernel(AuditLaunch p)
{
    shv_disjoint_report* r = p.report;
    const uint64_t a = r->pe_a;
    if (a == kEmpty) return;
    const Win v = load_win(p.rows, a);
    uint64_t i = home(mix(v), p.cap);
    while ((p.slots[i] & kCodeMask) != a)
        if (++i == p.cap) i = 0;
    const uint64_t b = p.second[i];
    r->disjoint = 0;
    r->pe_a = a / p.horizon;
    r->pos_a = a % p.horizon;
    r->pe_b = b / p.horizon;
    r->pos_b = b % p.horizon;
}

}  // namespace

cudaError_t launch_audit(const AuditLaunch& p, unsigned blocks, cudaStream_t s)
{
    audit_init_kernel<<<1, 1, 0, s>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || p.windows == 0) return e;
    e = cudaMemsetAsync(p.slots, 0xFF, p.cap * sizeof(unsigned long long), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(p.second, 0xFF, p.cap * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    audit_insert_kernel<<<blocks, 256, 0, s>>>(p);
    audit_second_kernel<<<blocks, 256, 0, s>>>(p);
    audit_reduce_kernel<<<blocks, 256, 0, s>>>(p);
    audit_final_kernel<<<1, 1, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace shv
