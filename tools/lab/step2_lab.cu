// step2_lab.cu — compute-only throughput (no stores) of the MRG32k3a step
// formulations in include/shv_device.cuh: MrgFF (both components, floor
// reductions), MrgIF (component 1 integer, component 2 floor) and the
// all-integer step, with the constants as immediates or read from the
// parameter block; 1 or 2 streams per thread. Checks that every variant gives
// the integer step's sequence.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "lab_variants.cuh"
using namespace shv::dev;

constexpr int ITER = 1024;  // x 8 steps

struct KP { double v[6]; uint32_t a12, a13n; };
__device__ __forceinline__ MrgFpK kp(const KP& p) { return MrgFpK{p.v[0], p.v[1], p.v[2], p.v[3], p.v[4], p.v[5], p.a12, p.a13n}; }

__device__ __forceinline__ Mrg seed_of(uint32_t t)
{
    return Mrg{12345u + t, 12345u, 12345u ^ t, 12345u, 777u + t, 12345u};
}
__device__ __forceinline__ uint32_t nx(Mrg& s, const MrgFpK& K) { return mrg_next(s, K); }
__device__ __forceinline__ uint32_t nx(MrgFF& s, const MrgFpK& K) { return mrg_next(s, K); }
__device__ __forceinline__ uint32_t nx(MrgIF& s, const MrgFpK& K) { return mrg_next(s, K); }
template <int M> __device__ __forceinline__ uint32_t nx(MrgFW<M>& s, const MrgFpK& K) { return mrg_next(s, K); }
template <class G> __device__ __forceinline__ G mk(const Mrg& s);
template <> __device__ __forceinline__ Mrg mk<Mrg>(const Mrg& s) { return s; }
template <> __device__ __forceinline__ MrgFF mk<MrgFF>(const Mrg& s) { return to_mrg_ff(s); }
template <> __device__ __forceinline__ MrgIF mk<MrgIF>(const Mrg& s) { return to_mrg_if(s); }
template <> __device__ __forceinline__ MrgFW<1> mk<MrgFW<1>>(const Mrg& s) { return to_mrg_fw<1>(s); }
template <> __device__ __forceinline__ MrgFW<2> mk<MrgFW<2>>(const Mrg& s) { return to_mrg_fw<2>(s); }
template <> __device__ __forceinline__ MrgFW<3> mk<MrgFW<3>>(const Mrg& s) { return to_mrg_fw<3>(s); }

// PK: constants from the parameter block (1) or immediates (0); S streams per thread
template <class G, int PK, int S>
__global__ void __launch_bounds__(256) k_step(uint32_t* out, const __grid_constant__ KP p, int iters)
{
    const MrgFpK K = PK ? kp(p) : mrg_fpk();
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    G s[S];
#pragma unroll
    for (int j = 0; j < S; ++j) s[j] = mk<G>(seed_of(t * S + j));
    uint32_t acc[S] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int j = 0; j < S; ++j) acc[j] ^= nx(s[j], K) * (2u * u + 1u);
    }
#pragma unroll
    for (int j = 0; j < S; ++j) out[t * S + j] = acc[j];
}

// Mixed warps: warp w runs the integer step if w % R == R - 1, else MrgFF
// (the FP64 pipe and the FMA-heavy/ALU pipes work side by side on one SMSP).
template <int R>
__global__ void __launch_bounds__(256) k_mixed(uint32_t* out, const __grid_constant__ KP p, int iters, int iters_int)
{
    const MrgFpK K = kp(p);
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    if ((t >> 5) % R == R - 1) {
        Mrg s = seed_of(t);
        for (int i = 0; i < iters_int; ++i)
#pragma unroll
            for (int u = 0; u < 8; ++u) acc ^= nx(s, K) * (2u * u + 1u);
    } else {
        MrgFF s = mk<MrgFF>(seed_of(t));
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int u = 0; u < 8; ++u) acc ^= nx(s, K) * (2u * u + 1u);
    }
    out[t] = acc;
}

template <class F> float tms(F f) { cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); f(); cudaDeviceSynchronize();
    float best = 1e30f; for (int r = 0; r < 5; ++r) { cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; } return best; }

int main()
{
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    KP p{{6755399441055744.0, 1.0 / 4294967087.0, 0x1.000059451f212p-32, 4294967087.0, 4294944443.0, 5886603609186927.0}, 1403580u, 810728u};
    const int thr = 256;
    const size_t maxn = (size_t)sms * 16 * thr * 2;
    uint32_t *ref, *o; cudaMalloc(&ref, maxn * 4); cudaMalloc(&o, maxn * 4);
    uint32_t* h1 = new uint32_t[maxn]; uint32_t* h2 = new uint32_t[maxn];
    printf("[");
    bool first = true;
    auto run = [&](const char* name, auto kern, int S, int blocks_per_sm) {
        const int blocks = sms * blocks_per_sm;
        const size_t n = (size_t)blocks * thr * S;
        k_step<Mrg, 0, 1><<<(unsigned)(n / thr), thr>>>(ref, p, ITER);
        float ms = tms([&] { kern<<<blocks, thr>>>(o, p, ITER); });
        cudaMemcpy(h1, ref, n * 4, cudaMemcpyDeviceToHost); cudaMemcpy(h2, o, n * 4, cudaMemcpyDeviceToHost);
        size_t bad = 0; for (size_t i = 0; i < n; ++i) bad += h1[i] != h2[i];
        int occ; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, thr, 0);
        cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, kern);
        printf("%s{\"v\": \"%s\", \"bps\": %d, \"occ\": %d, \"regs\": %d, \"Tnum_s\": %.4f, \"mismatch\": %zu}\n", first ? "" : ",", name,
               blocks_per_sm, occ, fa.numRegs, (double)n * ITER * 8 / (ms * 1e-3) / 1e12, bad);
        first = false;
    };
    for (int bps : {4, 8}) {
        run("int", k_step<Mrg, 0, 1>, 1, bps);
        run("int_par", k_step<Mrg, 1, 1>, 1, bps);
        run("FF_imm", k_step<MrgFF, 0, 1>, 1, bps);
        run("FF_par", k_step<MrgFF, 1, 1>, 1, bps);
        run("FF_par_x2", k_step<MrgFF, 1, 2>, 2, bps);
        run("FW1_par", k_step<MrgFW<1>, 1, 1>, 1, bps);
        run("FW2_par", k_step<MrgFW<2>, 1, 1>, 1, bps);
        run("FW3_par", k_step<MrgFW<3>, 1, 1>, 1, bps);
        run("IF_imm", k_step<MrgIF, 0, 1>, 1, bps);
        run("IF_par", k_step<MrgIF, 1, 1>, 1, bps);
        run("IF_par_x2", k_step<MrgIF, 1, 2>, 2, bps);
    }
    printf("]\n");
    return 0;
}
