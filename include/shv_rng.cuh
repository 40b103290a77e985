/*
 * shv_rng.cuh — device-side generator objects for user kernels: the paper's
 * device API (P L387-399 [§5.2]: "create an instance of the PRNG you want to
 * use and let its class' constructor do the rest ... pick random numbers by
 * calling the next() method"; Listing 1, P L485-490).
 *
 *   __global__ void fooKernel(float* ddata, shv_device_view v) {   // Listing 1
 *       const uint64_t i = blockDim.x * blockIdx.x + threadIdx.x;
 *       shv::Rng<SHV_GEN_MRG32K3A> rng(v, i);
 *       ddata[i] = rng.next_f32();
 *   }
 *   // host: h = shv_streams_create(...block_num * thread_num streams...);
 *   //       shv_get_device_view(h, &v); fooKernel<<<block_num, thread_num>>>(d, v);
 *   //       shv_jump(h, SHV_JUMP_DRAWS, draws_per_thread, stream); ...; shv_streams_destroy(h);
 *
 * Thread i's sequence is stream i of the handle at the view's offset, value
 * for value the one shv_generate_u32/f32/f64 writes (R7, R8); the state lives
 * in registers. The arithmetic is shv_device.cuh's (MRG32k3a on the FP64 pipe in
 * the subnormal range,
 * Philox4x32-10 with the warp-uniform key schedule when keys are shared).
 */
#pragma once
#include "shv.h"
#include "shv_device.cuh"

namespace shv {

template <int GEN>
class Rng;

template <>
class Rng<SHV_GEN_MRG32K3A> {
public:
    // Stream i: its start state (offset 0) jumped by the view's A^o.
    __device__ Rng(const shv_device_view& v, uint64_t i)
    {
        const uint32_t* st = v.state;
        const uint64_t n = v.n_streams;
        dev::Mrg m{st[i], st[n + i], st[2 * n + i], st[3 * n + i], st[4 * n + i], st[5 * n + i]};
        dev::apply(v.jump, v.jump + 9, m);
        s_ = dev::to_mrg_mf(m);
    }
    // z in [1, m1]; the row-tile fill's step (MrgMF: subnormal-range state, magic-free quotients)
    __device__ uint32_t next_u32() { return dev::mrg_next(s_); }
    __device__ float next_f32() { return dev::to_f32(next_u32()); }
    __device__ double next_f64() { return dev::mrg_f64(next_u32()); }

private:
    dev::MrgMF s_;
};

template <>
class Rng<SHV_GEN_PHILOX4X32_10> {
public:
    __device__ Rng(const shv_device_view& v, uint64_t i)
    {
        if (v.spacing == SHV_SPACING_KEYED) {
            k0_ = (uint32_t)(v.first_stream + i);
            k1_ = v.key1;
            g_ = 0;
        } else {
            k0_ = v.key0;
            k1_ = v.key1;
            g_ = v.first_stream + i;
        }
        blk_ = (v.offset_lo >> 2) | (v.offset_hi << 62);  // draw o -> block o/4, lane o%4
        lane_ = (uint32_t)(v.offset_lo & 3);
        buf_ = dev::philox_blk(blk_, g_, k0_, k1_);
    }
    __device__ uint32_t next_u32()
    {
        if (lane_ == 4) {
            ++blk_;
            buf_ = dev::philox_blk(blk_, g_, k0_, k1_);
            lane_ = 0;
        }
        return dev::lane_of(buf_, lane_++);
    }
    __device__ float next_f32() { return dev::to_f32(next_u32()); }
    __device__ double next_f64()  // two draws per value (R7)
    {
        const uint32_t lo = next_u32();
        return dev::philox_f64(lo, next_u32());
    }

private:
    uint32_t k0_, k1_;
    uint64_t g_, blk_;
    uint32_t lane_;
    dev::W4 buf_;
};

template <>
class Rng<SHV_GEN_THREEFRY4X64_20> {
public:
    __device__ Rng(const shv_device_view& v, uint64_t i)
        : k0_((uint64_t)v.key0 | ((uint64_t)v.key1 << 32)), k1_((uint64_t)v.key2 | ((uint64_t)v.key3 << 32)),
          g_(v.first_stream + i), blk_((v.offset_lo >> 3) | (v.offset_hi << 61)), word_((uint32_t)(v.offset_lo & 7))
    {
        buf_ = dev::threefry20(blk_, g_, k0_, k1_);
    }
    __device__ uint32_t next_u32()
    {
        if (word_ == 8) {
            ++blk_;
            buf_ = dev::threefry20(blk_, g_, k0_, k1_);
            word_ = 0;
        }
        const uint32_t w = word_++;
        const uint64_t lane = (w >> 1) == 0 ? buf_.x : (w >> 1) == 1 ? buf_.y : (w >> 1) == 2 ? buf_.z : buf_.w;
        return (w & 1) ? (uint32_t)(lane >> 32) : (uint32_t)lane;
    }
    __device__ float next_f32() { return dev::to_f32(next_u32()); }
    __device__ double next_f64()
    {
        const uint32_t lo = next_u32();
        return dev::philox_f64(lo, next_u32());
    }

private:
    uint64_t k0_, k1_, g_, blk_;
    uint32_t word_;
    dev::Q4 buf_;
};

template <>
class Rng<SHV_GEN_TINYMT32> {
public:
    // Stream i: its current state (TinyMT handles are stateful) and the
    // parameter set of its group.
    __device__ Rng(const shv_device_view& v, uint64_t i)
    {
        const uint32_t* st = v.state;
        const uint64_t n = v.n_streams;
        const uint32_t* pr = v.params + 3 * ((v.first_stream + i) / v.group_size - v.group0);
        t_ = dev::TinyMT{st[i], st[n + i], st[2 * n + i], st[3 * n + i], pr[0], pr[1], pr[2]};
    }
    __device__ uint32_t next_u32() { return dev::tinymt_next(t_); }
    __device__ float next_f32() { return dev::to_f32(next_u32()); }
    __device__ double next_f64()
    {
        const uint32_t lo = next_u32();
        return dev::philox_f64(lo, next_u32());
    }

private:
    dev::TinyMT t_;
};

}  // namespace shv
