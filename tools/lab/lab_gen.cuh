// lab_gen.cuh — stand-in generators for the MRG fill kernels, compiled only
// into tools/lab builds (-DSHV_LAB_GEN_HEADER='"path"' -DSHV_LAB_GEN=Name);
// included inside kernels_mrg.cu's namespace shv::(anonymous).
//   MrgNull: one IADD per value (the fill's store-path ceiling).
struct MrgNull {
    uint32_t c;
};
__device__ __forceinline__ void make_gen(const Mrg& s, MrgNull& g) { g.c = s.x0 ^ s.y2; }
__device__ __forceinline__ uint32_t mrg_next(MrgNull& s, const MrgFpK&) { return s.c += 0x9E3779B9u; }
// Row-tile fill hooks (GenRows = SHV_LAB_GEN with -DSHV_MRG_ROWS_STEP=9): the
// lane start still runs (its cost stays in), its result only seeds the counter.
struct MrgNullRows {
    uint32_t x0, x1, x2, y0, y1, y2;
};
__device__ __forceinline__ void make_gen(const Mrg& s, MrgNullRows& g) { g = MrgNullRows{s.x0, s.x1, s.x2, s.y0, s.y1, s.y2}; }
__device__ __forceinline__ uint32_t mrg_next(MrgNullRows& s, const MrgFpK&) { return s.x0 += 0x9E3779B9u; }
__device__ __forceinline__ void set_state(MrgNullRows& g, const double r[6], const MrgFpK&)
{
    g.x0 = (uint32_t)__double2loint(r[0]) ^ (uint32_t)__double2loint(r[3]);
}
__device__ __forceinline__ void pin_state(MrgNullRows& g) { asm volatile("" : "+r"(g.x0)); }
__device__ __forceinline__ void pin_state(MrgNull& g) { asm volatile("" : "+r"(g.c)); }
