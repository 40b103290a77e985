// lab_gen.cuh — stand-in generators for the MRG fill kernels, compiled only
// into tools/lab builds (-DSHV_LAB_GEN_HEADER='"path"' -DSHV_LAB_GEN=Name);
// included inside kernels_mrg.cu's namespace shv::(anonymous).
//   MrgNull: one IADD per value (the fill's store-path ceiling).
struct MrgNull {
    uint32_t c;
};
__device__ __forceinline__ void make_gen(const Mrg& s, MrgNull& g) { g.c = s.x0 ^ s.y2; }
__device__ __forceinline__ uint32_t mrg_next(MrgNull& s, const MrgFpK&) { return s.c += 0x9E3779B9u; }
