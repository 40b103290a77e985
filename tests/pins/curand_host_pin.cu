// curand_host_pin.cu — TEST-ONLY independent pin for the CPU oracle.
//
// Compiles NVIDIA cuRAND's own header implementations of MRG32k3a and
// Philox4x32-10 (curand_kernel.h, curand_philox4x32_x.h) as HOST code and
// answers queries on stdin, so tests/test_oracle_pins.py can check the oracle
// against a library implementation of the same generators that shares no code
// with it. Needs nvcc to build, no GPU to run. Not part of the product.
//
// Queries (one per line, decimal integers), answers one line each:
//   mrg s10 s11 s12 s20 s21 s22 n        -> n outputs z of curand_MRG32k3a
//   mrgskip s10..s22 seq subseq off      -> state after skipahead_sequence,
//                                           skipahead_subsequence, skipahead
//   philox c0 c1 c2 c3 k0 k1             -> curand_Philox4x32_10 block
//   pstream seed g offset n              -> n draws of curand() after
//                                           curand_init(seed, g, offset)
#define QUALIFIERS static inline __host__ __device__
#include <curand_kernel.h>
#include <cstdio>
#include <cstring>

int main() {
  char cmd[32];
  while (std::scanf("%31s", cmd) == 1) {
    if (!std::strcmp(cmd, "mrg")) {
      curandStateMRG32k3a_t st;
      unsigned long long n;
      std::scanf("%u %u %u %u %u %u %llu", &st.s1[0], &st.s1[1], &st.s1[2],
                 &st.s2[0], &st.s2[1], &st.s2[2], &n);
      for (unsigned long long i = 0; i < n; ++i)
        std::printf("%s%.0f", i ? " " : "", curand_MRG32k3a(&st));
      std::printf("\n");
    } else if (!std::strcmp(cmd, "mrgskip")) {
      curandStateMRG32k3a_t st;
      unsigned long long seq, sub, off;
      std::scanf("%u %u %u %u %u %u %llu %llu %llu", &st.s1[0], &st.s1[1], &st.s1[2],
                 &st.s2[0], &st.s2[1], &st.s2[2], &seq, &sub, &off);
      skipahead_sequence(seq, &st);
      skipahead_subsequence(sub, &st);
      skipahead(off, &st);
      std::printf("%u %u %u %u %u %u\n", st.s1[0], st.s1[1], st.s1[2], st.s2[0],
                  st.s2[1], st.s2[2]);
    } else if (!std::strcmp(cmd, "philox")) {
      uint4 c;
      uint2 k;
      std::scanf("%u %u %u %u %u %u", &c.x, &c.y, &c.z, &c.w, &k.x, &k.y);
      uint4 r = curand_Philox4x32_10(c, k);
      std::printf("%u %u %u %u\n", r.x, r.y, r.z, r.w);
    } else if (!std::strcmp(cmd, "pstream")) {
      unsigned long long seed, g, off, n;
      std::scanf("%llu %llu %llu %llu", &seed, &g, &off, &n);
      curandStatePhilox4_32_10_t st;
      curand_init(seed, g, off, &st);
      for (unsigned long long i = 0; i < n; ++i)
        std::printf("%s%u", i ? " " : "", curand(&st));
      std::printf("\n");
    } else {
      std::printf("error\n");
    }
    std::fflush(stdout);
  }
  return 0;
}
