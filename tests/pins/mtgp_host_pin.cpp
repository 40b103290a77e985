// mtgp_host_pin.cpp — TEST-ONLY independent pin for the CPU oracle's MTGP32.
//
// Compiles NVIDIA cuRAND's own MTGP32 implementation (curand_mtgp32_host.h:
// mtgp32_init_state; curand_mtgp32_kernel.h: para_rec / temper / curand(),
// which the header makes host-callable with a one-thread "block") and its
// 200 MTGP32-11213 parameter sets (curand_mtgp32dc_p_11213.h, the authors'
// Dynamic Creator output) with the HOST compiler, so tests can check the
// oracle against a library implementation that shares no code with it.
// Not part of the product.
//
// Queries on stdin, one answer line each:
//   params p            -> pos sh1 sh2 mask tbl[16] tmp_tbl[16] of set p
//   gen p seed n        -> n outputs of curand() on state p after
//                          curandMakeMTGP32KernelState's init with u64 seed
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
#include <curand_mtgp32_host.h>
#include <curand_mtgp32dc_p_11213.h>
#include <curand_mtgp32_kernel.h>

const dim3 blockDim(1, 1, 1);   // one-thread block: curand() steps one word per call
const uint3 threadIdx = {0, 0, 0};

static mtgp32_kernel_params_t K;

int main()
{
    for (int i = 0; i < CURAND_NUM_MTGP32_PARAMS; ++i) {
        K.pos_tbl[i] = mtgp32dc_params_fast_11213[i].pos;
        K.sh1_tbl[i] = mtgp32dc_params_fast_11213[i].sh1;
        K.sh2_tbl[i] = mtgp32dc_params_fast_11213[i].sh2;
        for (int j = 0; j < 16; ++j) {
            K.param_tbl[i][j] = mtgp32dc_params_fast_11213[i].tbl[j];
            K.temper_tbl[i][j] = mtgp32dc_params_fast_11213[i].tmp_tbl[j];
        }
    }
    K.mask[0] = mtgp32dc_params_fast_11213[0].mask;
    char cmd[32];
    while (std::scanf("%31s", cmd) == 1) {
        if (!std::strcmp(cmd, "params")) {
            int p;
            std::scanf("%d", &p);
            const mtgp32_params_fast_t& q = mtgp32dc_params_fast_11213[p];
            std::printf("%d %d %d %u", q.pos, q.sh1, q.sh2, q.mask);
            for (int j = 0; j < 16; ++j) std::printf(" %u", q.tbl[j]);
            for (int j = 0; j < 16; ++j) std::printf(" %u", q.tmp_tbl[j]);
            std::printf("\n");
        } else if (!std::strcmp(cmd, "gen")) {
            int p;
            unsigned long long seed, n;
            std::scanf("%d %llu %llu", &p, &seed, &n);
            static curandStateMtgp32_t st;
            seed = seed ^ (seed >> 32);  // as curandMakeMTGP32KernelState
            mtgp32_init_state(&st.s[0], &mtgp32dc_params_fast_11213[p], (unsigned int)seed + p + 1);
            st.offset = 0;
            st.pIdx = p;
            st.k = &K;
            for (unsigned long long i = 0; i < n; ++i) std::printf("%s%u", i ? " " : "", curand(&st));
            std::printf("\n");
        } else {
            std::printf("error\n");
        }
        std::fflush(stdout);
    }
    return 0;
}
