// Dispatch of the N-level kernels to their per-N instantiation units.
#include "mbg_kernels.h"

#ifndef MBG_VARIANT
#error "compile with -DMBG_VARIANT=fast|exact"
#endif

namespace mbg {
namespace MBG_VARIANT {
namespace dense {
#define MBG_DECL(n)                                                                        \
    cudaError_t launch_split_##n(const void *params, long long tiles, cudaStream_t st);       \
    cudaError_t launch_rk4_##n(const void *params, long long tiles, cudaStream_t st);         \
    cudaError_t launch_batch_split_##n(const void *params, int systems, cudaStream_t st);     \
    cudaError_t launch_batch_rk4_##n(const void *params, int systems, cudaStream_t st);
MBG_DECL(2)
MBG_DECL(3)
MBG_DECL(4)
MBG_DECL(5)
MBG_DECL(6)
MBG_DECL(7)
MBG_DECL(8)
}  // namespace dense

cudaError_t launch_dense_split(int n, const void *params, long long tiles, cudaStream_t st) {
    switch (n) {
        case 3: return dense::launch_split_3(params, tiles, st);
        case 4: return dense::launch_split_4(params, tiles, st);
        case 5: return dense::launch_split_5(params, tiles, st);
        case 6: return dense::launch_split_6(params, tiles, st);
        case 7: return dense::launch_split_7(params, tiles, st);
        case 8: return dense::launch_split_8(params, tiles, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_dense_rk4(int n, const void *params, long long tiles, cudaStream_t st) {
    switch (n) {
        case 2: return dense::launch_rk4_2(params, tiles, st);
        case 3: return dense::launch_rk4_3(params, tiles, st);
        case 4: return dense::launch_rk4_4(params, tiles, st);
        case 5: return dense::launch_rk4_5(params, tiles, st);
        case 6: return dense::launch_rk4_6(params, tiles, st);
        case 7: return dense::launch_rk4_7(params, tiles, st);
        case 8: return dense::launch_rk4_8(params, tiles, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_batch_dense(int n, bool rk4, const void *params, int systems, cudaStream_t st) {
#define MBG_BATCH_CASE(k)                                                                  \
    case k:                                                                                \
        return rk4 ? dense::launch_batch_rk4_##k(params, systems, st)                      \
                   : dense::launch_batch_split_##k(params, systems, st);
    switch (n) {
        MBG_BATCH_CASE(2)
        MBG_BATCH_CASE(3)
        MBG_BATCH_CASE(4)
        MBG_BATCH_CASE(5)
        MBG_BATCH_CASE(6)
        MBG_BATCH_CASE(7)
        MBG_BATCH_CASE(8)
        default: return cudaErrorInvalidValue;
    }
#undef MBG_BATCH_CASE
}

}  // namespace MBG_VARIANT
}  // namespace mbg
