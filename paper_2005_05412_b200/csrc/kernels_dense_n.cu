// Instantiation unit of the N-level kernels for N = MBG_LEVELS (one file per
// N so the heavily unrolled templates compile in parallel).
#include "kernels_dense.cuh"

#ifndef MBG_LEVELS
#error "compile with -DMBG_LEVELS=N"
#endif

namespace mbg {
namespace MBG_VARIANT {
namespace dense {

template <int N, bool RK4, class Q, int MINB>
static cudaError_t launch_variant(const DenseParams<N, Q> &P, long long tiles, int dev, cudaStream_t st) {
    constexpr size_t smem = Layout<N, RK4>::smem_bytes();
    static bool configured[64] = {};
    if (!configured[dev]) {
        cudaError_t err = cudaFuncSetAttribute(dense_step_kernel<N, RK4, Q, MINB>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (err != cudaSuccess) return err;
        configured[dev] = true;
    }
    dense_step_kernel<N, RK4, Q, MINB><<<(unsigned)tiles, Layout<N, RK4>::TW, smem, st>>>(P);
    return cudaGetLastError();
}

template <int N, bool RK4, class Q>
static cudaError_t launch_n(const void *params, long long tiles, cudaStream_t st) {
    static_assert(sizeof(DenseParams<N, Q>) <= 32764, "kernel parameter block over the 32 KB launch limit");
    const auto &P = *static_cast<const DenseParams<N, Q> *>(params);
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    constexpr int kSmall = dense_min_blocks(N, RK4), kLarge = dense_min_blocks_large(N, RK4);
    if constexpr (kSmall != kLarge) {
        // the occupancy variant once the grid gives every CTA slot two tiles
        static int sms[64] = {};
        if (!sms[dev] && cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            sms[dev] = 148;
        if (tiles >= 2LL * kLarge * sms[dev]) return launch_variant<N, RK4, Q, kLarge>(P, tiles, dev, st);
    }
    return launch_variant<N, RK4, Q, kSmall>(P, tiles, dev, st);
}

template <int N, bool RK4, class Q>
static cudaError_t batch_n(const void *params, int systems, cudaStream_t st) {
    const auto &P = *static_cast<const BatchParams<N, Q> *>(params);
    static_assert(sizeof(BatchParams<N, Q>) <= 32764, "kernel parameter block over the 32 KB launch limit");
    constexpr size_t smem = Layout<N, RK4>::smem_bytes();
    constexpr int W = Layout<N, RK4>::TW;
#if defined(MBG_EXACT) && MBG_EXACT
    constexpr bool kRa = false;
#else
    constexpr bool kRa = true;  // as the step kernel chooses
#endif
    static bool configured[64][2] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    const bool ra = kRa && P.real_a;
    if (!configured[dev][ra]) {
        cudaError_t err = ra ? cudaFuncSetAttribute(dense_batch_kernel<N, RK4, Q, kRa>,
                                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                             : cudaFuncSetAttribute(dense_batch_kernel<N, RK4, Q, false>,
                                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (err != cudaSuccess) return err;
        configured[dev][ra] = true;
    }
    const unsigned blocks = (unsigned)((systems + W - 1) / W);
    if (ra)
        dense_batch_kernel<N, RK4, Q, kRa><<<blocks, W, smem, st>>>(P);
    else
        dense_batch_kernel<N, RK4, Q, false><<<blocks, W, smem, st>>>(P);
    return cudaGetLastError();
}

#define MBG_CAT2(a, b) a##b
#define MBG_CAT(a, b) MBG_CAT2(a, b)

cudaError_t MBG_CAT(launch_split_, MBG_LEVELS)(const void *params, long long tiles, cudaStream_t st) {
#if MBG_LEVELS >= 3
    return launch_n<MBG_LEVELS, false, DenseQm<MBG_LEVELS>>(params, tiles, st);
#else
    return cudaErrorInvalidValue;
#endif
}

cudaError_t MBG_CAT(launch_rk4_, MBG_LEVELS)(const void *params, long long tiles, cudaStream_t st) {
    return launch_n<MBG_LEVELS, true, Rk4Qm<MBG_LEVELS>>(params, tiles, st);
}

cudaError_t MBG_CAT(launch_batch_split_, MBG_LEVELS)(const void *params, int systems, cudaStream_t st) {
#if MBG_LEVELS >= 3
    return batch_n<MBG_LEVELS, false, DenseQm<MBG_LEVELS>>(params, systems, st);
#else
    return cudaErrorInvalidValue;
#endif
}

cudaError_t MBG_CAT(launch_batch_rk4_, MBG_LEVELS)(const void *params, int systems, cudaStream_t st) {
    return batch_n<MBG_LEVELS, true, Rk4Qm<MBG_LEVELS>>(params, systems, st);
}

}  // namespace dense
}  // namespace MBG_VARIANT
}  // namespace mbg
