// vlc_common.cuh -- device helpers shared by the sm_100a kernels of the
// VL-Cache compress + compressed-decode path.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#define VLC_DEV __device__ __forceinline__

namespace vlc {

constexpr unsigned kFull = 0xffffffffu;
constexpr float kLog2e = 1.4426950408889634f;

// exp2 on the MUFU pipe (ex2.approx.ftz: ~2 ulp, -inf -> +0).
// Programmatic dependent launch between the path's kernels: each is launched
// with launch_pdl, waits for its predecessor's completion (and memory) before
// touching any of its outputs, then lets its own successor pre-launch.
VLC_DEV void pdl_wait_then_release() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

VLC_DEV float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__host__ __device__ __forceinline__ int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }

VLC_DEV float bf16_lo(uint32_t packed) { return __uint_as_float(packed << 16); }
VLC_DEV float bf16_hi(uint32_t packed) { return __uint_as_float(packed & 0xffff0000u); }

// 32 values per lane in, lane c out holds the sum over the warp's 32 lanes of
// value index c.  Every column is reduced by the same tree (pairs of lanes
// grouped by lane bit 4, then 3, ... 0), and IEEE addition is commutative, so
// bit-identical columns produce bit-identical sums regardless of position --
// the property top-k tie-breaking needs (reference scoring.py:209-210).
template <typename T>
VLC_DEV T transpose_reduce32(T (&v)[32], int lane) {
#pragma unroll
    for (int width = 16; width >= 1; width >>= 1) {
        const bool upper = (lane & width) != 0;
#pragma unroll
        for (int k = 0; k < width; ++k) {
            T send = upper ? v[k] : v[k + width];
            T keep = upper ? v[k + width] : v[k];
            v[k] = keep + __shfl_xor_sync(kFull, send, width);
        }
    }
    return v[0];
}

template <typename T>
VLC_DEV T warp_sum(T x) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
    return x;
}

VLC_DEV float warp_max(float x) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) x = fmaxf(x, __shfl_xor_sync(kFull, x, o));
    return x;
}
VLC_DEV float warp_min(float x) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) x = fminf(x, __shfl_xor_sync(kFull, x, o));
    return x;
}

// Inclusive block scan (sum) of one value per thread; blockDim.x <= 1024,
// multiple of 32.  `scratch` holds >= 32 entries.
template <typename T>
VLC_DEV T block_inclusive_scan(T x, T* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) scratch[warp] = x;
    __syncthreads();
    if (warp == 0) {
        T s = lane < nwarps ? scratch[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(kFull, s, o);
            if (lane >= o) s += y;
        }
        scratch[lane] = s;
    }
    __syncthreads();
    T base = warp > 0 ? scratch[warp - 1] : T(0);
    __syncthreads();
    return x + base;
}

}  // namespace vlc
