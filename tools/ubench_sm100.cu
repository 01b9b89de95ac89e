// ubench_sm100.cu -- microbenchmarks behind K1's design choices (sm_100a):
// per-SM throughput of TMEM reads (tcgen05.ld 32x32b), MUFU ex2, warp
// shuffles, packed f32x2 FMA and 3-input max.  One CTA per SM, cycles from
// clock64 inside the CTA.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 \
//   -I paper_2410_23317_b200/csrc tools/ubench_sm100.cu -o /tmp/ubench -lcuda
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

constexpr int kIters = 4096;

__global__ void tmem_read(int nwarps_active, float* sink, long long* cyc) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) sm100::tmem_alloc(&slot, 512);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t base = slot + (uint32_t(32 * (warp & 3)) << 16);
    const uint32_t col0 = (warp >> 2) * 32;
    float acc = 0.f;
    __syncthreads();
    long long t0 = clock64();
    if (warp < nwarps_active) {
        for (int i = 0; i < kIters; ++i) {
            float v[32];
            sm100::tmem_ld32(base + ((col0 + (i & 7) * 64) & 511), v);
#pragma unroll
            for (int k = 0; k < 32; ++k) acc += v[k];
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (acc == 12345.f) sink[threadIdx.x] = acc;
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        sm100::tc_fence_after();
        sm100::tmem_dealloc(slot, 512);
    }
}

// 2 loads in flight before one wait
__global__ void tmem_read2(int nwarps_active, float* sink, long long* cyc) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) sm100::tmem_alloc(&slot, 512);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t base = slot + (uint32_t(32 * (warp & 3)) << 16);
    float acc = 0.f;
    __syncthreads();
    long long t0 = clock64();
    if (warp < nwarps_active) {
        for (int i = 0; i < kIters / 2; ++i) {
            uint32_t r[64];
            const uint32_t a0 = base + ((i * 64) & 511), a1 = base + ((i * 64 + 32) & 511);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
                "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                  "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                  "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                  "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                : "r"(a0));
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
                "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]),
                  "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]),
                  "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]),
                  "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]),
                  "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
                : "r"(a1));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 64; ++k) acc += __uint_as_float(r[k]);
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (acc == 12345.f) sink[threadIdx.x] = acc;
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        sm100::tc_fence_after();
        sm100::tmem_dealloc(slot, 512);
    }
}

__global__ void mufu(float* sink, long long* cyc) {
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = -0.001f * (threadIdx.x + k);
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[k]));
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.f) sink[threadIdx.x] = s;
}

__global__ void shfl(float* sink, long long* cyc) {
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __shfl_xor_sync(0xffffffffu, x[k], 1 + (k & 15));
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.f) sink[threadIdx.x] = s;
}

__global__ void ffma2(float* sink, long long* cyc) {
    float2 x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = make_float2(threadIdx.x * 1e-3f + k, k * 0.5f);
    const float2 a = make_float2(0.999f, 0.998f), b = make_float2(1e-3f, 2e-3f);
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            unsigned long long xv = *reinterpret_cast<unsigned long long*>(&x[k]);
            const unsigned long long av = *reinterpret_cast<const unsigned long long*>(&a);
            const unsigned long long bv = *reinterpret_cast<const unsigned long long*>(&b);
            asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(xv) : "l"(av), "l"(bv));
            x[k] = *reinterpret_cast<float2*>(&xv);
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k].x + x[k].y;
    if (s == 12345.f) sink[threadIdx.x] = s;
}

__global__ void ffma1(float* sink, long long* cyc) {
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32 %0, %0, 0f3F7FBE77, 0f3A83126F;" : "+f"(x[k]));
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.f) sink[threadIdx.x] = s;
}

__global__ void max3(float* sink, long long* cyc) {
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
    const float y = 0.5f, z = 0.25f;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(x[k]) : "f"(y + k), "f"(z));
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.f) sink[threadIdx.x] = s;
}

static double avg_cycles(long long* d, int n) {
    long long h[1024];
    cudaMemcpy(h, d, n * sizeof(long long), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < n; ++i) s += h[i];
    return s / n;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* sink;
    long long* cyc;
    cudaMalloc(&sink, 4096 * 4);
    cudaMalloc(&cyc, 1024 * 8);
    for (int w : {4, 8, 16}) {
        for (int rep = 0; rep < 2; ++rep) tmem_read<<<sms, 512>>>(w, sink, cyc);
        cudaDeviceSynchronize();
        double c = avg_cycles(cyc, sms);
        const double bytes = (double)w * 32 * 32 * 4 * kIters;   // per SM
        printf("tmem ld32 x1-in-flight warps=%2d: %.1f B/clk/SM (%.0f cycles)\n", w, bytes / c, c);
        for (int rep = 0; rep < 2; ++rep) tmem_read2<<<sms, 512>>>(w, sink, cyc);
        cudaDeviceSynchronize();
        c = avg_cycles(cyc, sms);
        printf("tmem ld32 x2-in-flight warps=%2d: %.1f B/clk/SM (%.0f cycles)\n", w, bytes / c, c);
    }
    for (int threads : {256, 512, 1024}) {
        for (int rep = 0; rep < 2; ++rep) mufu<<<sms, threads>>>(sink, cyc);
        cudaDeviceSynchronize();
        double c = avg_cycles(cyc, sms);
        printf("ex2 threads=%4d: %.2f ops/clk/SM\n", threads, (double)threads * 8 * kIters / c);
        for (int rep = 0; rep < 2; ++rep) shfl<<<sms, threads>>>(sink, cyc);
        cudaDeviceSynchronize();
        c = avg_cycles(cyc, sms);
        printf("shfl threads=%4d: %.2f lanes/clk/SM\n", threads, (double)threads * 8 * kIters / c);
        for (int rep = 0; rep < 2; ++rep) ffma1<<<sms, threads>>>(sink, cyc);
        cudaDeviceSynchronize();
        c = avg_cycles(cyc, sms);
        printf("ffma threads=%4d: %.2f lanes/clk/SM\n", threads, (double)threads * 8 * kIters / c);
        for (int rep = 0; rep < 2; ++rep) ffma2<<<sms, threads>>>(sink, cyc);
        cudaDeviceSynchronize();
        c = avg_cycles(cyc, sms);
        printf("ffma2 threads=%4d: %.2f fma/clk/SM (2 per lane-op)\n", threads, (double)threads * 16 * kIters / c);
        for (int rep = 0; rep < 2; ++rep) max3<<<sms, threads>>>(sink, cyc);
        cudaDeviceSynchronize();
        c = avg_cycles(cyc, sms);
        printf("max3 threads=%4d: %.2f lanes/clk/SM\n", threads, (double)threads * 8 * kIters / c);
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
