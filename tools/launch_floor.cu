// Back-to-back launch floor on this GPU: 99 launches of a near-empty kernel
// captured in one CUDA graph, per-launch time for grid/smem/PDL variants
// matching K5's launch shape (256 CTAs x 256 threads, 99 KB dynamic smem).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/launch_floor tools/launch_floor.cu
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return -1.f; } } while (0)

__global__ void k_plain(float* out) {
    __shared__ float sm[1];
    if (threadIdx.x == 0) sm[0] = out[blockIdx.x];
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = sm[0] + 1.f;
}
__global__ void k_pdl(float* out) {
    __shared__ float sm[1];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) sm[0] = out[blockIdx.x];
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = sm[0] + 1.f;
}

static float run(bool pdl, int grid, int smem, float* buf) {
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    void (*fn)(float*) = pdl ? k_pdl : k_plain;
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < 99; ++i) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 1 : 0;
        CK(cudaLaunchKernelEx(&cfg, fn, buf));
    }
    CK(cudaStreamEndCapture(st, &g));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("capture: %s\n", cudaGetErrorString(e)); return -1.f; }
    cudaGraphExec_t ge;
    e = cudaGraphInstantiate(&ge, g, 0);
    if (e != cudaSuccess) { printf("instantiate: %s\n", cudaGetErrorString(e)); return -1.f; }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9;
    for (int rep = 0; rep < 10; ++rep) {
        CK(cudaEventRecord(a, st));
        CK(cudaGraphLaunch(ge, st));
        CK(cudaEventRecord(b, st));
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep >= 2 && ms < best) best = ms;
    }
    return best * 1000.f / 99.f;
}

int main() {
    float* buf;
    cudaMalloc(&buf, 4096 * sizeof(float));
    cudaMemset(buf, 0, 4096 * sizeof(float));
    for (int pdl = 0; pdl < 2; ++pdl)
        for (int grid : {148, 256, 296})
            for (int smem : {0, 101376})
                { printf("pdl=%d grid=%d smem=%6d: %.2f us per launch\n", pdl, grid, smem, run(pdl, grid, smem, buf)); fflush(stdout); }
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
