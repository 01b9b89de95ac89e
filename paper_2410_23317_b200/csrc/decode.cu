// decode.cu -- K5: one decode step over the ragged compressed cache.
//
// reference: bench.py:356-372 (_decode_sequence: append the step's K/V row,
// then decode_step over the first k + s + 1 rows for the G query heads of each
// KV head) and _core.pyx:245-278 (decode_step: softmax(q K^T / sqrt(d)) V, fp32).
//
// One CTA per (b, l, kv) slot streams the slot's K and V rows through a
// kStages-deep shared-memory ring of 64-row chunks, loaded by 2-D TMA with the
// 128-byte swizzle so tensor-core fragments come out of shared memory
// conflict-free.  The G <= 8 query heads of the KV head form the M rows of
// mma.sync tiles (GQA: every key row is read from HBM once per step for the
// whole group):
//   S = Q K^T     m16n8k16, bf16 in, fp32 accumulate (exact products);
//   O += P V      m16n8k8, P split into bf16 hi + lo parts (~2^-16 relative),
//                 V exact bf16, fp32 accumulate.
// Each of the 8 warps owns 8 rows of every chunk with its own online-softmax
// state; the warps' (max, sum, O) partials merge once at the end.  The chunk
// holding row k + step takes it from k_new / v_new (patched into the swizzled
// tile) and also appends it to the cache for later steps.
#include "sm100.cuh"
#include "vlc_common.cuh"
#include "vlc_kernels.h"

namespace vlc {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kMaxG = 8;
constexpr int kChunk = 64;      // rows per ring stage (8 per warp)
#ifndef VLC_DEC_STAGES
#define VLC_DEC_STAGES 2
#endif
constexpr int kStages = VLC_DEC_STAGES;

template <int D>
struct Cfg {
    static constexpr int KB = D / 64;                        // 64-dim (128 B) swizzle boxes per row
    static constexpr uint32_t kBox = kChunk * 128;           // bytes of one box (64 rows x 128 B)
    static constexpr uint32_t kTile = KB * kBox;             // K (or V) tile of a chunk
    static constexpr uint32_t kStage = 2 * kTile;            // K + V
    static constexpr uint32_t kBytes = kStages * kStage + 1024;   // + alignment slack
    static constexpr int NT = D / 8;                         // 8-dim output tiles
};

// byte offset of 16-byte piece `c` (of the row's D/8) of row r inside a tile
template <int D>
VLC_DEV uint32_t swz(int r, int c) {
    return (uint32_t)((c >> 3) * Cfg<D>::kBox + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

VLC_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
VLC_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
// D = A(16x16, rows 8..15 zero) * B(16x8) + C, bf16 -> f32
VLC_DEV void mma_k16(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
// D = A(16x8, rows 8..15 zero) * B(8x8) + C
VLC_DEV void mma_k8(float (&d)[4], uint32_t a0, uint32_t b0) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(0u), "r"(b0));
}
VLC_DEV uint32_t pack_bf16(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
VLC_DEV float bf16_round(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

template <int D, int G>
__global__ void __launch_bounds__(kThreads, 2)
decode_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap, DecodeArgs a) {
    using C = Cfg<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar[kStages];
    __shared__ float part_m[kWarps][kMaxG], part_s[kWarps][kMaxG];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int row = lane >> 2, quad = lane & 3;              // fragment row (query head), column pair
    const int s = blockIdx.x;
    const int64_t n = a.base_len[s / a.Hkv] + a.step + 1;    // rows this step
    const int64_t new_row = n - 1;
    const int64_t seg = a.cache_off[s];
    const int nchunks = (int)((n + kChunk - 1) / kChunk);

    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) sm100::mbar_init(&bar[i], 1);
        sm100::fence_barrier_init();
        sm100::tma_prefetch(&kmap);
        sm100::tma_prefetch(&vmap);
    }
    __syncthreads();
    auto issue = [&](int c) {
        const int st = c % kStages;
        uint8_t* kdst = smem + st * C::kStage;
        const int y = (int)(seg + (int64_t)c * kChunk);
        sm100::mbar_expect_tx(&bar[st], C::kStage);
        for (int kb = 0; kb < C::KB; ++kb) {
            sm100::tma_load_2d(kdst + kb * C::kBox, &kmap, &bar[st], kb * 64, y);
            sm100::tma_load_2d(kdst + C::kTile + kb * C::kBox, &vmap, &bar[st], kb * 64, y);
        }
    };
    // Programmatic dependent launch: everything up to griddepcontrol.wait may
    // overlap the previous kernel.  When the caller guarantees that kernel is
    // this cache's decode step `step - 1` (a.chained), rows written before it
    // are final (that step waited for them), so only the chunk holding row
    // k + step - 1 (its append) must wait; the others stream in right away.
    // Without that guarantee (a.chained == 0) every load waits.
    const int pend = a.chained ? (int)((n - 2) / kChunk) : 0;
    if (tid == 0 && a.chained)
        for (int c = 0; c < kStages && c < nchunks; ++c)
            if (c != pend) issue(c);

    // Q as A fragments (rows = heads; rows >= G and 8..15 are zero), per 16-dim k-step
    const uint32_t* qw = reinterpret_cast<const uint32_t*>(a.q);
    uint32_t qa[D / 16][2];
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
        if (row < G) {
            const int64_t base = (((int64_t)s * G + row) * a.q_stride + kk * 16) / 2;
            qa[kk][0] = qw[base + quad];
            qa[kk][1] = qw[base + 4 + quad];
        } else {
            qa[kk][0] = qa[kk][1] = 0u;
        }
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (tid == 0) {
        if (a.chained) {
            if (pend < kStages && pend < nchunks) issue(pend);
        } else {
            for (int c = 0; c < kStages && c < nchunks; ++c) issue(c);
        }
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    float o[C::NT][4];
#pragma unroll
    for (int t = 0; t < C::NT; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
    float run_m = -INFINITY, run_s = 0.f;                    // head `row`, this thread's columns
    const float c1 = a.inv_scale * kLog2e;

    for (int c = 0; c < nchunks; ++c) {
        const int st = c % kStages;
        const int64_t j0 = (int64_t)c * kChunk;
        uint8_t* ks = smem + st * C::kStage;
        uint8_t* vs = ks + C::kTile;
        sm100::mbar_wait(&bar[st], (c / kStages) & 1);
        if (new_row < j0 + kChunk) {   // last chunk: patch in the new row (CTA-uniform)
            const int r = (int)(new_row - j0);
            if (tid < 2 * (D / 8)) {
                const bool isv = tid >= D / 8;
                const int piece = tid % (D / 8);
                const uint4 val = reinterpret_cast<const uint4*>(
                    static_cast<const __nv_bfloat16*>(isv ? a.v_new : a.k_new) + (int64_t)s * a.kv_stride)[piece];
                *reinterpret_cast<uint4*>((isv ? vs : ks) + swz<D>(r, piece)) = val;
                reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(isv ? a.v_cache : a.k_cache) +
                                         (seg + new_row) * D)[piece] = val;
            }
            __syncthreads();
        }
        // ---- S = Q K^T for this warp's 8 rows (keys) of the chunk
        const int kr = warp * 8;                               // first key of the warp
        float sacc[4] = {0.f, 0.f, 0.f, 0.f};
        const uint32_t kbase = sm100::smem_u32(ks);
#pragma unroll
        for (int kk = 0; kk < D / 16; kk += 2) {
            uint32_t b0, b1, b2, b3;
            ldsm_x4(kbase + swz<D>(kr + (lane & 7), kk * 2 + (lane >> 3)), b0, b1, b2, b3);
            mma_k16(sacc, qa[kk][0], qa[kk][1], b0, b1);
            mma_k16(sacc, qa[kk + 1][0], qa[kk + 1][1], b2, b3);
        }
        // ---- online softmax of head `row` over keys kr + 2*quad, +1
        const int64_t jk = j0 + kr + 2 * quad;
        const float l0 = jk < n ? sacc[0] : -INFINITY;
        const float l1 = jk + 1 < n ? sacc[1] : -INFINITY;
        float tm = fmaxf(l0, l1);
        tm = fmaxf(tm, __shfl_xor_sync(kFull, tm, 1));
        tm = fmaxf(tm, __shfl_xor_sync(kFull, tm, 2));
        const float mn = fmaxf(run_m, tm);
        const float mnb = mn == -INFINITY ? 0.f : mn * c1;    // rows of an empty tail chunk
        const float p0 = ex2(fmaf(l0, c1, -mnb));
        const float p1 = ex2(fmaf(l1, c1, -mnb));
        if (__any_sync(kFull, mn != run_m)) {
            const float sc = run_m == -INFINITY ? 0.f : ex2(fmaf(run_m, c1, -mnb));
#pragma unroll
            for (int t = 0; t < C::NT; ++t) { o[t][0] *= sc; o[t][1] *= sc; }
            run_s *= sc;
        }
        run_m = mn;
        run_s += p0 + p1;
        // P as the A operand of m16n8k8: hi + lo bf16 parts
        const float h0 = bf16_round(p0), h1 = bf16_round(p1);
        const uint32_t phi = pack_bf16(h0, h1);
        const uint32_t plo = pack_bf16(p0 - h0, p1 - h1);
        // ---- O += P V over the warp's 8 keys, 8-dim output tiles
        const uint32_t vbase = sm100::smem_u32(vs);
#pragma unroll
        for (int t = 0; t < C::NT; t += 4) {
            uint32_t v0, v1, v2, v3;
            ldsm_x4_t(vbase + swz<D>(kr + (lane & 7), t + (lane >> 3)), v0, v1, v2, v3);
            mma_k8(o[t], phi, v0);     mma_k8(o[t], plo, v0);
            mma_k8(o[t + 1], phi, v1); mma_k8(o[t + 1], plo, v1);
            mma_k8(o[t + 2], phi, v2); mma_k8(o[t + 2], plo, v2);
            mma_k8(o[t + 3], phi, v3); mma_k8(o[t + 3], plo, v3);
        }
        __syncthreads();                                       // stage consumed by every warp
        if (tid == 0 && c + kStages < nchunks) issue(c + kStages);
    }

    // ---- merge the 8 warps: per head, (max, sum) then O, through shared memory
    run_s += __shfl_xor_sync(kFull, run_s, 1);
    run_s += __shfl_xor_sync(kFull, run_s, 2);
    if (quad == 0 && row < G) { part_m[warp][row] = run_m; part_s[warp][row] = run_s; }
    float* po = reinterpret_cast<float*>(smem);               // [kWarps][G][D], ring is idle now
    if (row < G) {
#pragma unroll
        for (int t = 0; t < C::NT; ++t)
            *reinterpret_cast<float2*>(po + (warp * G + row) * D + t * 8 + 2 * quad) = make_float2(o[t][0], o[t][1]);
    }
    __syncthreads();
    for (int idx = tid; idx < G * D; idx += kThreads) {
        const int g = idx / D, dim = idx % D;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) M = fmaxf(M, part_m[w][g]);
        float S = 0.f, O = 0.f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            if (part_m[w][g] == -INFINITY) continue;
            const float f = ex2((part_m[w][g] - M) * c1);
            S = fmaf(part_s[w][g], f, S);
            O = fmaf(po[(w * G + g) * D + dim], f, O);
        }
        a.out[((int64_t)s * G + g) * D + dim] = O / S;
    }
}

template <int D, int G>
cudaError_t launch_dg(const DecodeArgs& a, const CUtensorMap& km, const CUtensorMap& vm, cudaStream_t st) {
    using C = Cfg<D>;
    cudaError_t e = cudaFuncSetAttribute(decode_kernel<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::kBytes);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(a.slots);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL (see kernel)
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, decode_kernel<D, G>, km, vm, a);
}

template <int D>
cudaError_t launch_d(const DecodeArgs& a, cudaStream_t st) {
    CUtensorMap km, vm;
    if (!make_tmap_2d(&km, a.k_cache, a.cache_rows, D, kChunk) ||
        !make_tmap_2d(&vm, a.v_cache, a.cache_rows, D, kChunk))
        return cudaErrorInvalidValue;
    switch (a.G) {
        case 1: return launch_dg<D, 1>(a, km, vm, st);
        case 2: return launch_dg<D, 2>(a, km, vm, st);
        case 3: return launch_dg<D, 3>(a, km, vm, st);
        case 4: return launch_dg<D, 4>(a, km, vm, st);
        case 5: return launch_dg<D, 5>(a, km, vm, st);
        case 6: return launch_dg<D, 6>(a, km, vm, st);
        case 7: return launch_dg<D, 7>(a, km, vm, st);
        case 8: return launch_dg<D, 8>(a, km, vm, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

cudaError_t launch_decode(const DecodeArgs& a, cudaStream_t st) {
    if (a.G < 1 || a.G > kMaxG) return cudaErrorInvalidValue;
    if (a.d == 64) return launch_d<64>(a, st);
    if (a.d == 128) return launch_d<128>(a, st);
    return cudaErrorInvalidValue;
}

}  // namespace vlc
