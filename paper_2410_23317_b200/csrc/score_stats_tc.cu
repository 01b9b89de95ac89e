// score_stats_tc.cu -- K1 on the 5th-generation tensor cores (sm_100a).
//
// reference: pkg/src/vlcache/_kernels/_core.pyx:110-242 (two-pass tiled
// statistics) for all G query heads of a KV head at once.
//
// CTA = (slot, block of 128 window rows).  Warp roles (384 threads):
//   warp 0      TMA producer: the Q block once, then every 128-key tile of the
//               slot twice (pass 1, pass 2) into a 3-stage swizzled ring
//   warp 1      MMA issuer: S = Q K^T, M=128 x N=128, K = head_dim, bf16 in,
//               fp32 accumulate in TMEM (two accumulator stages, 256 columns)
//   warp 2      TMEM allocator
//   warps 4-11  epilogue: thread = (window row, half of the tile's columns);
//               tcgen05.ld 32 columns at a time -> score_epilogue.cuh.
// The score matrix never leaves the SM: TMEM -> registers -> column sums.
#include <cuda.h>

#include <mutex>

#include "score_epilogue.cuh"
#include "sm100.cuh"
#include "vlc_kernels.h"

namespace vlc {
namespace {

constexpr int kM = 128;          // window rows per CTA (UMMA M)
constexpr int kN = 128;          // keys per tile (UMMA N)
constexpr int kStages = 3;       // K tile ring
constexpr int kEpiWarps = 8;
constexpr int kThreads = 128 + kEpiWarps * 32;
constexpr uint32_t kTmemCols = 2 * kN;

template <int D>
struct Layout {
    static constexpr int KB = D / 64;                       // 64-element (128 B) k-blocks
    static constexpr uint32_t kQRegion = kM * 128;          // bytes per Q k-block
    static constexpr uint32_t kKRegion = kN * 128;          // bytes per K k-block
    static constexpr uint32_t kQBytes = KB * kQRegion;
    static constexpr uint32_t kKBytes = KB * kKRegion;      // one stage
    static constexpr uint32_t kBarOff = kQBytes + kStages * kKBytes;
    static constexpr uint32_t kColOff = kBarOff + 256;      // 2 x 4 x 128 floats
    static constexpr uint32_t kRowOff = kColOff + 2 * 4 * kN * 4;   // 2 x 128 x (m, s)
    static constexpr uint32_t kBytes = kRowOff + 2 * kM * 8 + 1024; // + alignment slack
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
score_stats_tc(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
               ScoreArgs a, int nrb) {
    using LY = Layout<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + LY::kBarOff);
    uint64_t* full = bars;                    // [kStages]
    uint64_t* empty = bars + kStages;         // [kStages]
    uint64_t* qfull = bars + 2 * kStages;     // [1]
    uint64_t* tfull = qfull + 1;              // [2]
    uint64_t* tempty = tfull + 2;             // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    float* colbuf = reinterpret_cast<float*>(smem + LY::kColOff);   // [2][4][kN]
    float2* rowstat = reinterpret_cast<float2*>(smem + LY::kRowOff); // [2][kM]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.y, rb = blockIdx.x;
    const int64_t R = (int64_t)a.G * a.w;
    const int64_t r_first = (int64_t)rb * kM;
    const int64_t r_last = imin(R, r_first + kM) - 1;
    const int64_t i_max = (r_last / a.w == r_first / a.w) ? r_last % a.w : a.w - 1;
    const int64_t blk_end = imin(a.n, a.q_base + i_max + 1);   // keys any row here can see
    const int T = (int)((blk_end + kN - 1) / kN);
    const int iters = 2 * T;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) { sm100::mbar_init(full + i, 1); sm100::mbar_init(empty + i, 1); }
        sm100::mbar_init(qfull, 1);
        for (int i = 0; i < 2; ++i) { sm100::mbar_init(tfull + i, 1); sm100::mbar_init(tempty + i, kEpiWarps); }
        sm100::fence_barrier_init();
        sm100::fence_proxy_async();
    }
    if (warp == 2) sm100::tmem_alloc(tmem_slot, kTmemCols);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ------------------------------------------------ TMA producer
        sm100::tma_prefetch(&qmap);
        sm100::tma_prefetch(&kmap);
        sm100::mbar_expect_tx(qfull, LY::kQBytes);
        for (int kb = 0; kb < LY::KB; ++kb)
            sm100::tma_load_2d(smem + kb * LY::kQRegion, &qmap, qfull, kb * 64, (int)(s * R + r_first));
        for (int it = 0; it < iters; ++it) {
            const int st = it % kStages;
            const uint32_t ph = (it / kStages) & 1;
            const int t = it < T ? it : it - T;
            sm100::mbar_wait(empty + st, ph ^ 1);
            sm100::mbar_expect_tx(full + st, LY::kKBytes);
            uint8_t* kdst = smem + LY::kQBytes + st * LY::kKBytes;
            for (int kb = 0; kb < LY::KB; ++kb)
                sm100::tma_load_2d(kdst + kb * LY::kKRegion, &kmap, full + st, kb * 64,
                                   (int)(s * a.T + (int64_t)t * kN));
        }
    } else if (warp == 1 && lane == 0) {
        // ------------------------------------------------ MMA issuer
        constexpr uint32_t idesc = sm100::idesc_bf16_f32(kM, kN);
        const uint32_t q_base_addr = sm100::smem_u32(smem);
        sm100::mbar_wait(qfull, 0);
        for (int it = 0; it < iters; ++it) {
            const int st = it % kStages;
            const uint32_t ph = (it / kStages) & 1;
            const int acc = it & 1;
            const uint32_t aph = (it >> 1) & 1;
            sm100::mbar_wait(tempty + acc, aph ^ 1);
            sm100::mbar_wait(full + st, ph);
            sm100::tc_fence_after();
            const uint32_t k_addr = sm100::smem_u32(smem + LY::kQBytes + st * LY::kKBytes);
#pragma unroll
            for (int kb = 0; kb < LY::KB; ++kb) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {   // 4 x 16 elements = one 128 B swizzle row
                    const uint64_t ad = sm100::sdesc_k_sw128(q_base_addr + kb * LY::kQRegion + kk * 32);
                    const uint64_t bd = sm100::sdesc_k_sw128(k_addr + kb * LY::kKRegion + kk * 32);
                    sm100::mma_bf16(tmem + acc * kN, ad, bd, idesc, (kb | kk) != 0);
                }
            }
            sm100::mma_commit(empty + st);   // K stage reusable once these MMAs retire
            sm100::mma_commit(tfull + acc);  // accumulator ready for the epilogue
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue
        const int ew = warp - 4, sub = warp & 3, half = ew >> 2;
        const int row_local = 32 * sub + lane;
        const int64_t r = r_first + row_local;
        const bool row_ok = r < R;
        const int64_t i = row_ok ? r % a.w : 0;
        const int64_t row_end = row_ok ? imin(a.n, a.q_base + i + 1) : 0;
        const uint32_t lane_addr = tmem + (uint32_t(32 * sub) << 16);
        float l[32];

        RowStats st{-INFINITY, 0.f};
        for (int it = 0; it < T; ++it) {
            const int acc = it & 1;
            sm100::mbar_wait(tfull + acc, (it >> 1) & 1);
            sm100::tc_fence_after();
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int col0 = half * 64 + c * 32;
                sm100::tmem_ld32(lane_addr + acc * kN + col0, l);
#pragma unroll
                for (int k = 0; k < 32; ++k) l[k] *= a.inv_scale;
                const int valid = (int)imax(0, imin(32, row_end - ((int64_t)it * kN + col0)));
                pass1_chunk(l, valid, st);
            }
            sm100::tc_fence_before();
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(tempty + acc);
        }
        // merge the two column halves of each row (same formula on both sides)
        rowstat[half * kM + row_local] = make_float2(st.m, st.s);
        sm100::named_bar_sync(1, kEpiWarps * 32);
        {
            const float2 h0 = rowstat[row_local], h1 = rowstat[kM + row_local];
            const float m = fmaxf(h0.x, h1.x);
            float sum = 0.f;
            if (h0.x != -INFINITY) sum += h0.y * ex2((h0.x - m) * kLog2e);
            if (h1.x != -INFINITY) sum += h1.y * ex2((h1.x - m) * kLog2e);
            st.m = m;
            st.s = sum;
        }
        const float log2s = row_ok ? __log2f(st.s) : 0.f;

        int below = 0;
        float* colp = a.col_partial + ((int64_t)s * nrb + rb) * a.n;
        for (int it = T; it < iters; ++it) {
            const int acc = it & 1;
            const int t = it - T;
            const int p = t & 1;
            sm100::mbar_wait(tfull + acc, (it >> 1) & 1);
            sm100::tc_fence_after();
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int col0 = half * 64 + c * 32;
                sm100::tmem_ld32(lane_addr + acc * kN + col0, l);
#pragma unroll
                for (int k = 0; k < 32; ++k) l[k] *= a.inv_scale;
                const int64_t j0 = (int64_t)t * kN + col0;
                const int valid = (int)imax(0, imin(32, row_end - j0));
                float e[32];
                below += pass2_chunk(l, valid, st.m, log2s, a.t_star, e);
                colbuf[(p * 4 + sub) * kN + col0 + lane] = transpose_reduce32(e, lane);
                if (a.below_col) {
                    int bc[32];
#pragma unroll
                    for (int k = 0; k < 32; ++k) bc[k] = (k < valid && (l[k] - st.m) < a.t_star) ? 1 : 0;
                    const int cnt = transpose_reduce32(bc, lane);
                    if (cnt && j0 + lane < a.n) atomicAdd(a.below_col + (int64_t)s * a.n + j0 + lane, cnt);
                }
            }
            sm100::tc_fence_before();
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(tempty + acc);
            sm100::named_bar_sync(1, kEpiWarps * 32);
            if (ew < 4) {
                const int col = ew * 32 + lane;
                const int64_t j = (int64_t)t * kN + col;
                if (j < a.n) {
                    const float* cb = colbuf + p * 4 * kN + col;
                    colp[j] = ((cb[0] + cb[kN]) + (cb[2 * kN] + cb[3 * kN]));
                }
            }
        }
        // columns no row of this block can see
        for (int64_t j = (int64_t)T * kN + (ew * 32 + lane); j < a.n; j += kEpiWarps * 32) colp[j] = 0.f;
        if (row_ok) {
            if (half == 0) {
                a.row_max[(int64_t)s * R + r] = st.m;
                a.row_sum[(int64_t)s * R + r] = st.s;
            }
            if (below)
                atomicAdd(a.below_head + (int64_t)s * a.G + r / a.w, (unsigned long long)below);
        }
    }
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        sm100::tc_fence_after();
        sm100::tmem_dealloc(tmem, kTmemCols);
    }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// 2-D bf16 map over [rows, d]: box = 64 elements (128 B, swizzled) x box_rows
bool make_map(CUtensorMap* map, const void* base, int64_t rows, int d, int box_rows) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    cuuint64_t gdim[2] = {(cuuint64_t)d, (cuuint64_t)rows};
    cuuint64_t gstride[1] = {(cuuint64_t)d * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t estride[2] = {1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstride, box, estride,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D>
cudaError_t launch_tc(const ScoreArgs& a, int nrb, cudaStream_t st) {
    CUtensorMap qmap, kmap;
    const int64_t R = (int64_t)a.G * a.w;
    if (!make_map(&qmap, a.q, (int64_t)a.slots * R, a.d, kM)) return cudaErrorInvalidValue;
    if (!make_map(&kmap, a.k, (int64_t)a.slots * a.T, a.d, kN)) return cudaErrorInvalidValue;
    const size_t sm = Layout<D>::kBytes;
    cudaError_t e = cudaFuncSetAttribute(score_stats_tc<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    dim3 grid(nrb, a.slots);
    score_stats_tc<D><<<grid, kThreads, sm, st>>>(qmap, kmap, a, nrb);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_score_stats_tc(const ScoreArgs& a, int nrb, cudaStream_t st) {
    if (a.d == 64) return launch_tc<64>(a, nrb, st);
    if (a.d == 128) return launch_tc<128>(a, nrb, st);
    return cudaErrorInvalidValue;
}

}  // namespace vlc
