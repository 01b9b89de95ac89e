// budget.cu -- K2: layer-adaptive budget allocation on the device, numpy-exact.
//
// reference: sparsity.py:79 (gamma = below.sum() / causal.sum()),
//            sparsity.py:41-43 (gamma' = gamma.mean(axis=1)),
//            budget.py:107-110 (Z = sum(1 - gamma'); pre = (1 - gamma') / Z * (alpha*L)),
//            budget.py:75 (beta = clip(pre, beta_min, beta_max)),
//            budget.py:70-71 (k = clip(ceil(beta*m), 1, m)).
// numpy reduces contiguous float64 rows with pairwise summation
// (8 strided accumulators for n <= 128, recursive halving above); the same
// association is reproduced here with round-to-nearest intrinsics so that no
// FMA contraction can creep in.  Bit-exact given equal integer counts.
#include "vlc_common.cuh"
#include "vlc_kernels.h"

namespace vlc {
namespace {

__device__ double pairwise_sum(const double* a, int64_t n, int64_t stride) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, a[i * stride]);
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j * stride];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[(i + j) * stride]);
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; ++i) res = __dadd_rn(res, a[i * stride]);
        return res;
    }
    // numpy halves, rounding the split down to a multiple of the unroll (8)
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    const double left = pairwise_sum(a, n2, stride);
    return __dadd_rn(left, pairwise_sum(a + n2 * stride, n - n2, stride));
}

// One block.  Phase 1: a thread per (b, l, h) divides the counts; phase 2: a
// thread per (b, l) takes the numpy-order head mean; phase 3: a thread per b
// forms Z and the budgets; phase 4: block scan of per-slot sizes -> offsets.
constexpr int kAllocThreads = 1024;

// The intermediates are staged in dynamic shared memory when they fit
// (SMEM == true: gamma [B*L*Hq], one minus gamma' [B*L], kept counts [B*L]),
// so the phases' read-backs are shared-memory loads, not global round trips;
// the global outputs are written alongside.
template <bool SMEM>
__global__ void __launch_bounds__(kAllocThreads) allocate_kernel(BudgetArgs a) {
    pdl_wait_then_release();
    extern __shared__ double dyn[];
    __shared__ long long scan_k[32], scan_c[32];
    const int64_t BL = (int64_t)a.B * a.L;
    double* gam = SMEM ? dyn : a.gamma;
    double* omg = SMEM ? dyn + (a.below_head ? BL * a.Hq : 0) : a.beta_pre;           // 1 - gamma'
    int64_t* kc_s = SMEM ? reinterpret_cast<int64_t*>(omg + BL) : a.kept_counts;
    if (a.below_head) {
        const double causal = (double)a.causal_per_head;
        for (int64_t idx = threadIdx.x; idx < BL * a.Hq; idx += blockDim.x) {
            const double g = __ddiv_rn((double)a.below_head[idx], causal);
            if (SMEM) a.gamma[idx] = g;
            gam[idx] = g;
        }
        __syncthreads();
        for (int64_t bl = threadIdx.x; bl < BL; bl += blockDim.x) {
            const double gm = __ddiv_rn(pairwise_sum(gam + bl * a.Hq, a.Hq, 1), (double)a.Hq);
            a.gamma_mean[bl] = gm;
            omg[bl] = __dadd_rn(1.0, -gm);
        }
    } else {
        for (int64_t bl = threadIdx.x; bl < BL; bl += blockDim.x) {
            const double gm = a.gamma_mean_in[bl];
            a.gamma_mean[bl] = gm;
            omg[bl] = __dadd_rn(1.0, -gm);
        }
    }
    __syncthreads();
    __shared__ double z_s[1024];
    for (int b = threadIdx.x; b < a.B; b += blockDim.x) {
        const double z = pairwise_sum(omg + (int64_t)b * a.L, a.L, 1);
        z_s[b] = z;
        a.status[b] = (z == 0.0) ? 1 : 0;
    }
    __syncthreads();
    for (int64_t bl = threadIdx.x; bl < BL; bl += blockDim.x) {
        const double z = z_s[bl / a.L];
        const double p = __dmul_rn(__ddiv_rn(omg[bl], z), a.alpha_times_L);
        const double be = fmin(fmax(p, a.beta_min), a.beta_max);
        a.beta[bl] = be;
        const double kc = ceil(__dmul_rn(be, (double)a.prompt_len));
        int64_t k = (z == 0.0) ? 1 : (int64_t)kc;
        if (k < 1) k = 1;
        if (k > a.prompt_len) k = a.prompt_len;
        a.kept_counts[bl] = k;
        if (SMEM) kc_s[bl] = k;
        if (SMEM) a.beta_pre[bl] = p;   // (global path: rewritten after the barrier below)
    }
    __syncthreads();
    if (!SMEM)
        for (int64_t bl = threadIdx.x; bl < BL; bl += blockDim.x) {
            const double z = z_s[bl / a.L];
            a.beta_pre[bl] = __dmul_rn(__ddiv_rn(a.beta_pre[bl], z), a.alpha_times_L);
        }
    // offsets: chunked exclusive scan over slots (slot s uses kept_counts[s / Hkv])
    const int64_t slots = BL * a.Hkv;
    const int64_t chunk = (slots + blockDim.x - 1) / blockDim.x;
    const int64_t c0 = imin(slots, (int64_t)threadIdx.x * chunk), c1 = imin(slots, c0 + chunk);
    long long sk = 0, sc = 0;
    for (int64_t sl = c0; sl < c1; ++sl) {
        const int64_t k = kc_s[sl / a.Hkv];
        sk += k;
        sc += k + a.cache_extra;
    }
    const long long ik = block_inclusive_scan<long long>(sk, scan_k);
    const long long ic = block_inclusive_scan<long long>(sc, scan_c);
    long long ok = ik - sk, oc = ic - sc;
    for (int64_t sl = c0; sl < c1; ++sl) {
        const int64_t k = kc_s[sl / a.Hkv];
        a.kept_off[sl] = ok;
        a.cache_off[sl] = oc;
        ok += k;
        oc += k + a.cache_extra;
    }
    if (threadIdx.x == blockDim.x - 1) {
        a.kept_off[slots] = ik;
        a.cache_off[slots] = ic;
    }
}

}  // namespace

cudaError_t launch_allocate(const BudgetArgs& a, cudaStream_t st) {
    if (a.B > 1024) return cudaErrorInvalidValue;
    const int64_t BL = (int64_t)a.B * a.L;
    const int64_t bytes = 8 * ((a.below_head ? BL * a.Hq : 0) + 2 * BL);
    if (bytes <= 160 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(allocate_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)bytes);
        if (e != cudaSuccess) return e;
        return launch_pdl(allocate_kernel<true>, dim3(1), dim3(kAllocThreads), (size_t)bytes, st, a);
    }
    return launch_pdl(allocate_kernel<false>, dim3(1), dim3(kAllocThreads), 0, st, a);
}

}  // namespace vlc
