// select.cu -- K3: per-(b, l, kv) eviction = recent reserve + top-k by score.
//
// reference: scoring.py:185-201 (score = sum over the query-head group / G),
//            scoring.py:213-235 (reserve = min(ceil(frac*k), k); recent
//            positions [m-reserve, m) kept unconditionally; the rest by
//            top_k_indices over scores[:m-reserve]),
//            scoring.py:204-210 (lexsort: descending score, ties toward the
//            larger index; output ascending).
// One CTA per slot.  Each float64 score maps to an order-preserving uint64
// key (sign-flip trick; -0.0 folded onto +0.0 so equal values tie as numpy
// sees them); an MSB-first 8-bit radix select finds the exact k-th key T;
// a bucket whose keys are all equal (a run of ties, common with planted
// duplicate keys) ends the passes at once; ties at T are resolved toward larger
// indices by a right-to-left rank; warp ballots + a prefix over the per-warp
// counts (register path) or a block scan compact the kept flags in index order.
#include "vlc_common.cuh"
#include "vlc_kernels.h"

namespace vlc {
namespace {

constexpr int kThreads = 512;
constexpr int64_t kSmemKeysMax = 24 * 1024;   // scores kept in shared memory up to this many

__device__ __forceinline__ unsigned long long order_key(double x) {
    if (x == 0.0) x = 0.0;  // -0.0 == +0.0
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// RK > 0: n <= RK * kThreads, each thread keeps its RK keys (j = tid + u *
// kThreads) in registers for the radix passes and issues all their partial
// loads at once; RK == 0: any n, keys re-read from shared / global memory.
template <int RK>
__global__ void __launch_bounds__(kThreads, 2) select_kernel(SelectArgs a) {
    // scores_ready (vlc_select_after_allocate): col_partial was final before the
    // preceding K2 released this grid, so phase 1 runs under K2 and only the
    // budgets wait; its loads bypass L1 (ld.global.cg) since this grid has not
    // passed a dependency wait yet
    const bool early = a.scores_ready && !a.scores_in;
    if (!early) pdl_wait_then_release();
    extern __shared__ unsigned long long keys_smem[];
    __shared__ unsigned int hist[256];
    __shared__ long long scan_scratch[32];
    __shared__ unsigned long long s_prefix, s_mask;
    __shared__ long long s_want;
    __shared__ unsigned long long s_min, s_max;
    __shared__ unsigned long long s_bmin, s_bmax;   // current bucket's extremes
    __shared__ int s_small;                        // bucket small enough for the warp finish
    __shared__ unsigned long long s_cand[32];      // its keys
    __shared__ int s_ncand;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int s = blockIdx.x;
    const int64_t n = a.n;
    unsigned long long* keys = (n <= kSmemKeysMax) ? keys_smem : a.key_scratch + (int64_t)s * n;

    // 1. score = (sum over row blocks, fixed order, fp64) / G  (scoring.py:198-201),
    //    or the caller's float64 scores when scores_in is given (evict API)
    unsigned long long kmin = ~0ull, kmax = 0ull;
    const double group = (double)a.G;
    const bool pow2 = (a.G & (a.G - 1)) == 0;
    const double inv_group = 1.0 / group;
    // U keys per thread at a time with all their partial loads issued before
    // any is consumed (4 x U loads in flight instead of one dependent load at a
    // time); the partials still add in row-block order (fixed, position-free)
    constexpr int U = RK > 0 ? RK : 4;
    unsigned long long kreg[RK > 0 ? RK : 1];
    for (int64_t j0 = tid; j0 < n; j0 += U * kThreads) {
        double sc[U];
        if (a.scores_in) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t j = j0 + (int64_t)u * kThreads;
                sc[u] = j < n ? a.scores_in[(int64_t)s * n + j] : 0.0;
            }
        } else {
            const float* cp = a.col_partial + (int64_t)s * a.nrb * n;
            double acc[U];
#pragma unroll
            for (int u = 0; u < U; ++u) acc[u] = 0.0;
            for (int rb0 = 0; rb0 < a.nrb; rb0 += 4) {
                float x[4][U];
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int64_t j = j0 + (int64_t)u * kThreads;
                        x[r][u] = (rb0 + r < a.nrb && j < n) ? __ldcg(cp + (int64_t)(rb0 + r) * n + j) : 0.f;
                    }
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (rb0 + r < a.nrb) acc[u] = __dadd_rn(acc[u], (double)x[r][u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u)   // x / G == x * (1/G) exactly when G is a power of two
                sc[u] = pow2 ? __dmul_rn(acc[u], inv_group) : __ddiv_rn(acc[u], group);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t j = j0 + (int64_t)u * kThreads;
            if (RK > 0) kreg[RK > 0 ? u : 0] = order_key(sc[u]);
            if (j >= n) continue;
            if (!a.scores_in && a.scores) a.scores[(int64_t)s * n + j] = sc[u];
            keys[j] = order_key(sc[u]);
        }
    }
    if (early) pdl_wait_then_release();   // K2 done: the budgets are final
    const int64_t k = a.kept_counts[s / a.Hkv];  // same budget for every KV head of a layer
    const int64_t reserve = imin((int64_t)ceil(a.recent_frac * (double)k), k);
    const int64_t nk = k - reserve;
    const int64_t ncand = n - reserve;
    if (RK > 0) {
#pragma unroll
        for (int u = 0; u < (RK > 0 ? RK : 1); ++u)
            if (tid + (int64_t)u * kThreads < ncand) { kmin = min(kmin, kreg[u]); kmax = max(kmax, kreg[u]); }
    } else {
        for (int64_t j = tid; j < ncand; j += kThreads) { kmin = min(kmin, keys[j]); kmax = max(kmax, keys[j]); }
    }
    __syncthreads();
#ifdef VLC_K3_PROBE    // timing probe (wrong results): phase 1 only -- scores and keys
    if (tid == 0 && kmin == 12345ull) a.kept_idx[0] = 0;
    return;
#endif
    if (tid == 0) { s_min = ~0ull; s_max = 0ull; s_prefix = 0ull; s_mask = 0ull; s_want = nk; s_small = 0; s_ncand = 0; }
    __syncthreads();
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(kFull, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(kFull, kmax, o));
    }
    if (nk > 0 && lane == 0) {
        atomicMin(&s_min, kmin);
        atomicMax(&s_max, kmax);
    }
    __syncthreads();

    // 2. radix select of the nk-th largest key among candidates [0, ncand)
    if (nk > 0) {
        // bytes above the first differing byte of (min, max) are common: skip them
        const unsigned long long diff = s_min ^ s_max;
        int top_pass = diff ? (63 - __clzll(diff)) / 8 : -1;
        if (tid == 0 && top_pass < 7) {
            const int keep_bits = (top_pass + 1) * 8;
            const unsigned long long m = keep_bits >= 64 ? 0ull : (~0ull << keep_bits);
            s_prefix = s_min & m;
            s_mask = m;
        }
        __syncthreads();
        for (int pass = top_pass; pass >= 0; --pass) {
            const int shift = pass * 8;
            for (int i = tid; i < 256; i += kThreads) hist[i] = 0;
            if (tid == 0) { s_bmin = ~0ull; s_bmax = 0ull; }
            __syncthreads();
            const unsigned long long prefix = s_prefix, mask = s_mask;
            unsigned long long bmin = ~0ull, bmax = 0ull;   // the bucket's extremes
            if (RK > 0) {
#pragma unroll
                for (int u = 0; u < (RK > 0 ? RK : 1); ++u) {
                    const int64_t j = tid + (int64_t)u * kThreads;
                    const bool in = j < ncand && ((kreg[u] & mask) == prefix);
                    if (!__any_sync(kFull, in)) continue;   // warp-uniform
                    if (in) { bmin = min(bmin, kreg[u]); bmax = max(bmax, kreg[u]); }
                    const unsigned dgt = in ? (unsigned)((kreg[u] >> shift) & 255u) : 256u;
                    const unsigned peers = __match_any_sync(kFull, dgt);
                    if (in && lane == __ffs(peers) - 1) atomicAdd(&hist[dgt], __popc(peers));
                }
            } else {
                for (int64_t j0 = 0; j0 < ncand; j0 += kThreads) {
                    const int64_t j = j0 + tid;
                    const bool in = j < ncand && ((keys[j] & mask) == prefix);
                    if (!__any_sync(kFull, in)) continue;   // warp-uniform
                    if (in) { bmin = min(bmin, keys[j]); bmax = max(bmax, keys[j]); }
                    const unsigned dgt = in ? (unsigned)((keys[j] >> shift) & 255u) : 256u;
                    const unsigned peers = __match_any_sync(kFull, dgt);
                    if (in && lane == __ffs(peers) - 1) atomicAdd(&hist[dgt], __popc(peers));
                }
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                bmin = min(bmin, __shfl_xor_sync(kFull, bmin, o));
                bmax = max(bmax, __shfl_xor_sync(kFull, bmax, o));
            }
            if (lane == 0 && bmin <= bmax) { atomicMin(&s_bmin, bmin); atomicMax(&s_bmax, bmax); }
            __syncthreads();
            if (s_bmin == s_bmax) {
                // one distinct key left in the bucket (a run of ties): it is T and
                // the remaining want are ties at T -- no further passes
                if (tid == 0) s_prefix = s_bmin;
                __syncthreads();
                break;
            }
            if (warp == 0) {
                // lane L covers digits 255-8L .. 248-8L (descending)
                unsigned c[8];
                unsigned tot = 0;
#pragma unroll
                for (int q = 0; q < 8; ++q) { c[q] = hist[255 - 8 * lane - q]; tot += c[q]; }
                unsigned incl = tot;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    unsigned y = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o) incl += y;
                }
                const unsigned excl = incl - tot;
                const long long want = s_want;
                __syncwarp();   // every lane has read s_want before the selecting lane rewrites it
                const bool mine = (long long)excl < want && want <= (long long)incl;
                if (mine) {
                    long long cum = excl;
                    int sel = 0;
                    unsigned cnt = 0;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        if (cum + c[q] >= want) { sel = 255 - 8 * lane - q; cnt = c[q]; break; }
                        cum += c[q];
                    }
                    s_want = want - cum;
                    s_prefix = prefix | ((unsigned long long)sel << shift);
                    s_mask = mask | (255ull << shift);
                    // a bucket of <= 32 keys is finished by one warp (no more passes)
                    s_small = (pass > 0 && cnt <= 32) ? 1 : 0;
                }
            }
            __syncthreads();
            if (s_small) break;
        }
        if (s_small) {
            // gather the bucket's keys, sort them descending in one warp (bitonic
            // over the lanes), the want-th is T
            const unsigned long long prefix = s_prefix, mask = s_mask;
            if (RK > 0) {
#pragma unroll
                for (int u = 0; u < (RK > 0 ? RK : 1); ++u) {
                    const int64_t j = tid + (int64_t)u * kThreads;
                    if (j < ncand && (kreg[u] & mask) == prefix) s_cand[atomicAdd(&s_ncand, 1)] = kreg[u];
                }
            } else {
                for (int64_t j = tid; j < ncand; j += kThreads)
                    if ((keys[j] & mask) == prefix) s_cand[atomicAdd(&s_ncand, 1)] = keys[j];
            }
            __syncthreads();
            if (warp == 0) {
                unsigned long long x = lane < s_ncand ? s_cand[lane] : 0ull;
#pragma unroll
                for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
                    for (int stride = size >> 1; stride > 0; stride >>= 1) {
                        const unsigned long long y = __shfl_xor_sync(kFull, x, stride);
                        const bool desc = (lane & size) == 0;          // descending blocks
                        const bool lower = (lane & stride) == 0;
                        x = (lower == desc) ? max(x, y) : min(x, y);
                    }
                }
                const long long want = s_want;                         // 1 <= want <= bucket size
                const unsigned long long t = __shfl_sync(kFull, x, (int)(want - 1));
                const long long above = __popc(__ballot_sync(kFull, lane < s_ncand && x > t));
                if (lane == 0) { s_prefix = t; s_want = want - above; }
            }
            __syncthreads();
        }
    }
#ifdef VLC_K3_PROBE2   // timing probe (wrong results): phases 1-2 -- no emission
    if (tid == 0 && s_prefix == 12345ull) a.kept_idx[0] = 0;
    return;
#endif
    const unsigned long long T = s_prefix;
    const long long need = s_want;   // ties at T to keep (largest indices first)

    if (RK > 0) {
        // 3'. keys in registers: j = tid + u*kThreads orders as (u, warp, lane),
        //     so warp ballots + one prefix over the (u, warp) counts give each
        //     tie its rank from the right and each kept key its output slot
        constexpr int W = kThreads / 32, E = (RK > 0 ? RK : 2) * W / 32;
        static_assert(RK == 0 || (RK * W) % 32 == 0, "prefix layout");
        __shared__ int s_cnt[RK > 0 ? RK * W : 1], s_pre[RK > 0 ? RK * W : 1], s_tot;
        auto prefix_counts = [&]() {   // s_pre = exclusive prefix of s_cnt, s_tot = sum (warp 0)
            if (warp == 0) {
                int c[E], t = 0;
#pragma unroll
                for (int e = 0; e < E; ++e) { c[e] = s_cnt[lane * E + e]; t += c[e]; }
                int incl = t;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o) incl += y;
                }
                int run = incl - t;
#pragma unroll
                for (int e = 0; e < E; ++e) { s_pre[lane * E + e] = run; run += c[e]; }
                if (lane == 31) s_tot = incl;
            }
        };
        const unsigned below = (1u << lane) - 1u;
        unsigned tb[RK > 0 ? RK : 1];
#pragma unroll
        for (int u = 0; u < (RK > 0 ? RK : 1); ++u) {
            const int64_t j = tid + (int64_t)u * kThreads;
            tb[u] = __ballot_sync(kFull, nk > 0 && j < ncand && kreg[u] == T);
            if (lane == 0) s_cnt[u * W + warp] = __popc(tb[u]);
        }
        __syncthreads();
        prefix_counts();
        __syncthreads();
        const int ties_total = s_tot;
        unsigned kb[RK > 0 ? RK : 1];
#pragma unroll
        for (int u = 0; u < (RK > 0 ? RK : 1); ++u) {
            const int64_t j = tid + (int64_t)u * kThreads;
            bool keep = false;
            if (j < n) {
                if (j >= ncand) keep = true;
                else if (nk > 0) {
                    if (kreg[u] > T) keep = true;
                    else if ((tb[u] >> lane) & 1u) {   // ties strictly to the right
                        const int right = ties_total - (s_pre[u * W + warp] + __popc(tb[u] & below)) - 1;
                        keep = right < need;
                    }
                }
            }
            kb[u] = __ballot_sync(kFull, keep);
        }
        __syncthreads();   // every thread has read s_pre / s_tot
#pragma unroll
        for (int u = 0; u < (RK > 0 ? RK : 1); ++u)
            if (lane == 0) s_cnt[u * W + warp] = __popc(kb[u]);
        __syncthreads();
        prefix_counts();
        __syncthreads();
        const int64_t base = a.kept_off[s];
#pragma unroll
        for (int u = 0; u < (RK > 0 ? RK : 1); ++u)
            if ((kb[u] >> lane) & 1u) {
                const int64_t pos = base + s_pre[u * W + warp] + __popc(kb[u] & below);
                a.kept_idx[pos] = (int32_t)(tid + u * kThreads);
                a.kept_slot[pos] = s;
            }
        return;
    }

    // 3. chunked flags in index order.  A tie at T is kept iff fewer than
    //    `need` ties lie strictly to its right (ties toward the larger index).
    const int64_t chunk = (n + kThreads - 1) / kThreads;
    const int64_t c0 = imin(n, (int64_t)tid * chunk), c1 = imin(n, c0 + chunk);
    long long ties = 0;
    if (nk > 0)
        for (int64_t j = c0; j < c1 && j < ncand; ++j) ties += (keys[j] == T);
    const long long ties_incl = block_inclusive_scan<long long>(ties, scan_scratch);
    __shared__ long long s_ties_total;
    if (tid == kThreads - 1) s_ties_total = ties_incl;
    __syncthreads();
    const long long ties_from_c0 = s_ties_total - ties_incl + ties;   // ties with index >= c0
    auto walk = [&](bool write, int64_t out_pos) -> long long {
        long long right = ties_from_c0, kept = 0;
        for (int64_t j = c0; j < c1; ++j) {
            bool keep;
            if (j >= ncand) keep = true;
            else if (nk == 0) keep = false;
            else if (keys[j] > T) keep = true;
            else if (keys[j] == T) { --right; keep = right < need; }
            else keep = false;
            if (keep) {
                if (write) {
                    a.kept_idx[out_pos + kept] = (int32_t)j;
                    a.kept_slot[out_pos + kept] = s;
                }
                ++kept;
            }
        }
        return kept;
    };
    const long long kept_here = walk(false, 0);
    const long long pos_incl = block_inclusive_scan<long long>(kept_here, scan_scratch);
    walk(true, a.kept_off[s] + (pos_incl - kept_here));
}

}  // namespace

cudaError_t launch_select(const SelectArgs& a, cudaStream_t st) {
    if (a.n > kSmemKeysMax && !a.key_scratch) return cudaErrorInvalidValue;  // needs global scratch
    const size_t sm = a.n <= kSmemKeysMax ? sizeof(unsigned long long) * (size_t)a.n : 0;
    if (a.n <= 6 * kThreads) return launch_pdl(select_kernel<6>, dim3(a.slots), dim3(kThreads), sm, st, a);
    cudaFuncSetAttribute(select_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kSmemKeysMax * 8));
    return launch_pdl(select_kernel<0>, dim3(a.slots), dim3(kThreads), sm, st, a);
}

}  // namespace vlc
