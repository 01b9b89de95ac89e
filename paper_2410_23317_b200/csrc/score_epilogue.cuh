// score_epilogue.cuh -- per-row softmax-statistics epilogue of K1 (score_stats).
//
// One thread owns one window row and sees its logits 32 keys at a time (a
// "chunk": 32 TMEM columns from tcgen05.ld, or 32 CUDA-core dots).  Two
// passes over all keys, as in the reference (pkg/src/vlcache/_kernels/
// _core.pyx:110-207):
//   pass 1: running row max M and rescaled row sum S         (_core.pyx:142-155)
//   pass 2: t = l - M; e = exp(t) / S; column sums of e;     (_core.pyx:198-205)
//           below-threshold count as the float32 compare t < t*, where t* is
//           the smallest float with (double)expf(t*) >= p -- equivalent to the
//           reference's "(double)expf(l - max) < p" for the monotone libm expf,
//           and independent of the device exp implementation.
#pragma once

#include "vlc_common.cuh"

namespace vlc {

struct RowStats {
    float m;  // running max of logits (f32, as _core.pyx:119)
    float s;  // running sum of exp(l - m)
};

VLC_DEV void pass1_chunk(const float (&l)[32], int valid, RowStats& st) {
    float cmax = -INFINITY;
#pragma unroll
    for (int c = 0; c < 32; ++c)
        if (c < valid) cmax = fmaxf(cmax, l[c]);
    if (cmax > st.m) {
        st.s *= ex2((st.m - cmax) * kLog2e);  // s == 0 while m == -inf
        st.m = cmax;
    }
    float acc = 0.f;
#pragma unroll
    for (int c = 0; c < 32; ++c)
        if (c < valid) acc += ex2((l[c] - st.m) * kLog2e);
    st.s += acc;
}

// e[c] = exp(l - m) / s for visible keys, 0 otherwise; returns the number of
// visible entries with (l - m) < t_star.
VLC_DEV int pass2_chunk(const float (&l)[32], int valid, float m, float log2s, float t_star,
                        float (&e)[32]) {
    int below = 0;
#pragma unroll
    for (int c = 0; c < 32; ++c) {
        const float t = l[c] - m;  // bitwise the reference's float argument of expf
        const bool vis = c < valid;
        e[c] = vis ? ex2(fmaf(t, kLog2e, -log2s)) : 0.f;
        below += (vis && t < t_star) ? 1 : 0;
    }
    return below;
}

}  // namespace vlc
