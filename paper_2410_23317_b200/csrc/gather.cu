// gather.cu -- K4: compact the kept K/V rows into ragged cache segments.
//
// reference: bench.py:331-353 (_make_seq_buffers: keys[l][kv, idx] and
// values[l][kv, idx] copied into a buffer of k_l + n_out rows).
// Segment of slot s starts at cache_off[s] and holds k_s kept rows followed by
// decode headroom.  Grid-stride over 16-byte pieces of all kept rows (K and V
// together): every load and store is a coalesced 128-bit access.
#include "vlc_common.cuh"
#include "vlc_kernels.h"

namespace vlc {
namespace {

__global__ void __launch_bounds__(256) gather_kernel(GatherArgs a) {
    pdl_wait_then_release();
    const int64_t total_rows = a.kept_off[a.slots];
    const int pieces = a.d / 8;   // 8 bf16 per 16-byte piece
    const int64_t total = total_rows * pieces;
    const uint4* kin = static_cast<const uint4*>(a.k);
    const uint4* vin = static_cast<const uint4*>(a.v);
    uint4* kout = static_cast<uint4*>(a.k_cache);
    uint4* vout = static_cast<uint4*>(a.v_cache);
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / pieces;
        const int c = (int)(t - r * pieces);
        const int s = a.kept_slot[r];
        const int64_t src = ((int64_t)s * a.T + a.kept_idx[r]) * pieces + c;
        const int64_t dst = (a.cache_off[s] + (r - a.kept_off[s])) * pieces + c;
        const uint4 kv = __ldg(kin + src);
        const uint4 vv = __ldg(vin + src);
        kout[dst] = kv;
        vout[dst] = vv;
    }
}

}  // namespace

cudaError_t launch_gather(const GatherArgs& a, cudaStream_t st) {
    const int64_t total = a.max_rows * (a.d / 8);
    int blocks = (int)imin((total + 255) / 256, 148 * 16);
    if (blocks < 1) blocks = 1;
    return launch_pdl(gather_kernel, dim3(blocks), dim3(256), 0, st, a);
}

}  // namespace vlc
