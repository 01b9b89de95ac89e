// score_stats.cu -- K1 launcher: zeroes the count outputs, then runs the
// tcgen05 kernel (score_stats_tc.cu).  reference _core.pyx:210-242.
#include "vlc_kernels.h"

namespace vlc {

// col_partial rows per slot: 4 row groups of 32 rows per 128-row block
int score_partials(int64_t rows) { return (int)(4 * ((rows + 127) / 128)); }

cudaError_t launch_score_stats(const ScoreArgs& a, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(a.below_head, 0, sizeof(unsigned long long) * a.slots * a.G, st);
    if (e != cudaSuccess) return e;
    if (a.below_col) {
        e = cudaMemsetAsync(a.below_col, 0, sizeof(int) * a.slots * a.n, st);
        if (e != cudaSuccess) return e;
    }
    return launch_score_stats_tc(a, score_partials((int64_t)a.G * a.w), st);
}

}  // namespace vlc
