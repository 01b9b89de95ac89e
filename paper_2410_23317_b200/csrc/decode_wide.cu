// decode_wide.cu -- K5 with the wide CTA for grids smaller than the GPU:
// decode.cu built again with two-warp groups on 32-row tiles (256 threads,
// 96 KB), entry point launch_decode_wide (launch_decode picks it when there
// are fewer slots than SMs).
#define VLC_DEC_GROUP_WARPS 2
#define VLC_DEC_LAUNCH launch_decode_wide
#include "decode.cu"
