rm -f gpurun_out/k5_ref*.npy
for a in ${ALPHAS:-0.1}; do
for f in "$@"; do ALPHA=$a VLC_LIB_PATH=$f timeout 300 python tools/k5_quick.py 2>&1 | grep "graph" | tail -1; done
done
