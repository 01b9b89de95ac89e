ALPHAS="0.1" bash tools/_k5v.sh exp_libs/dec_pf0.so exp_libs/dec_pf1.so exp_libs/dec_pf0.so exp_libs/dec_pf1.so
BATCH=8 VLC_LIB_PATH=exp_libs/dec_pf0.so python tools/k5_quick.py 2>&1 | grep graph
BATCH=8 VLC_LIB_PATH=exp_libs/dec_pf1.so python tools/k5_quick.py 2>&1 | grep graph
