for f in "$@"; do VLC_LIB_PATH=$f timeout 300 python tools/k1_quick.py 2>&1 | tail -1; done
