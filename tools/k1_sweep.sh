#!/bin/bash
# K1 variants (exp_libs/k1*.so) at the bench workload, cold L2
for f in exp_libs/k1*.so; do VLC_LIB_PATH=$f timeout 300 python tools/k1_timing.py 2>&1 | tail -1; done
