#!/bin/bash
# K5 variants (exp_libs/*.so built with other defines) at the bench workload
for f in exp_libs/*.so; do case $f in *trace*|*prof*) continue;; esac
  VLC_LIB_PATH=$f timeout 300 python tools/diag_m7b.py 2>&1 | tail -1 | sed "s|^|$f |"; done
