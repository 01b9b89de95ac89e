"""Per-warp timeline of the 99 K5 launches of one CUDA-graph decode (library
built with -DVLC_DEC_TRACE):
  python -c "from paper_2410_23317_b200 import build; build.build(out='exp_libs/trace.so', defines=['VLC_DEC_TRACE'])"
  VLC_LIB_PATH=exp_libs/trace.so python tools/decode_trace.py
events per (step, CTA*warps+warp): 0 start, 1 plan loaded, 2 first tiles issued,
3 past griddepcontrol.wait, 4 first tile landed, 5 end, 6 tiles, 7 slots of the CTA."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_23317_b200 import _lib  # noqa: E402
from paper_2410_23317_b200.engine import Shape, VLCache  # noqa: E402

c = bench.CFG
n_dec = c["n_out"] - 1
qw, qd, ks, vs = bench.synth_inputs(1, 0, c["tau"])
dev = lambda a: torch.from_numpy(a).to(torch.bfloat16).cuda()  # noqa: E731
d_qw, d_qd, d_k, d_v = dev(qw), dev(qd), dev(ks), dev(vs)
eng = VLCache(Shape(1, c["layers"], c["q_heads"], c["kv_heads"], c["head_dim"], c["prompt_len"], c["tau"]),
              alpha=c["alpha"], p=c["p"], recent_frac=c["recent"], decode_steps=n_dec)
lib = _lib.load()
lib.vlc_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_longlong]
buf = np.zeros((100, 4096, 12), dtype=np.uint64)
for rep in range(3):
    eng.compress(d_qw, d_k, d_v)
    eng.decode(d_qd, d_k, d_v, graph=True)
    torch.cuda.synchronize()
lib.vlc_debug_trace(buf.ctypes.data_as(ctypes.c_void_p), buf.nbytes)
t = buf.astype(np.int64)
used = t[0, :, 5] > 0
t = t[:, used]
T0 = t[0, :, 0].min()
starts, ends = t[:, :, 0].min(1), t[:, :, 5].max(1)
print(f"warps {used.sum()}  tiles/warp median {np.median(t[50, :, 6]):.0f} max {t[50, :, 6].max()}")
print("step start end dur | median rel. to step start: plan issued waited landed end | p90 end")
for s in [0, 1, 2, 3, 50, 51, 97, 98]:
    st = starts[s]
    rel = lambda e: np.median(t[s, :, e] - st) / 1e3  # noqa: E731
    print(f"{s:3d} {(st - T0) / 1e3:8.2f} {(ends[s] - T0) / 1e3:8.2f} {(ends[s] - st) / 1e3:6.2f} | "
          f"{rel(1):5.2f} {rel(2):5.2f} {rel(3):5.2f} {rel(4):5.2f} {rel(5):5.2f} | "
          f"{np.percentile(t[s, :, 5] - st, 90) / 1e3:5.2f}")
print(f"99 steps: {(ends[98] - starts[0]) / 1e3:.1f} us ({(ends[98] - starts[0]) / 1e3 / 99:.2f} us/step); "
      f"start(s+1)-end(s) median {np.median(starts[1:99] - ends[:98]) / 1e3:.2f} us")
s = 50
st = starts[s]
loop = (t[s, :, 5] - t[s, :, 4]) / 1e3
tiles = t[s, :, 6]
print(f"step 50 loop (landed->end) median {np.median(loop):.2f} us max {loop.max():.2f}; per tile median "
      f"{np.median(loop / np.maximum(tiles, 1)):.2f} us; start spread {(t[s, :, 0].max() - st) / 1e3:.2f} us")
slow = np.argsort(-(t[s, :, 5] - st))[:6]
for w in slow:
    x = (t[s, w, :6] - st) / 1e3
    print("   warp", w, np.round(x, 2).tolist(), "tiles", t[s, w, 6], "slots", t[s, w, 7])
cw, cc, ci = t[s, :, 8], t[s, :, 9], t[s, :, 10]
print(f"step 50 per warp cycles: wait median {np.median(cw):.0f} compute {np.median(cc):.0f} issue {np.median(ci):.0f}"
      f"  (per tile: wait {np.median(cw / tiles):.0f} compute {np.median(cc / tiles):.0f} issue {np.median(ci / tiles):.0f})")
