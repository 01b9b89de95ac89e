"""Write tests/golden/ref_small.vlct (+ .json) with the REFERENCE's own writer
(reference pkg/src/vlcache/trace.py:332-356) on a small generator trace.
Run here, where /root/reference is mounted:  python tests/golden/make_vlct.py
The file is committed; tests/test_trace_io.py checks our reader / writer
against it byte for byte (the GPU box never reads /root/reference)."""
import os
import sys

os.environ["VLCACHE_PURE_PYTHON"] = "1"
sys.path.insert(0, "/root/reference/pkg/src")
import vlcache  # noqa: E402
from vlcache import trace as T  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
spec = T.GenSpec(num_layers=2, num_query_heads=4, num_kv_heads=2, head_dim=16, prompt_len=40,
                 post_vision_len=8, decode_len=3, seed=5)
tr, _ = T.generate_trace(spec)
T.write_trace(tr, os.path.join(HERE, "ref_small.vlct"))
print("wrote", os.path.join(HERE, "ref_small.vlct"), vlcache.BACKEND)
