"""The .vlct trace format (reference trace.py:329-394): our reader reads the
file the REFERENCE writer produced (tests/golden/ref_small.vlct, made by
tests/golden/make_vlct.py) and our writer reproduces it byte for byte; the
reference's failure modes map to the same error types.  Host I/O, no GPU."""

import os

import numpy as np
import pytest

from conftest import ROOT
from paper_2410_23317_b200 import errors
from paper_2410_23317_b200.trace import GenSpec, generate_trace, read_trace, write_trace

GOLD = os.path.join(ROOT, "tests", "golden", "ref_small.vlct")


def test_reads_reference_file_and_matches_generator():
    tr = read_trace(GOLD)
    h = tr.header
    assert (h.num_layers, h.num_query_heads, h.num_kv_heads, h.head_dim, h.prompt_len, h.post_vision_len,
            h.decode_len, h.seed) == (2, 4, 2, 16, 40, 8, 3, 5)
    ours, _ = generate_trace(GenSpec(2, 4, 2, 16, 40, 8, 3, 5))
    for l in range(2):
        np.testing.assert_array_equal(tr.queries[l], ours.queries[l])
        np.testing.assert_array_equal(tr.keys[l], ours.keys[l])
    mm = read_trace(GOLD, mmap=True)
    np.testing.assert_array_equal(mm.keys[1], tr.keys[1])


def test_writer_is_byte_identical(tmp_path):
    tr, _ = generate_trace(GenSpec(2, 4, 2, 16, 40, 8, 3, 5))
    out = tmp_path / "t.vlct"
    write_trace(tr, out)
    assert out.read_bytes() == open(GOLD, "rb").read()
    assert (tmp_path / "t.vlct.json").read_text() == open(GOLD + ".json").read()


def test_error_modes(tmp_path):
    raw = open(GOLD, "rb").read()
    (tmp_path / "short").write_bytes(raw[:20])
    with pytest.raises(errors.TraceTruncatedError):
        read_trace(tmp_path / "short")
    (tmp_path / "cut").write_bytes(raw[:-4])
    with pytest.raises(errors.TraceTruncatedError):
        read_trace(tmp_path / "cut")
    (tmp_path / "magic").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(errors.TraceFormatError):
        read_trace(tmp_path / "magic")
    (tmp_path / "ver").write_bytes(raw[:4] + (2).to_bytes(4, "little") + raw[8:])
    with pytest.raises(errors.TraceFormatError):
        read_trace(tmp_path / "ver")
