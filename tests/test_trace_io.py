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


def _cli_kwargs(args):
    """The reference CLI flags of a golden run as compress_outputs arguments."""
    kw, i = {}, 0
    names = {"--policy": ("policy", str), "--budget": ("budget", str), "--sliding-window": ("sliding_window", int),
             "--alpha": ("alpha", float), "--recent-frac": ("recent_frac", float),
             "--stats-window": ("stats_window", int)}
    while i < len(args):
        key, typ = names[args[i]]
        kw[key] = typ(args[i + 1])
        i += 2
    return kw


@pytest.mark.gpu
def test_compress_outputs_equal_reference_cli_files(tmp_path):
    """allocation.json / kept_sets.json byte-identical to the reference CLI's
    `compress` (cli.py:195-203) for several policy x budget choices
    (tests/golden/cli_golden.json, tests/golden/make_cli_golden.py)."""
    import json as _json
    import os as _os

    from paper_2410_23317_b200.outputs import write_compress_outputs
    from paper_2410_23317_b200.trace import AttentionTrace, GenSpec, generate_trace, round_to_bf16

    with open(_os.path.join(_os.path.dirname(_os.path.abspath(__file__)), "golden", "cli_golden.json")) as f:
        golden = _json.load(f)
    traces = {}
    for name, spec in golden["specs"].items():
        tr, _ = generate_trace(GenSpec(**spec))
        traces[name] = AttentionTrace(header=tr.header, layout=tr.layout,
                                      queries=[round_to_bf16(x) for x in tr.queries],
                                      keys=[round_to_bf16(x) for x in tr.keys])
    for i, run in enumerate(golden["runs"]):
        out = tmp_path / f"run{i}"
        stdout = write_compress_outputs(out, traces[run["trace"]], **_cli_kwargs(run["args"]))
        assert (out / "allocation.json").read_text() == run["allocation.json"], run["args"]
        assert (out / "kept_sets.json").read_text() == run["kept_sets.json"], run["args"]
        assert _json.dumps(stdout) == run["stdout"].strip(), run["args"]
