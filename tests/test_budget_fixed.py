"""Uniform / pyramid budgets (reference budget.py:114-147): the reference's own
known-answer tests (pkg/tests/test_budget.py TestKeptCounts / TestUniform /
TestPyramid), restated.  Host arithmetic only -- no GPU needed."""

import numpy as np
import pytest

from paper_2410_23317_b200 import ValidationError, allocate_pyramid, allocate_uniform


def test_uniform_kept_counts_ceil_and_cap():
    np.testing.assert_array_equal(allocate_uniform(0.1, 3, 100).kept_counts, [10, 10, 10])
    np.testing.assert_array_equal(allocate_uniform(1.0, 2, 17).kept_counts, [17, 17])
    a = allocate_uniform(0.1, 8, 100)
    np.testing.assert_array_equal(a.beta, np.full(8, 0.1))
    assert a.kept_counts.sum() == 80
    assert all(r["gamma_mean"] is None for r in a.to_rows())


def test_pyramid_known_answers():
    np.testing.assert_allclose(allocate_pyramid(0.2, 5, 100, decay_ratio=1.0).beta_preclip, 0.2, atol=1e-15)
    np.testing.assert_allclose(allocate_pyramid(0.2, 4, 100, decay_ratio=0.5).beta_preclip,
                               [0.3, 0.7 / 3.0, 0.5 / 3.0, 0.1], atol=1e-12)
    rng = np.random.default_rng(11)
    for _ in range(30):
        alpha, n, ratio = float(rng.uniform(0.02, 0.5)), int(rng.integers(1, 16)), float(rng.uniform(0.05, 1.0))
        a = allocate_pyramid(alpha, n, 200, decay_ratio=ratio)
        assert a.beta_preclip.mean() == pytest.approx(alpha, abs=1e-9)
        assert (np.diff(a.beta_preclip) <= 1e-15).all()
        np.testing.assert_array_equal(a.kept_counts, np.clip(np.ceil(a.beta * 200), 1, 200).astype(np.int64))


def test_bad_arguments():
    for bad in (0.0, 1.5, -1.0):
        with pytest.raises(ValidationError, match="decay_ratio"):
            allocate_pyramid(0.1, 4, 100, decay_ratio=bad)
    with pytest.raises(ValidationError, match="num_layers"):
        allocate_uniform(0.1, 0, 100)
    with pytest.raises(ValidationError, match="alpha"):
        allocate_uniform(0.0, 4, 100)
