"""The CPU oracle pinned against the reference: its golden vectors and its KATs.

Golden vectors come from running the reference itself (tests/golden/make_golden.py);
the known-answer tests restate pkg/tests/test_oracle.py:23-146 of the reference.
"""

import numpy as np
import pytest

from oracle import conv_ref
from tests import golden_cases


CASES, ARRAYS = golden_cases.load()


def test_golden_inventory():
    ids = [c["id"] for c in CASES]
    assert sum(i.startswith("rand") for i in ids) == 40
    assert sum(i.startswith("twin") for i in ids) == 43
    assert {"full34", "full02", "full13", "full36"} <= set(ids)


@pytest.mark.parametrize("case", CASES, ids=[c["id"] for c in CASES])
def test_noise_matches_reference_inputs(case):
    x, f, b = golden_cases.inputs(case)
    assert golden_cases.digest(x) == case["x_digest"]
    assert golden_cases.digest(f) == case["f_digest"]
    assert golden_cases.digest(b) == case["b_digest"]


@pytest.mark.parametrize("case", CASES, ids=[c["id"] for c in CASES])
def test_oracle_matches_reference_outputs(case):
    x, f, b = golden_cases.inputs(case)
    got = conv_ref.ref_conv(x, f, b, case["stride"], case["pad"], relu=case["act"] == "relu")
    assert list(got.shape) == case["out_shape"]
    want, step = golden_cases.expected(case, ARRAYS)
    flat = got.reshape(-1)[::step]
    # both sides accumulate in float64 and round once to fp32: at most 1 ulp apart
    np.testing.assert_allclose(flat, want, rtol=2.5e-7, atol=0)
    assert conv_ref.compare(flat, want, conv_ref.Tol(1e-6, 0.0)).ok


def test_kat_single_fma():
    out = conv_ref.ref_conv(np.full((1, 1, 1, 1), 3, np.float32), np.full((1, 1, 1, 1), 2, np.float32),
                            np.array([1], np.float32), 1, 0)
    assert out[0, 0, 0, 0] == 7.0


def test_kat_identity_kernel():
    x = np.random.default_rng(0).uniform(0.1, 1, (1, 3, 4, 4)).astype(np.float32)
    f = np.zeros((3, 3, 1, 1), np.float32)
    for c in range(3):
        f[c, c, 0, 0] = 1
    assert np.array_equal(conv_ref.ref_conv(x, f, np.zeros(3, np.float32), 1, 0), x)


def test_kat_window_is_363_term_dot():
    x = conv_ref.noise((1, 3, 15, 15), 1)
    f = conv_ref.noise((2, 3, 11, 11), 2)
    out = conv_ref.ref_conv(x, f, np.array([0.5, -0.5], np.float32), 4, 0)
    manual = float(np.sum(x[0, :, :11, :11].astype(np.float64) * f[0].astype(np.float64)) + 0.5)
    assert out[0, 0, 0, 0] == pytest.approx(manual, rel=1e-6)
    assert out.shape == (1, 2, 2, 2)


def test_kat_linearity_and_zero_filters():
    x = conv_ref.noise((1, 2, 5, 5), 3)
    f = conv_ref.noise((4, 2, 3, 3), 4)
    z = np.zeros(4, np.float32)
    base = conv_ref.ref_conv(x, f, z, 1, 1).astype(np.float64)
    assert np.allclose(conv_ref.ref_conv(3 * x, f, z, 1, 1), 3 * base, rtol=1e-6)
    out = conv_ref.ref_conv(x[:, :2, :4, :4], np.zeros((2, 2, 3, 3), np.float32), np.array([0.25, -1.5], np.float32), 1, 1)
    assert np.all(out[0, 0] == np.float32(0.25)) and np.all(out[0, 1] == np.float32(-1.5))


def test_compare_rules():
    one = np.array([1.0], np.float32)
    assert conv_ref.compare(one, np.array([1.0005], np.float32), conv_ref.Tol(1e-3)).ok
    res = conv_ref.compare(one, np.array([1.01], np.float32), conv_ref.Tol(1e-3))
    assert not res.ok and res.worst_index == (0,)
    a = conv_ref.noise((32,), 9)
    b = (a * np.float32(1.000004)).astype(np.float32)
    assert conv_ref.compare(a, b).ok == conv_ref.compare(b, a).ok
    assert conv_ref.compare(np.zeros(1, np.float32), np.array([5e-7], np.float32)).ok
    assert conv_ref.tolerance_for(100).rel_tol == 1e-5 and conv_ref.tolerance_for(5000).rel_tol == 1e-3


def test_noise_range_and_determinism():
    a = conv_ref.noise((7, 13), conv_ref.seed_for("sig"))
    assert np.array_equal(a, conv_ref.noise((7, 13), conv_ref.seed_for("sig")))
    assert a.min() >= 0.1 and a.max() < 1.0


def test_relu_clips_signed():
    x = conv_ref.noise((1, 2, 6, 6), 5, -1.0, 1.0)
    f = conv_ref.noise((3, 2, 3, 3), 6, -1.0, 1.0)
    b = np.zeros(3, np.float32)
    plain = conv_ref.ref_conv(x, f, b, 1, 1)
    fused = conv_ref.ref_conv(x, f, b, 1, 1, relu=True)
    assert (plain < 0).any()
    assert np.array_equal(fused, np.maximum(plain, 0))
