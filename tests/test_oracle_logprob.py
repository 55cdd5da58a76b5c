"""Pins for oracle.logprob (S3): normalisation, closed forms, library routines (scipy),
SPEC's toyrl softmax examples and central finite differences."""
import numpy as np
import pytest
from scipy.special import log_softmax as sp_log_softmax
from scipy.stats import entropy as sp_entropy

from oracle import logprob as L
from tests.conftest import read_golden


def test_normalisation_all_targets():
    rng = np.random.default_rng(0)
    x = rng.normal(0, 2, size=(1, 300))
    lp = np.array([L.log_softmax_gather(x, [j])["logp"][0] for j in range(300)])
    assert abs(np.exp(lp).sum() - 1.0) < 1e-13


@pytest.mark.parametrize("row", [r for r in read_golden("softmax_examples.csv") if r[0] == "uniform"])
def test_uniform_row(row):
    V, exp = int(row[1]), float(row[2])
    f = L.log_softmax_gather(np.full((2, V), 0.37), [0, V - 1])
    assert np.allclose(f["logp"], exp, atol=1e-13, rtol=0)
    assert np.allclose(f["entropy"], np.log(V), atol=1e-10)


def test_matches_scipy_log_softmax_and_entropy():
    rng = np.random.default_rng(1)
    x = rng.normal(0, 3, size=(20, 513))
    t = rng.integers(0, 513, size=20)
    f = L.log_softmax_gather(x, t)
    ref = sp_log_softmax(x, axis=1)
    np.testing.assert_allclose(f["logp"], ref[np.arange(20), t], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(f["entropy"], [sp_entropy(np.exp(r)) for r in ref], rtol=1e-10)


def test_saturation_and_shift_invariance():
    V = 32000
    x = np.full((1, V), -30.0)
    x[0, 5] = 30.0
    f = L.log_softmax_gather(x, [5])
    assert -1e-20 < f["logp"][0] <= 0.0      # 1 - p >= 1 - 1e-40
    rng = np.random.default_rng(2)
    y = rng.normal(size=(5, 64))
    a = L.log_softmax_gather(y, [1, 2, 3, 4, 5])["logp"]
    b = L.log_softmax_gather(y + 1234.5, [1, 2, 3, 4, 5])["logp"]
    np.testing.assert_allclose(a, b, atol=1e-10)


def test_tied_maxima_and_neg_inf_columns():
    x = np.array([[5.0, 5.0, -np.inf, -np.inf]])
    f = L.log_softmax_gather(x, [1])
    assert abs(f["logp"][0] + np.log(2)) < 1e-15 and f["status"][0] == 0
    assert abs(f["entropy"][0] - np.log(2)) < 1e-15
    rng = np.random.default_rng(3)
    y = rng.normal(size=(1, 40))
    keep = rng.random(40) > 0.3
    keep[7] = True
    z = np.where(keep, y, -np.inf)
    ref = sp_log_softmax(y[:, keep], axis=1)[0, keep[:7].sum()]
    assert abs(L.log_softmax_gather(z, [7])["logp"][0] - ref) < 1e-13


def test_status_codes():
    x = np.zeros((5, 8))
    x[3, 2] = np.nan
    x[4, :] = -np.inf
    f = L.log_softmax_gather(x, [-1, 8, 0, 0, 0])
    assert f["status"].tolist() == [1, 2, 0, 3, 3]
    assert f["logp"][0] == 0 and f["logp"][1] == 0
    assert np.isnan(f["logp"][3]) and np.isnan(f["logp"][4])


def test_spec_uniform4_gradient():
    row = [r for r in read_golden("softmax_examples.csv") if r[0] == "grad_uniform4"][0]
    exp = np.array([float(v) for v in row[2].split()])
    x = np.zeros((1, 4))
    f = L.log_softmax_gather(x, [0])
    dx = L.log_softmax_grad(x, [0], f["lse"], [1.0])
    np.testing.assert_allclose(dx[0], exp, atol=1e-15)


def test_grad_sums_to_zero_and_finite_differences():
    rng = np.random.default_rng(4)
    for V in (2, 5, 16):
        x = rng.normal(0, 1.5, size=(3, V))
        t = rng.integers(0, V, size=3)
        g = rng.normal(size=3)
        f = L.log_softmax_gather(x, t)
        dx = L.log_softmax_grad(x, t, f["lse"], g)
        assert np.abs(dx.sum(axis=1)).max() < 1e-14
        h = 1e-5
        for r in range(3):
            for j in range(V):
                xp, xm = x.copy(), x.copy()
                xp[r, j] += h
                xm[r, j] -= h
                fd = g[r] * (L.log_softmax_gather(xp, t)["logp"][r] -
                             L.log_softmax_gather(xm, t)["logp"][r]) / (2 * h)
                assert abs(fd - dx[r, j]) <= 1e-6 * max(1.0, abs(dx[r, j]))


def test_saturated_target_gradient_closed_form():
    """Target +30, V-1 others -30: 1 - p_a = (V-1)e^-60 / (1 + (V-1)e^-60) (closed form);
    the oracle must not cancel it to 0 (cf. S:398 saturation example)."""
    for V in (4, 256, 32000):
        x = np.full((1, V), -30.0)
        x[0, 2] = 30.0
        f = L.log_softmax_gather(x, [2])
        dx = L.log_softmax_grad(x, [2], f["lse"], [-2.0])
        q = (V - 1) * np.exp(-60.0)
        assert abs(dx[0, 2] - (-2.0) * q / (1 + q)) <= 1e-12 * abs(dx[0, 2])
        assert abs(dx[0, 0] - 2.0 * np.exp(-60.0) / (1 + q)) <= 1e-12 * abs(dx[0, 0])
        assert abs(dx.sum()) <= 1e-12 * abs(dx[0, 2])
