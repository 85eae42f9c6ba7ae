"""CPU tests of the Eq.1 / Eq.2 solo-run predictors and the best-fit split rule
(paper_2504_14489_b200/costmodel.py; SPEC best_fit_partition)."""
import numpy as np
import pytest

from paper_2504_14489_b200 import costmodel as cm


def test_features_follow_eq1_eq2():
    # Eq.1 terms: sum n^2, sum n r, sum n, 1 ; Eq.2 terms: sum r, bs, 1
    np.testing.assert_array_equal(cm.prefill_features([0, 10], [3, 4]), [9 + 16, 0 + 40, 7, 1])
    np.testing.assert_array_equal(cm.decode_features([5, 7, 9]), [21, 3, 1])


@pytest.mark.parametrize("kind", ["prefill", "decode"])
def test_fit_recovers_exact_coefficients(kind):
    g = np.random.default_rng(1)
    if kind == "prefill":
        theta = np.array([2e-5, 5e-5, 0.05, 30.0])
        X = np.stack([cm.prefill_features(g.integers(0, 20000, size=k), g.integers(1, 8192, size=k))
                      for k in g.integers(1, 5, size=40)])
    else:
        theta = np.array([6e-4, 0.3, 45.0])
        X = np.stack([cm.decode_features(g.integers(1, 8192, size=k)) for k in g.integers(1, 256, size=40)])
    t = X @ theta
    f = cm.fit(X, t)
    np.testing.assert_allclose(f.theta, theta, rtol=1e-6)
    assert f.max_dev < 1e-8


def test_fit_is_nonnegative():
    # data generated with a negative constant: NNLS keeps every cost term >= 0
    X = np.stack([cm.decode_features([r] * 4) for r in (100, 1000, 5000, 9000)])
    t = X @ np.array([1e-3, 0.5, -2.0]) + 10
    assert (cm.fit(X, t).theta >= 0).all()


def test_best_fit_split_spec_example():
    """SPEC best_fit_partition example: worst-case TBT per config {96:40, 80:55, 64:70, 48:95,
    32:130} ms with a 100 ms SLO -> 48 decode SMs; a loose SLO -> the smallest config; an
    impossible one -> None."""
    tbt_ms = {96: 40, 80: 55, 64: 70, 48: 95, 32: 130}
    dec = {s: cm.Fit(np.array([0.0, 0.0, t * 1000.0]), 0.0, 0.0, 1) for s, t in tbt_ms.items()}
    model = cm.CostModel(prefill={}, decode=dec, max_slowdown_dec={s: 1.0 for s in tbt_ms})
    splits = [(s, 148 - s) for s in tbt_ms]
    assert model.best_fit_split(splits, [1000], 1, 100_000)[0] == 48
    assert model.best_fit_split(splits, [1000], 1, 1_000_000)[0] == 32
    assert model.best_fit_split(splits, [1000], 1, 30_000) is None


def test_worst_case_applies_guard_slowdown():
    dec = {32: cm.Fit(np.array([1e-3, 0.0, 10.0]), 0, 0, 1)}
    model = cm.CostModel({}, dec, max_slowdown_dec={32: 1.25})
    assert model.worst_case_decode(32, [9999, 1]) == pytest.approx((10.0 + 10.0) * 1.25)


def test_json_roundtrip():
    dec = {16: cm.Fit(np.array([1e-3, 0.2, 40.0]), 0.05, 0.02, 14)}
    pf = {132: cm.Fit(np.array([1e-5, 2e-5, 0.03, 40.0]), 0.1, 0.05, 20)}
    m = cm.CostModel(pf, dec, {16: 1.2}, {132: 1.1})
    m2 = cm.CostModel.from_json(m.to_json())
    assert m2.t_decode(16, [100, 200]) == pytest.approx(m.t_decode(16, [100, 200]))
    assert m2.t_prefill(132, [0], [1024]) == pytest.approx(m.t_prefill(132, [0], [1024]))
    assert m2.max_slowdown_dec == {16: 1.2}
