"""Correlation pruning with the statistics on the GPU vs the
reference prune_two_stage (tests/golden/prune_cases.json, recorded from
gpukalc_trainer with pandas 3.0 / scipy): identical drop decisions; Kendall
coefficients bit-identical (exact integer counts + scipy's expression),
Pearson within 1e-12."""

import json

import numpy as np
import pytest

from goldens import G


def frame(n, seed):
    """Synthetic feature frame: linear and monotone (non-linear) correlates,
    heavy ties (integer columns), signed zeros, one constant column."""
    import pandas as pd

    rng = np.random.default_rng(seed)
    a = rng.random(n)
    b = rng.integers(0, 12, n).astype(float)
    X = pd.DataFrame({
        "occupancy": a,
        "a_lin": 3.0 * a + rng.normal(0, 0.05, n),          # Pearson-correlated with occupancy
        "a_exp": np.exp(6.0 * a) + rng.normal(0, 0.01, n),   # monotone: Kendall catches it
        "block_size": b,
        "b_tie": np.floor(b / 3.0) + 0.0,                     # tied, rank-correlated
        "noise": rng.normal(0, 1, n),
        "zeros": np.where(rng.random(n) < 0.5, 0.0, -0.0) * rng.integers(0, 2, n),
        "const": np.full(n, 7.0),
        "neg": -a * a + rng.normal(0, 0.02, n),
        "cnt": rng.poisson(3.0, n).astype(float),
    })
    y = pd.Series(30.0 + 40.0 * a + rng.normal(0, 1, n), name="power_w")
    return X, y


def _cases():
    return json.loads((G / "prune_cases.json").read_text())


@pytest.mark.gpu
def test_kendall_matrix_bit_identical_to_reference():
    from paper_2305_01886_b200.pruning import kendall_matrix

    for c in _cases():
        X, _ = frame(c["n"], c["seed"])
        X = X.loc[:, X.nunique() > 1]
        got = kendall_matrix(X.to_numpy(dtype=float))
        want = np.asarray(c["kendall"])
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (c["n"], got - want)


@pytest.mark.gpu
def test_pearson_matrix_matches_reference():
    from paper_2305_01886_b200.pruning import pearson_matrix

    for c in _cases():
        X, _ = frame(c["n"], c["seed"])
        X = X.loc[:, X.nunique() > 1]
        np.testing.assert_allclose(pearson_matrix(X.to_numpy(dtype=float)),
                                   np.asarray(c["pearson"]), rtol=0, atol=1e-12)


@pytest.mark.gpu
def test_prune_two_stage_decisions_match_reference():
    from paper_2305_01886_b200.pruning import Dataset, prune_two_stage

    for c in _cases():
        X, y = frame(c["n"], c["seed"])
        kept, drops = prune_two_stage(Dataset(X=X, y=y))
        assert list(kept.X.columns) == c["kept"]
        assert [[d.dropped, d.kept, d.method] for d in drops] == [r[:3] for r in c["drops"]]
        for d, r in zip(drops, c["drops"]):
            if d.method == "kendall":
                assert repr(d.coefficient) == r[3]
            elif d.method == "pearson":
                assert abs(d.coefficient - float(r[3])) <= 1e-12


@pytest.mark.gpu
def test_kendall_large_n_against_scipy_sample():
    """n = 300k (several radix passes, many inversion levels) vs scipy on the
    same columns."""
    from scipy.stats import kendalltau

    from paper_2305_01886_b200.pruning import kendall_matrix

    rng = np.random.default_rng(9)
    n = 300_000
    a = rng.random(n)
    X = np.stack([a, a + rng.normal(0, 0.3, n), rng.integers(0, 1000, n).astype(float),
                  np.round(a * 50)], axis=1)
    got = kendall_matrix(X)
    for i, j in ((0, 1), (0, 2), (1, 3), (2, 3)):
        assert got[i, j] == kendalltau(X[:, i], X[:, j])[0]


def test_prune_validation_messages():
    from paper_2305_01886_b200.errors import TrainerError
    from paper_2305_01886_b200.pruning import Dataset, prune_correlated

    X, y = frame(50, 0)
    ds = Dataset(X=X, y=y)
    with pytest.raises(TrainerError, match="unknown correlation method 'spearman'"):
        prune_correlated(ds, "spearman")
    with pytest.raises(TrainerError, match=r"correlation threshold must be in \(0, 1\)"):
        prune_correlated(ds, "pearson", 1.0)
    with pytest.raises(TrainerError, match="missing values"):
        Dataset(X=X.where(X > 0.5), y=y)
