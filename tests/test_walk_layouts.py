"""Compact ensemble walk layouts (gk_node8 / gk_block2, include/gk.h): the
f32-bucket decision with an exact fp64 tie test must equal the reference's
`x <= threshold` (power.py:156-168) for every input, so power stays
bit-identical in every layout.

CPU: the decision rule and the encodings (host logic: pure-numpy walks of the
compact forms must reproduce the 16-byte node walk).
GPU: K4 and the fused sweep with tie-heavy ensembles (thresholds placed on and
one ulp around the rows' own feature values) against the CPU oracle, in each
layout."""

from __future__ import annotations

import numpy as np
import pytest

from goldens import bits_equal, load_set
from paper_2305_01886_b200 import pack
from paper_2305_01886_b200.ensemble import (BLOCK2_MAX_FEAT, GK_LEAF, NODE8_MAX_FEAT, blocked,
                                            blocked3, f32_round_down, key16, nodes8,
                                            random_forest_flat)

LAYOUTS = ("nodes", "nodes8", "blocks", "blocks3")


def _adversarial_pairs(rng, n=200_000):
    base = np.concatenate([rng.standard_normal(n // 4) * 10.0 ** rng.integers(-40, 40, n // 4),
                           rng.random(n // 4),
                           rng.random(n // 4).astype(np.float32).astype(np.float64),
                           np.array([0.0, -0.0, 1.0, -1.0, 3.4028234663852886e38, 1e39, -1e39,
                                     1e-45, 1.4e-45, 5e-324, -5e-324, np.inf, -np.inf, np.nan])])
    x = np.repeat(base, 5)
    T = x.copy()
    k = np.arange(len(x)) % 5
    T[k == 1] = np.nextafter(x[k == 1], np.inf)
    T[k == 2] = np.nextafter(x[k == 2], -np.inf)
    T[k == 3] = f32_round_down(x[k == 3]).astype(np.float64)
    T[k == 4] = rng.permutation(x[k == 4])
    return x, T


def test_decision_rule_equals_fp64_compare():
    rng = np.random.default_rng(0)
    x, T = _adversarial_pairs(rng)
    with np.errstate(invalid="ignore"):
        a, t = f32_round_down(x), f32_round_down(T)
        le = (a < t) | ((a == t) & (x <= T))
        want = x <= T
    assert np.array_equal(le, want)
    tie = (a == t)
    assert tie.sum() > 1000  # the exact path is exercised


def test_key16_decision_rule_equals_fp64_compare():
    """gk_block3: 16-bit order keys of round-down-f32 (zeros canonical, NaN
    top) with the exact test on equal keys == `x <= thr` for every pair."""
    rng = np.random.default_rng(5)
    x, T = _adversarial_pairs(rng)
    ok = ~np.isnan(T)              # thresholds are never NaN
    x, T = x[ok], T[ok]
    a, t = key16(x).astype(np.int64), key16(T).astype(np.int64)
    with np.errstate(invalid="ignore"):
        le = (a < t) | ((a == t) & (x <= T))
        want = x <= T
    assert np.array_equal(le, want)
    assert (a == t).sum() > 1000 and ((x == 0) & (T == 0)).sum() > 0


def test_f32_round_down_is_the_largest_float_below():
    rng = np.random.default_rng(1)
    x, _ = _adversarial_pairs(rng, 40_000)
    f = f32_round_down(x)
    fin = np.isfinite(x)
    with np.errstate(invalid="ignore", over="ignore"):
        assert np.all(f[fin].astype(np.float64) <= x[fin])
        nxt = np.nextafter(f[fin], np.float32(np.inf)).astype(np.float64)
    assert np.all((nxt > x[fin]) | (f[fin] == np.float32(3.4028235e38)))


def _walk_blocks(bl, flat, X):
    """numpy emulation of walk_ensemble_b2 (device) for a few rows."""
    out = np.full(len(X), float(flat.base_score))
    for i, x in enumerate(X):
        xf = f32_round_down(x)
        for t in range(flat.n_trees):
            ref = int(bl.root[t])
            while not ref & GK_LEAF:
                b = bl.blocks[ref]
                f = [(int(b["f"]) >> (8 * k)) & 0xFF for k in range(3)]
                tt = b["t"].view(np.float32)

                def le(s):
                    a = xf[f[s]]
                    if a == tt[s]:
                        return bool(x[f[s]] <= bl.thr64[3 * ref + s])
                    return bool(a < tt[s])

                c0 = le(0)
                c1 = le(1 if c0 else 2)
                ref = int(b["e"][(0 if c0 else 2) + (0 if c1 else 1)])
            out[i] = out[i] + bl.leaf_val[ref & ~GK_LEAF]
    return out


def _walk_nodes8(n8, flat, X):
    out = np.full(len(X), float(flat.base_score))
    for i, x in enumerate(X):
        xf = np.append(f32_round_down(x), np.float32(np.inf))   # index -1 = +inf slot
        for o in flat.tree_off:
            k = 0
            for _ in range(int(flat.max_depth)):
                t, meta = n8["t"][o + k].view(np.float32), int(n8["meta"][o + k])
                f = meta >> 24
                f = -1 if f == 0xFF else f
                a = xf[f]
                le = bool(x[f] <= flat.nodes["v"][o + k]) if a == t else bool(a < t)
                r = meta & 0xFFFFFF
                k = r - 1 if le else r
            out[i] = out[i] + flat.nodes["v"][o + k]
    return out


def _walk_nodes(flat, X):
    out = np.full(len(X), float(flat.base_score))
    for i, x in enumerate(X):
        for o in flat.tree_off:
            k = 0
            while flat.nodes["feature"][o + k] >= 0:
                nd = flat.nodes[o + k]
                k = int(nd["left"]) + (0 if x[nd["feature"]] <= nd["v"] else 1)
            out[i] = out[i] + flat.nodes["v"][o + k]
    return out


def _walk_blocks3(b3, flat, X):
    """numpy emulation of walk_ensemble_b3 (device) for a few rows."""
    from paper_2305_01886_b200.ensemble import B3_TERMINAL, key16
    out = np.full(len(X), float(flat.base_score))
    for i, x in enumerate(X):
        kx = key16(x).astype(np.int64)

        def le(key, f, ref, j):  # x[f] <= threshold j of block ref
            if kx[f] == key:
                return bool(x[f] <= b3.thr64[7 * ref + j])
            return bool(kx[f] < key)

        for t in range(flat.n_trees):
            ref = int(b3.root[t])
            val = None
            while val is None:
                if ref & GK_LEAF:
                    val = b3.leaf_val[ref & ~GK_LEAF]
                    break
                w = [int(v) for v in b3.blocks[ref]["w"]]
                if (w[5] >> 16) & 0xFF == B3_TERMINAL:
                    go_l = le(w[0] & 0xFFFF, (w[3] >> 16) & 0xFF, ref, 0)
                    lo, hi = (w[1], w[2]) if go_l else (w[6], w[7])
                    val = np.array([lo | (hi << 32)], np.uint64).view(np.float64)[0]
                    break
                keys = [w[0] & 0xFFFF, w[0] >> 16, w[1] & 0xFFFF, w[1] >> 16, w[2] & 0xFFFF,
                        w[2] >> 16, w[3] & 0xFFFF]
                feats = [(w[3] >> 16) & 0xFF, w[3] >> 24, w[4] & 0xFF, (w[4] >> 8) & 0xFF,
                         (w[4] >> 16) & 0xFF, w[4] >> 24, w[5] & 0xFF]
                k, s = 0, 0
                for _ in range(3):
                    b = 0 if le(keys[k], feats[k], ref, k) else 1
                    s = 2 * s + b
                    k = 2 * k + 1 + b
                mask = (w[5] >> 8) & 0xFF
                below = (1 << s) - 1
                if mask >> s & 1:
                    ref = GK_LEAF | (w[7] + bin(mask & below).count("1"))
                else:
                    ref = w[6] + bin(~mask & below & 0xFF).count("1")
            out[i] = out[i] + val
    return out


def test_block_encoding_walks_like_the_nodes():
    rng = np.random.default_rng(3)
    nf = 6
    flat = random_forest_flat(7, 7, [f"f{i}" for i in range(nf)], np.zeros(nf), np.ones(nf),
                              seed=3, split_p=0.7)
    X = rng.random((60, nf))
    X[:20] = flat.nodes["v"][rng.integers(0, len(flat.nodes), (20, nf))]  # exact ties
    bl = blocked(flat)
    want = _walk_nodes(flat, X)
    assert bits_equal(_walk_blocks(bl, flat, X), want)
    assert bits_equal(_walk_nodes8(nodes8(flat), flat, X), want)
    assert bits_equal(_walk_blocks3(blocked3(flat), flat, X), want)
    wide = random_forest_flat(2, 3, [f"f{i}" for i in range(BLOCK2_MAX_FEAT + 1)],
                              np.zeros(BLOCK2_MAX_FEAT + 1), np.ones(BLOCK2_MAX_FEAT + 1), seed=1)
    assert blocked(wide) is None and nodes8(wide) is None
    mid = random_forest_flat(2, 3, [f"f{i}" for i in range(NODE8_MAX_FEAT + 1)],
                             np.zeros(NODE8_MAX_FEAT + 1), np.ones(NODE8_MAX_FEAT + 1), seed=1)
    assert nodes8(mid) is None and blocked(mid) is not None


@pytest.mark.parametrize("n_trees,depth,split_p", [(5, 10, 0.9), (9, 4, 0.5), (3, 16, 0.95),
                                                   (4, 1, 1.0), (3, 0, 1.0)])
def test_block3_encoding_walks_like_the_nodes(n_trees, depth, split_p):
    """terminal blocks, padded subtrees, single-leaf trees, NaN / +-inf / -0.0
    rows and exact threshold ties"""
    rng = np.random.default_rng(depth)
    nf = 6
    flat = random_forest_flat(n_trees, depth, [f"f{i}" for i in range(nf)], np.zeros(nf),
                              np.ones(nf), seed=depth, split_p=split_p)
    X = rng.random((40, nf))
    X[:15] = flat.nodes["v"][rng.integers(0, len(flat.nodes), (15, nf))]
    X[15:18] = np.nan
    X[18, 0], X[19, 1], X[20, 2] = -0.0, np.inf, -np.inf
    nd = flat.nodes.copy()       # a NaN threshold: x <= NaN is always false
    sp = np.flatnonzero(nd["feature"] >= 0)
    if len(sp):
        nd["v"][sp[len(sp) // 2]] = np.nan
    flat.nodes = nd
    assert bits_equal(_walk_blocks3(blocked3(flat), flat, X), _walk_nodes(flat, X))


def test_fixture_ensembles_block_like_the_nodes():
    from goldens import fixtures
    from paper_2305_01886_b200.ensemble import flatten, load_ensemble

    fx = fixtures()["ensembles"]
    for name, X in (("stump", [[256.0], [513.0], [512.0], [768.0]]),):
        flat = flatten(load_ensemble(fx[name]))
        lo, hi = flat.scale_lo, flat.scale_hi
        Xs = np.where(hi > lo, (np.asarray(X) - lo) / (hi - lo), 0.0)
        bl = blocked(flat)
        assert bits_equal(_walk_blocks(bl, flat, Xs), _walk_nodes(flat, Xs))
    # one-leaf trees are leaf roots
    one = random_forest_flat(3, 0, ["a"], np.zeros(1), np.ones(1), seed=0)
    bl = blocked(one)
    assert np.all(bl.root & GK_LEAF)
    assert bits_equal(_walk_blocks(bl, one, np.zeros((2, 1))), _walk_nodes(one, np.zeros((2, 1))))


# ------------------------------------------------------------------ GPU


def _tie_heavy(flat, Xs, rng):
    """Replace split thresholds by the rows' own scaled feature values, one
    fp64 ulp around them, or their f32 round-down -- every decision is a tie
    candidate for the compact walk."""
    nd = flat.nodes.copy()
    sp = np.flatnonzero(nd["feature"] >= 0)
    rows = rng.integers(0, len(Xs), len(sp))
    v = Xs[rows, nd["feature"][sp]]
    kind = rng.integers(0, 4, len(sp))
    v = np.where(kind == 1, np.nextafter(v, np.inf), v)
    v = np.where(kind == 2, np.nextafter(v, -np.inf), v)
    v = np.where(kind == 3, f32_round_down(v).astype(np.float64), v)
    nd["v"][sp] = v
    flat.nodes = nd
    return flat


def _scaled(X, lo, hi):
    with np.errstate(invalid="ignore", divide="ignore"):
        return np.where(hi > lo, (X - lo) / (hi - lo), 0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("nf", [15, 64])
def test_k4_compact_layouts_tie_heavy_match_oracle(nf):
    import torch

    import oracle as O
    from paper_2305_01886_b200 import runtime as rt

    rng = np.random.default_rng(nf)
    n = 3000
    X = rng.random((n, nf)) * 3.0 - 1.0
    X[:50] = np.round(X[:50], 1)
    X[50, 0], X[51, 1], X[52, 2], X[53, 3] = np.nan, np.inf, -np.inf, 1e300
    X[54, :] = 5e-324
    lo, hi = np.full(nf, -1.0), np.full(nf, 2.0)
    hi[nf - 1] = lo[nf - 1]  # a constant column scales to 0.0
    flat = random_forest_flat(21, 9, [f"f{i}" for i in range(nf)], lo, hi, seed=nf)
    flat = _tie_heavy(flat, _scaled(X, lo, hi), rng)
    Xd = torch.tensor(X, device="cuda")
    want, _ = O.rf_predict(flat, X)
    for layout in LAYOUTS:
        de = rt.DeviceEnsemble.upload(flat, layout=layout)
        assert de.layout == layout
        p, _ = rt.rf_predict(de, Xd)
        assert bits_equal(p.cpu().numpy(), want), layout


@pytest.mark.gpu
def test_fused_sweep_compact_layouts_tie_heavy_match_oracle():
    import oracle as O
    from paper_2305_01886_b200 import runtime as rt

    d, gs, c, profs, cfgs = load_set("c5")
    sel = pack.manifest_indices(pack.SELECTED_FEATURES)
    F = np.nan_to_num(d["feat"][:, sel])
    ok = d["status"] == 0
    lo, hi = F[ok].min(0), F[ok].max(0)
    rng = np.random.default_rng(5)
    flats = [_tie_heavy(random_forest_flat(19, 9, pack.SELECTED_FEATURES, lo, hi, seed=a),
                        _scaled(F[ok], lo, hi), rng) for a in range(len(profs))]
    dc = rt.DeviceCorpus.upload(c)
    dg = rt.DeviceGrid.build(dc, profs, cfgs)
    n_cfg, n_arch = len(cfgs), len(profs)
    arch_of = (np.arange(len(d["status"])) // n_cfg) % n_arch
    want = {}
    for a in range(n_arch):
        m = ok & (arch_of == a)
        want[a] = O.rf_predict(flats[a], d["feat"][m][:, sel], time_us=d["sf"][m, 7])
    import os

    for layout in LAYOUTS:
        sw = rt.Sweep(dc, dg, [rt.DeviceEnsemble.upload(f, layout=layout) for f in flats], sel)
        os.environ["GK_FUSED_COMPACT"] = "1"  # the fused walk uses the compact layout
        try:
            status, t_us, power, energy = [x.cpu().numpy() for x in sw.run()]
        finally:
            del os.environ["GK_FUSED_COMPACT"]
        assert np.array_equal(status, d["status"])
        for a in range(n_arch):
            m = ok & (arch_of == a)
            assert bits_equal(power[m], want[a][0]), (layout, a)
            assert bits_equal(energy[m], want[a][1]), (layout, a)


@pytest.mark.gpu
@pytest.mark.parametrize("layout", ["blocks", "blocks3"])
def test_k4_persistent_rounds_match_oracle(layout):
    """Tables spanning several waves of resident CTAs take the grid-synchronised
    persistent path (k4_rf_predict_rounds); same bits as the oracle and as the
    one-tile-per-CTA launch."""
    import os

    import torch

    import oracle as O
    from paper_2305_01886_b200 import runtime as rt

    nf, n = 15, 700_000
    rng = np.random.default_rng(11)
    X = rng.random((n, nf))
    flat = random_forest_flat(30, 10, [f"f{i}" for i in range(nf)], np.zeros(nf), np.ones(nf), seed=4)
    flat = _tie_heavy(flat, X[:5000], rng)
    Xd = torch.tensor(X, device="cuda")
    de = rt.DeviceEnsemble.upload(flat, layout=layout)
    assert de.layout == layout
    p_rounds, _ = rt.rf_predict(de, Xd)
    os.environ["GK_RF_ROUNDS"] = "0"
    try:
        p_tiles, _ = rt.rf_predict(de, Xd)
    finally:
        del os.environ["GK_RF_ROUNDS"]
    want, _ = O.rf_predict(flat, X)
    assert bits_equal(p_rounds.cpu().numpy(), want)
    assert bits_equal(p_tiles.cpu().numpy(), want)
