"""Feature-CSV I/O (libgkhost gk_featcsv_*, featio.py) against the reference's
features_to_csv / features_from_csv outcomes (tests/golden/featio_cases.json,
made by make_featio_golden.py from features.py:250-272)."""

import json
import math
import struct
from pathlib import Path

import numpy as np
import pytest

from paper_2305_01886_b200 import featio
from paper_2305_01886_b200.pack import FEATURE_ORDER

CASES = json.loads((Path(__file__).parent / "golden" / "featio_cases.json").read_text())


def unhex(s: str) -> float:
    if s == "nan":
        return float("nan")
    if s == "-nan":
        return struct.unpack("<d", struct.pack("<Q", 0xFFF8000000000000))[0]
    return float.fromhex(s)


def hx(v: float) -> str:
    if math.isnan(v):
        return "nan" if math.copysign(1.0, v) > 0 else "-nan"
    return v.hex()


@pytest.mark.parametrize("i", range(len(CASES["write"])))
def test_writer_byte_identical(i):
    c = CASES["write"][i]
    feat = np.array([[unhex(x) for x in r] for r in c["feat"]], np.float64).reshape(-1, 32)
    assert featio.features_csv(c["kernels"], feat, selected=c["selected"]) == c["csv"]


def test_writer_threads_agree():
    rng = np.random.default_rng(5)
    n = 20000
    feat = rng.standard_normal((n, 32)) * 10.0 ** rng.integers(-30, 30, (n, 32))
    feat[rng.random((n, 32)) < 0.01] = np.nan
    names = [f"k{i}[{i % 977}x{64 * (1 + i % 16)}]" if i % 50 else f'odd,"{i}"' for i in range(n)]
    one = featio.features_csv(names, feat, n_threads=1)
    assert featio.features_csv(names, feat, n_threads=7) == one
    cols, kernels, vals = featio.features_from_csv_arrays(one)
    assert cols == ["kernel", *FEATURE_ORDER] and kernels == names
    back = vals[:, 1:]
    assert np.array_equal(np.isnan(back), np.isnan(feat))
    ok = ~np.isnan(feat)
    assert np.array_equal(back[ok].view(np.uint64), feat[ok].view(np.uint64))  # %.17g round trip


@pytest.mark.parametrize("i", range(len(CASES["read"])))
def test_parser_matches_reference(i):
    c = CASES["read"][i]
    if "error" in c:
        with pytest.raises(Exception) as ei:
            featio.features_from_csv(c["csv"])
        assert type(ei.value).__name__ == c["error"] and str(ei.value) == c["message"]
        return
    got = featio.features_from_csv(c["csv"])
    want = c["rows"]
    assert [list(r) for r in got] == [list(r) for r in want]
    assert [{k: (v if isinstance(v, str) else hx(v)) for k, v in r.items()} for r in got] == want


def test_native_parser_takes_writer_output():
    """The texts the writer produces never need the Python path."""
    for c in CASES["write"]:
        assert featio._parse_native(c["csv"]) is not None


def test_library_exports_every_header_symbol():
    import re

    from paper_2305_01886_b200.ptx_native import load_library

    hdr = (Path(__file__).resolve().parents[1] / "include" / "gk_featio.h").read_text()
    names = set(re.findall(r"^\s*(?:int|void \*|void)\s*(gk_\w+)\(", hdr, re.M))
    assert len(names) == 6
    L = load_library()
    assert not [n for n in names if not hasattr(L, n)]


def test_g17_matches_python_format():
    """The writer's %.17g (exact 128-bit fast path + to_chars) == format(v, ".17g")."""
    rng = np.random.default_rng(11)
    bits = rng.integers(0, 2 ** 63, 64000, dtype=np.int64).view(np.float64)   # every exponent
    mags = rng.random(64000) * 10.0 ** rng.integers(-8, 40, 64000)            # the fast path
    p10 = np.array([10.0 ** k for k in range(-10, 40)])
    edges = np.concatenate([p10, np.nextafter(p10, 0), np.nextafter(p10, np.inf),
                            [1e-5, 9.9999999999999991e-06, 1.7e38, 1.6999999999999999e38,
                             99999999999999995.0, 99999999999999999.0, 9999999999999999.5,
                             0.5, 0.25, 1.5, 2.5, 123456789012345678.0, 2 ** 53 + 2.0]])
    vals = np.concatenate([bits, mags, -mags[:1000], edges])
    vals = vals[np.isfinite(vals)]
    vals = vals[: len(vals) // 32 * 32].reshape(-1, 32)
    text = featio.features_csv([""] * len(vals), vals)
    got = [ln.split(",")[1:] for ln in text.splitlines()[1:]]
    want = [[format(v, ".17g") for v in row] for row in vals.tolist()]
    assert got == want


def test_g17_exact_ties_round_half_even():
    """m / 2^q with an 18-digit decimal ending in 5: the 17-digit rounding is
    an exact tie (the 128-bit path must round half to even, as printf)."""
    vals = []
    for q in range(1, 60):
        p5 = 5 ** q
        lo, hi = -(-10 ** 17 // p5), 10 ** 18 // p5
        for m in range(max(1, lo | 1), min(hi, lo + 400), 2):
            if m < 2 ** 53 and 1e-5 <= m / 2 ** q < 1.7e38:
                vals.append(m / 2 ** q)
    vals = np.array(vals + [-v for v in vals])
    vals = vals[: len(vals) // 32 * 32].reshape(-1, 32)
    text = featio.features_csv([""] * len(vals), vals)
    got = [ln.split(",")[1:] for ln in text.splitlines()[1:]]
    assert got == [[format(v, ".17g") for v in row] for row in vals.tolist()]
