"""Loaders for tests/golden/ (fixtures produced by running the reference;
see tests/golden/make_golden.py).  Inputs are regenerated deterministically
with this package's corpus generator + parser; the packed corpus digest is
checked against the digest of the reference-parsed corpus."""

from __future__ import annotations

import functools
import hashlib
import json
from pathlib import Path

import numpy as np

from paper_2305_01886_b200 import corpus as CG
from paper_2305_01886_b200 import pack, ptx
from paper_2305_01886_b200.profiles import profile_from_dict, resolve_profile

G = Path(__file__).resolve().parent / "golden"
SETS = ("c1", "c2", "rnd", "c5")


def corpus_digest(c) -> str:
    """Digest of the packed corpus's semantic fields (independent of record padding
    and of derived fields), so a layout change does not invalidate the goldens."""
    h = hashlib.sha256()
    t = c.tok
    for f in ("res", "cls", "sig", "pred0"):
        h.update(np.ascontiguousarray(t[f]).astype(np.int64).tobytes())
    b = c.blk
    for f in ("mult", "tok0", "n", "fpred0", "n_fpred", "n_glob", "res_cnt", "is_exit"):
        h.update(np.ascontiguousarray(b[f]).astype(np.int64).tobytes())
    k = c.ker
    for f in ("blk0", "n_blk", "topo0", "max_n", "tok0", "n_tok"):
        h.update(np.ascontiguousarray(k[f]).astype(np.int64).tobytes())
    for a in (c.preds, c.fpreds, c.topo):
        h.update(np.ascontiguousarray(a).astype(np.int64).tobytes())
    h.update(json.dumps([list(s) for s in c.sigs]).encode())
    return h.hexdigest()


@functools.lru_cache(maxsize=None)
def graphs(n_kernels: int, seed: int):
    return tuple(ptx.parse_ptx(t, n, loop_counts=l) for n, t, l in CG.synth_corpus(n_kernels, seed))


@functools.lru_cache(maxsize=None)
def load_set(name: str):
    d = dict(np.load(G / f"sched_{name}.npz"))
    gs = graphs(int(d["n_kernels"]), int(d["seed"]))
    c = pack.pack_corpus(gs)
    profs = [resolve_profile(str(a)) for a in d["archs"]]
    cfgs = [tuple(int(v) for v in row) for row in d["configs"]]
    return d, gs, c, profs, cfgs


@functools.lru_cache(maxsize=None)
def fixtures() -> dict:
    return json.loads((G / "ref_fixtures.json").read_text())


def fixture_profile():
    return profile_from_dict(fixtures()["fixture_profile"])


def bits_equal(a, b) -> bool:
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def mismatch_report(a, b, names=None, limit=5) -> str:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    bad = np.argwhere(a.view(np.uint64) != b.view(np.uint64))
    lines = [f"{len(bad)} mismatching values"]
    for idx in bad[:limit]:
        idx = tuple(idx)
        col = names[idx[-1]] if names is not None and len(idx) > 1 else ""
        lines.append(f"  at {idx} {col}: got {a[idx]!r} want {b[idx]!r}")
    return "\n".join(lines)
