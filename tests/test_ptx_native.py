"""Native PTX front-end (libgkhost, include/gk_ptx.h) vs the reference parser.

CPU tests: the tokenizer is host code.  Parity is byte-identity of the packed
corpus with pack_corpus(parse_ptx(...)), the digests of the reference-parsed
corpora behind the schedule goldens, and the reference's exception type and
message on edge cases + seeded random mutations (tests/golden/ptx_cases.json,
made by tests/golden/make_ptx_golden.py from /root/reference).
"""

from __future__ import annotations

import ctypes
import json
import logging
import re

import numpy as np
import pytest

from goldens import G, SETS, corpus_digest, fixtures
from paper_2305_01886_b200 import corpus as CG
from paper_2305_01886_b200 import pack, ptx
from paper_2305_01886_b200 import ptx_native as PN
from paper_2305_01886_b200.errors import PtxParseError, ScheduleError

ERRORS = {"PtxParseError": PtxParseError, "ScheduleError": ScheduleError, "ValueError": ValueError}
FIELDS = ("tok", "preds", "blk", "fpreds", "topo", "ker")


def same_corpus(a, b) -> bool:
    return (all(getattr(a, f).tobytes() == getattr(b, f).tobytes() for f in FIELDS)
            and a.sigs == b.sigs and a.names == b.names)


def python_pack(items, **kw):
    return pack.pack_corpus(ptx.parse_ptx(t, n, loop_counts=l, **kw) for n, t, l in items)


def test_library_exports_every_declared_symbol():
    L = PN.load_library()
    hdr = (G.parents[1] / "include" / "gk_ptx.h").read_text()
    declared = set(re.findall(r"\b(gk_ptx_\w+)\s*\(", hdr))
    assert declared == set(PN.EXPORTS)
    for name in declared:
        assert isinstance(getattr(L, name), ctypes._CFuncPtr)


@pytest.mark.parametrize("n,seed", [(1, 0), (50, 3), (300, 11)])
def test_byte_identical_to_python_parser(n, seed):
    items = CG.synth_corpus(n, seed)
    assert same_corpus(PN.pack_ptx(items), python_pack(items))


@pytest.mark.parametrize("threads", [1, 3])
def test_thread_count_does_not_change_output(threads):
    items = CG.synth_corpus(120, 5)
    assert same_corpus(PN.pack_ptx(items, threads=threads), PN.pack_ptx(items, threads=8))


@pytest.mark.parametrize("name", SETS)
def test_digest_equals_reference_parsed_corpus(name):
    d = np.load(G / f"sched_{name}.npz")
    c = PN.pack_ptx(CG.synth_corpus(int(d["n_kernels"]), int(d["seed"])))
    assert corpus_digest(c) == str(d["corpus_sha256"])


def test_reference_fixture_kernels():
    fx = fixtures()["ptx"]
    items = [("pair_load_add", fx["worked_example"], None), ("vecadd", fx["vecadd"], None),
             ("nn_euclid", fx["nn_euclid"], None)]
    assert same_corpus(PN.pack_ptx(items), python_pack(items))


def test_shared_text_multiple_kernels():
    text = "".join(t for _, t, _ in CG.synth_corpus(6, 2))
    items = [(n, text, l) for n, _, l in CG.synth_corpus(6, 2)][::-1]
    assert same_corpus(PN.pack_ptx(items), python_pack(items))


def _cases():
    return json.loads((G / "ptx_cases.json").read_text())["cases"]


def _outcome(fn):
    try:
        c = fn()
    except (PtxParseError, ScheduleError, ValueError) as exc:
        return {"error": type(exc).__name__, "message": str(exc)}
    return {"digest": corpus_digest(c), "n_tok": int(c.n_tok), "n_blk": int(len(c.blk))}


def test_reference_outcomes_edge_cases_and_mutations():
    cases = _cases()
    assert len(cases) > 250
    bad = []
    for c in cases:
        item = [(c["kernel"], c["text"], c["loops"])]
        got = _outcome(lambda: PN.pack_ptx(item, strict_opcodes=c["strict"]))
        if got != c["ref"]:
            bad.append((c["name"], got, c["ref"]))
    assert not bad, bad[:3]


def test_python_parser_matches_reference_outcomes():
    """Pins this package's own parse_ptx on the same cases (it is the oracle of
    the byte-identity tests above)."""
    bad = []
    for c in _cases():
        item = [(c["kernel"], c["text"], c["loops"])]
        got = _outcome(lambda: python_pack(item, strict_opcodes=c["strict"]))
        if got != c["ref"]:
            bad.append((c["name"], got, c["ref"]))
    assert not bad, bad[:3]


def test_first_failing_kernel_is_reported():
    items = CG.synth_corpus(40, 9)
    bad1 = (items[7][0], items[7][1].replace(";", "", 3), items[7][2])
    bad2 = (items[30][0], "no kernel here", items[30][2])
    items = items[:7] + [bad1] + items[8:30] + [bad2] + items[31:]
    with pytest.raises(PtxParseError) as a:
        PN.pack_ptx(items)
    with pytest.raises(PtxParseError) as b:
        python_pack(items)
    assert str(a.value) == str(b.value) and a.value.line == b.value.line


def test_unknown_opcode_warnings_logged_like_the_parser(caplog):
    text = ".visible .entry k()\n{\n\tfrob.b32 %r1, %r2;\n\tzap %r1;\n\tfrob %r3;\n\tret;\n}\n"
    items = [("k", text, None)] * 2
    with caplog.at_level(logging.WARNING, logger=ptx.__name__):
        PN.pack_ptx(items)
    native = [r.getMessage() for r in caplog.records]
    caplog.clear()
    with caplog.at_level(logging.WARNING, logger=ptx.__name__):
        python_pack(items)
    assert native == [r.getMessage() for r in caplog.records] and len(native) == 6


def test_custom_opcode_table_round_trips():
    doc = ptx._default_doc()
    doc["roots"]["frob"] = {"class": "Compute", "resource": "SFU"}
    doc["branch_roots"] = ["bra", "brx"]
    doc["roots"]["brx"] = {"class": "Miscellaneous", "resource": "WS"}
    t = ptx.OpcodeTable(doc)
    text = (".visible .entry k()\n{\n\tfrob.f64 %fd1, %fd2;\n\t@%p1 brx L;\n\tadd.f64 %fd3, %fd1, 1;\n"
            "L:\n\tret;\n}\n")
    items = [("k", text, None)]
    assert same_corpus(PN.pack_ptx(items, opcode_table=t), python_pack(items, opcode_table=t))


def test_non_ascii_goes_through_the_python_parser():
    text = ".visible .entry k()\n{\n\t// caf\u00e9\n\tadd.s32 %r1, %r2, 1;\n\tret;\n}\n"
    items = [("k", text, None)]
    assert same_corpus(PN.pack_ptx(items), python_pack(items))
