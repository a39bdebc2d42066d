"""Native PTX front-end: PTX text -> packed corpus in one C++ call.

``pack_ptx(sources)`` is the batched equivalent of

    pack.pack_corpus(ptx.parse_ptx(text, name, loop_counts=loops) for name, text, loops in sources)

(reference ``ptx/parser.py:156-257`` + ``ptx/classify.py:68-104`` +
``ptx/types.py:79-124``), run by ``libgkhost.so`` (``include/gk_ptx.h``) over
all host threads.  The result is byte-identical, including the latency
signature table and the error raised for the first bad kernel (same exception
type and message).  Unknown-opcode warnings are logged through this package's
``ptx`` logger exactly as often as the sequential loop would log them.

This is the host input stage, not the device path; it only removes the
~3 ms/kernel Python parse cost that caps config #5 end to end.
Inputs the C++ tokenizer does not model (non-ASCII text, trip counts outside
int64) go through the Python parser for the whole batch.
"""

from __future__ import annotations

import ctypes as C
import logging
from pathlib import Path

import numpy as np

from . import pack, ptx
from .errors import PtxParseError, ScheduleError
from .ir import CLASS_CODE, RESOURCE_CODE, InstClass

LIB_PATH = Path(__file__).resolve().parent / "libgkhost.so"
EXPORTS = ("gk_ptx_abi_version", "gk_ptx_pack", "gk_ptx_error", "gk_ptx_sizes_of", "gk_ptx_copy",
           "gk_ptx_sig", "gk_ptx_warning", "gk_ptx_free")
_CLASS_NAME = {v: k for k, v in CLASS_CODE.items()}
_lib = None
log = logging.getLogger(ptx.__name__)  # the parser's logger (classify warnings)


class _Sizes(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("n_tok", "n_preds", "n_blk", "n_fpreds", "n_topo",
                                          "n_ker", "n_sig", "n_warn")]


def load_library(path: Path | None = None):
    """ctypes handle of libgkhost (host-only; loads without a GPU)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path or LIB_PATH)
    if not p.exists():
        raise RuntimeError(f"{p} is missing: build it with `python -m paper_2305_01886_b200.build`")
    L = C.CDLL(str(p))
    vp, u64, i32 = C.c_void_p, C.c_uint64, C.c_int
    L.gk_ptx_abi_version.restype = i32
    L.gk_ptx_pack.restype = vp
    L.gk_ptx_pack.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, u64, C.c_char_p, i32, i32]
    L.gk_ptx_error.restype = i32
    L.gk_ptx_error.argtypes = [vp, vp, vp, C.c_char_p, C.c_size_t]
    L.gk_ptx_sizes_of.argtypes = [vp, vp]
    L.gk_ptx_copy.restype = i32
    L.gk_ptx_copy.argtypes = [vp] * 7
    L.gk_ptx_sig.restype = i32
    L.gk_ptx_sig.argtypes = [vp, u64, vp, C.c_char_p, C.c_size_t, vp]
    L.gk_ptx_warning.restype = i32
    L.gk_ptx_warning.argtypes = [vp, u64, vp, C.c_char_p, C.c_size_t]
    L.gk_ptx_free.argtypes = [vp]
    if L.gk_ptx_abi_version() != 1:
        raise RuntimeError("libgkhost ABI version mismatch")
    if path is None:
        _lib = L
    return L


def opcode_table_text(table: ptx.OpcodeTable) -> str:
    """An OpcodeTable in the line format gk_ptx.cpp reads (Table::parse)."""
    def pair(p):
        return f"{CLASS_CODE[p[0].value]} {RESOURCE_CODE[p[1].value]}"

    lines = [f"F {pair(table.fallback)}", "M " + " ".join(sorted(table.memory_roots)),
             f"D {RESOURCE_CODE[table.double_resource.value]}",
             "X " + " ".join(sorted(table.double_exempt)),
             "B " + " ".join(sorted(table.branch_roots))]
    for name, p in table.memory_spaces.items():
        lines.append(f"S {name or '-'} {pair(p)}")
    for root, p in table.roots.items():
        lines.append(f"R {root} {pair(p)}")
    return "\n".join(lines) + "\n"


def _python_path(items, table, strict):
    return pack.pack_corpus(ptx.parse_ptx(t, n, loop_counts=l, opcode_table=table,
                                          strict_opcodes=strict) for n, t, l in items)


def pack_ptx(sources, *, opcode_table: ptx.OpcodeTable | None = None,
             strict_opcodes: bool = False, threads: int = 0) -> pack.Corpus:
    """Parse + pack kernels given as (kernel_name, ptx_text, loop_counts | None)."""
    items = [(n, t, dict(l or {})) for n, t, l in sources]
    table = opcode_table or ptx.default_table()
    for _, t, l in items:
        if not t.isascii() or any(type(v) is not int or not -(1 << 63) <= v < (1 << 63)
                                  for v in l.values()):
            return _python_path(items, table, strict_opcodes)
    L = load_library()
    # one blob; items naming the same text object share its bytes
    chunks, where, at = [], {}, 0
    tb = np.empty(len(items), np.int64)
    te = np.empty(len(items), np.int64)
    for i, (_, t, _) in enumerate(items):
        k = id(t)
        if k not in where:
            b = t.encode("ascii")
            where[k] = (at, at + len(b))
            chunks.append(b)
            at += len(b)
        tb[i], te[i] = where[k]
    blob = b"".join(chunks)
    nb = [n.encode("utf-8") for n, _, _ in items]
    names = b"".join(nb)
    name_off = np.zeros(len(items) + 1, np.int64)
    name_off[1:] = np.cumsum([len(x) for x in nb])
    lab, cnt, loop_off = [], [], np.zeros(len(items) + 1, np.int64)
    for i, (_, _, l) in enumerate(items):
        for k, v in l.items():
            lab.append(str(k).encode("utf-8"))
            cnt.append(v)
        loop_off[i + 1] = len(lab)
    labels = b"".join(lab)
    label_off = np.zeros(len(lab) + 1, np.int64)
    label_off[1:] = np.cumsum([len(x) for x in lab]) if lab else []
    counts = np.asarray(cnt, np.int64) if cnt else np.zeros(1, np.int64)

    def p(a):
        return a.ctypes.data

    h = L.gk_ptx_pack(blob, p(tb), p(te), names, p(name_off), p(loop_off), labels or b"\0",
                      p(label_off), p(counts), len(items), opcode_table_text(table).encode(),
                      int(bool(strict_opcodes)), int(threads))
    if not h:
        raise RuntimeError("gk_ptx_pack: allocation failure or malformed opcode table")
    try:
        return _collect(L, h, items, table)
    finally:
        L.gk_ptx_free(h)


def _collect(L, h, items, table):
    sz = _Sizes()
    L.gk_ptx_sizes_of(h, C.byref(sz))
    buf = C.create_string_buffer(4096)
    kk = C.c_uint64()
    for w in range(sz.n_warn):
        L.gk_ptx_warning(h, w, C.byref(kk), buf, len(buf))
        log.warning("unknown opcode '%s': classified as %s", buf.value.decode(),
                    table.fallback[0].value)
    line = C.c_int64()
    kind = L.gk_ptx_error(h, C.byref(kk), C.byref(line), buf, len(buf))
    if kind:
        msg = buf.value.decode()
        if kind == 1:
            raise PtxParseError(msg, line.value if line.value >= 0 else None)
        if kind == 2:
            raise ScheduleError(msg)
        if kind == 3:
            raise ValueError(msg)
        return _python_path(items, table, False)
    tok = np.zeros(sz.n_tok + 1, pack.TOKEN_DT)
    preds = np.zeros(sz.n_preds, np.uint16)
    blk = np.zeros(sz.n_blk, pack.BLOCK_DT)
    fpreds = np.zeros(sz.n_fpreds, np.uint32)
    topo = np.zeros(sz.n_topo, np.uint32)
    ker = np.zeros(sz.n_ker, pack.KERNEL_DT)
    if L.gk_ptx_copy(h, tok.ctypes.data, preds.ctypes.data, blk.ctypes.data, fpreds.ctypes.data,
                     topo.ctypes.data, ker.ctypes.data):
        raise RuntimeError("gk_ptx_copy failed")
    sigs = []
    cls, knd = C.c_int(), C.c_int()
    for i in range(sz.n_sig):
        L.gk_ptx_sig(h, i, C.byref(cls), buf, len(buf), C.byref(knd))
        klass = _CLASS_NAME[cls.value]
        kind = chr(knd.value) if knd.value else None
        sigs.append((klass, buf.value.decode(), kind))
    return pack.Corpus(tok=tok, preds=preds, blk=blk, fpreds=fpreds, topo=topo, ker=ker,
                       sigs=sigs, names=[n for n, _, _ in items])


__all__ = ["pack_ptx", "opcode_table_text", "load_library", "InstClass"]
