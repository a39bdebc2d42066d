"""Feature-CSV I/O: the table ``gpukalc features`` writes
and the trainer reads, formatted / parsed natively (libgkhost,
``include/gk_featio.h``) in parallel.

* ``features_to_csv(rows, selected=False)`` -- reference ``features.py:250-261``
  (same signature, byte-identical text);
* ``features_csv(kernels, feat, selected=False)`` -- the batch form: feature
  rows straight from ``schedule_batch(...)["feat"]`` ([n, 32] in
  FEATURE_ORDER), no per-row FeatureVector objects;
* ``features_from_csv(text)`` -- reference ``features.py:264-272`` (list of
  dicts, "kernel" kept as text);
* ``features_from_csv_arrays(text)`` -> (column names, kernel ids, [n, k]
  float64) without building dicts.

The native parser takes the plain dialect the writer produces; any other text
(blank lines, ragged rows, '_' or spaces inside numbers, ...) runs the Python
parser below, which is the reference's own algorithm (csv.DictReader +
float) and so reproduces its rows or its exception.
"""

from __future__ import annotations

import csv
import ctypes as C
import io

import numpy as np

from .pack import FEATURE_ORDER, SELECTED_FEATURES

_bound = None


class _Sizes(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_cols", C.c_int32), ("kernel_col", C.c_int32),
                ("names_bytes", C.c_int64), ("kernel_bytes", C.c_int64)]


def _lib():
    global _bound
    if _bound is None:
        from .ptx_native import load_library

        L = load_library()
        vp, i64, i32, sz = C.c_void_p, C.c_int64, C.c_int32, C.c_size_t
        L.gk_featcsv_write.restype = C.c_int
        L.gk_featcsv_write.argtypes = [vp, vp, i32, vp, vp, vp, i64, i64, vp, C.c_int, vp, vp]
        L.gk_featcsv_buf_free.argtypes = [vp]
        L.gk_featcsv_parse.restype = vp
        L.gk_featcsv_parse.argtypes = [C.c_char_p, sz, C.c_int, vp, C.c_char_p, sz]
        L.gk_featcsv_sizes_of.argtypes = [vp, vp]
        L.gk_featcsv_copy.restype = C.c_int
        L.gk_featcsv_copy.argtypes = [vp] * 6
        L.gk_featcsv_free.argtypes = [vp]
        _bound = L
    return _bound


def _strings(items) -> tuple:
    enc = [s.encode("utf-8", "surrogatepass") for s in items]
    off = np.zeros(len(enc) + 1, np.int64)
    np.cumsum([len(b) for b in enc], out=off[1:])
    return b"".join(enc), off


def features_csv(kernels, feat, *, selected: bool = False, n_threads: int = 0) -> str:
    """CSV text of [n, 32] FEATURE_ORDER rows (NaN rows print "nan", as the
    reference formats a NaN); kernels: n ids."""
    names = SELECTED_FEATURES if selected else FEATURE_ORDER
    feat = np.ascontiguousarray(feat, dtype=np.float64)
    kernels = list(kernels)
    if feat.ndim != 2 or feat.shape[1] != len(FEATURE_ORDER) or feat.shape[0] != len(kernels):
        raise ValueError(f"feat must be [{len(kernels)}, {len(FEATURE_ORDER)}]")
    cols = np.asarray([FEATURE_ORDER.index(n) for n in names], np.int32)
    nb, noff = _strings(names)
    kb, koff = _strings(kernels)
    L = _lib()
    out, ln = C.c_void_p(), C.c_size_t()
    if L.gk_featcsv_write(nb, noff.ctypes.data, len(names), kb, koff.ctypes.data,
                          feat.ctypes.data, feat.shape[0], feat.shape[1], cols.ctypes.data,
                          n_threads, C.byref(out), C.byref(ln)):
        raise MemoryError("feature CSV buffer")
    try:
        return C.string_at(out.value, ln.value).decode("utf-8", "surrogatepass")
    finally:
        L.gk_featcsv_buf_free(out)


def features_to_csv(rows, *, selected: bool = False) -> str:
    """Reference ``features.py:250-261``: (kernel, FeatureVector) pairs -> CSV."""
    rows = list(rows)
    feat = np.array([vec.as_row() for _, vec in rows], np.float64).reshape(len(rows), 32)
    return features_csv([k for k, _ in rows], feat, selected=selected)


def _parse_native(text: str, n_threads: int = 0):
    raw = text.encode("utf-8", "surrogatepass")
    L = _lib()
    st, why = C.c_int(), C.create_string_buffer(160)
    h = L.gk_featcsv_parse(raw, len(raw), n_threads, C.byref(st), why, len(why))
    if not h:
        raise MemoryError("feature CSV parse")
    try:
        if st.value:
            return None
        s = _Sizes()
        L.gk_featcsv_sizes_of(h, C.byref(s))
        names = C.create_string_buffer(max(1, s.names_bytes))
        noff = np.zeros(s.n_cols + 1, np.int64)
        kern = C.create_string_buffer(max(1, s.kernel_bytes))
        koff = np.zeros(s.n_rows + 1, np.int64)
        vals = np.zeros((s.n_rows, s.n_cols), np.float64)
        L.gk_featcsv_copy(h, names, noff.ctypes.data, kern, koff.ctypes.data, vals.ctypes.data)
        nraw = names.raw
        cols = [nraw[noff[j]:noff[j + 1]].decode("utf-8", "surrogatepass")
                for j in range(s.n_cols)]
        kraw = kern.raw
        kernels = ([kraw[koff[i]:koff[i + 1]].decode("utf-8", "surrogatepass")
                    for i in range(s.n_rows)] if s.kernel_col >= 0 else None)
        return cols, s.kernel_col, kernels, vals
    finally:
        L.gk_featcsv_free(h)


def _parse_python(text: str) -> list:
    """The reference's algorithm (features.py:264-272), for texts the native
    parser declines; raises what the reference raises."""
    rows = []
    for rec in csv.DictReader(io.StringIO(text)):
        rows.append({k: (v if k == "kernel" else float(v)) for k, v in rec.items()})
    return rows


def features_from_csv(text: str) -> list:
    """Reference ``features.py:264-272``: per-row dicts, "kernel" kept as text."""
    got = _parse_native(text)
    if got is None:
        return _parse_python(text)
    cols, kc, kernels, vals = got
    out = []
    for i in range(vals.shape[0]):
        row = dict(zip(cols, vals[i].tolist()))
        if kc >= 0:
            row["kernel"] = kernels[i]
        out.append(row)
    return out


def features_from_csv_arrays(text: str):
    """(column names, kernel ids or None, [n, n_cols] float64; the kernel
    column's entries are 0)."""
    got = _parse_native(text)
    if got is not None:
        cols, kc, kernels, vals = got
        return cols, kernels, vals
    rows = _parse_python(text)
    cols = list(rows[0]) if rows else next(csv.reader(io.StringIO(text)), [])
    vals = np.array([[0.0 if c == "kernel" else r[c] for c in cols] for r in rows],
                    np.float64).reshape(len(rows), len(cols))
    kernels = [r["kernel"] for r in rows] if "kernel" in cols else None
    return cols, kernels, vals


__all__ = ["features_csv", "features_to_csv", "features_from_csv", "features_from_csv_arrays"]
