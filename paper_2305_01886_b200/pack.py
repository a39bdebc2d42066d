"""Host packing: KernelGraphs / ArchProfiles / configs -> the flat records of
``include/gk.h``.

Everything config-independent about a kernel is resolved here exactly once
(SURVEY §8(a) a5, a9): the DFG predecessor lists, the forward-CFG predecessor
lists, Kahn topological order (reference ``ptx/types.py:87-107``), exit blocks
(``types.py:79-82``) and loop multipliers (``types.py:109-124``).  Per
instruction only a latency *signature* (class, root, type kind) is kept; each
arch resolves signatures to a latency with the reference's lookup chain
(``profiles.py:185-228``) into a small ``[n_arch][n_sig]`` table that the
device stages in shared memory.

Works on graphs from this package's parser or the reference's (duck-typed:
``klass``/``resource`` may be either package's enums).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ProfileError, ScheduleError
from .ir import CLASS_CODE, RESOURCE_CODE, InstClass
from .profiles import ArchProfile, latency_kind, resolve_signature

GK_MAX_BP = 8
NRES = 5

TOKEN_DT = np.dtype({"names": ["res", "cls", "sig", "pred0", "lst_row", "lst_len"],
                     "formats": ["u1", "u1", "<u2", "<u4", "<u2", "<u2"],
                     "offsets": [0, 1, 2, 4, 8, 10], "itemsize": 16})
BLOCK_DT = np.dtype({"names": ["mult", "tok0", "n", "fpred0", "n_fpred", "n_glob", "res_cnt",
                               "is_exit"],
                     "formats": ["<i8", "<u4", "<u4", "<u4", "<u2", "<u2", ("<u2", (5,)), "u1"],
                     "offsets": [0, 8, 12, 16, 20, 22, 24, 34], "itemsize": 40})
KERNEL_DT = np.dtype({"names": ["blk0", "n_blk", "topo0", "max_n", "tok0", "n_tok"],
                      "formats": ["<u4"] * 6, "offsets": [0, 4, 8, 12, 16, 20], "itemsize": 32})
CONFIG_DT = np.dtype([("n_blocks", "<i4"), ("tpb", "<i4"), ("regs", "<i4"), ("shmem", "<i4")])
KSTAT_DT = np.dtype({"names": ["cnt", "branches", "loads", "stores"],
                     "formats": [("<i8", (4,)), "<i8", "<i8", "<i8"],
                     "offsets": [0, 32, 40, 48], "itemsize": 64})
_ARCH_FIELDS = [
    ("units", ("<i8", (5,))), ("gap", ("<f8", (5,))), ("pipeline", "<f8"),
    ("nSM", "<i8"), ("L2_sz", "<i8"), ("nTh_sm_max", "<i8"), ("reg_b_max", "<i8"),
    ("shm_b_max", "<i8"), ("nB_max", "<i8"), ("wSM_max", "<i8"), ("Sz_w", "<i8"),
    ("access_sz", "<i8"), ("access_gm_sz", "<i8"), ("access_shm_sz", "<i8"), ("nWS", "<i8"),
    ("nDU", "<i8"), ("nu_gpu", "<f8"), ("tpg_a", "<f8"), ("tpg_b", "<f8"), ("tpg_c", "<f8"),
    ("tps_a", "<f8"), ("tps_b", "<f8"), ("tps_c", "<f8"), ("tp_floor", "<f8"),
    ("ov_slope", "<f8"), ("ov_icpt", "<f8"), ("n_bp", "<i4"), ("pad_", "<i4"),
    ("bp", ("<f8", (GK_MAX_BP,))), ("seg_slope", ("<f8", (GK_MAX_BP + 1,))),
    ("seg_icpt", ("<f8", (GK_MAX_BP + 1,))),
]
ARCH_DT = np.dtype(_ARCH_FIELDS, align=True)
assert TOKEN_DT.itemsize == 16 and BLOCK_DT.itemsize == 40 and KERNEL_DT.itemsize == 32
assert ARCH_DT.itemsize == 488 and KSTAT_DT.itemsize == 64

_FLAG_BRANCH, _FLAG_GLOAD, _FLAG_GSTORE = 0x04, 0x08, 0x10


def _code(x, table):
    return table[getattr(x, "value", x)]


@dataclass
class Corpus:
    """A packed kernel corpus (host numpy; see ``to_device`` in :mod:`runtime`)."""

    tok: np.ndarray      # TOKEN_DT [n_tok + 1]
    preds: np.ndarray    # u16
    blk: np.ndarray      # BLOCK_DT
    fpreds: np.ndarray   # u32
    topo: np.ndarray     # u32
    ker: np.ndarray      # KERNEL_DT
    sigs: list           # [(class value, root, kind)] per signature id
    names: list          # kernel names

    @property
    def n_ker(self) -> int:
        return len(self.ker)

    @property
    def n_tok(self) -> int:
        return len(self.tok) - 1

    @property
    def max_n(self) -> int:
        return max(int(self.ker["max_n"].max()) if len(self.ker) else 1, 1)

    @property
    def max_blk(self) -> int:
        return max(int(self.ker["n_blk"].max()) if len(self.ker) else 1, 1)

    def check(self) -> "Corpus":
        """Guard the C layout (numpy drops struct padding on some operations)."""
        for name, dt in (("tok", TOKEN_DT), ("blk", BLOCK_DT), ("ker", KERNEL_DT)):
            a = getattr(self, name)
            if a.dtype != dt or not a.flags["C_CONTIGUOUS"]:
                raise ValueError(f"corpus.{name} must be a contiguous {dt.itemsize}-byte record array")
        if self.preds.dtype != np.uint16 or self.fpreds.dtype != np.uint32 or self.topo.dtype != np.uint32:
            raise ValueError("corpus index arrays have the wrong dtype")
        return self

    def slice(self, k0: int, k1: int) -> "Corpus":
        """Kernels [k0, k1) as a self-contained corpus (offsets rebased; the
        signature table is kept whole so latency tables stay identical)."""
        k0, k1 = max(0, k0), min(self.n_ker, k1)
        ker = self.ker[k0:k1].copy()
        if k1 <= k0:
            return Corpus(tok=np.zeros(1, TOKEN_DT), preds=np.zeros(0, np.uint16),
                          blk=np.zeros(0, BLOCK_DT), fpreds=np.zeros(0, np.uint32),
                          topo=np.zeros(0, np.uint32), ker=ker, sigs=list(self.sigs), names=[])
        b0 = int(ker["blk0"][0])
        b1 = int(ker["blk0"][-1] + ker["n_blk"][-1])
        t0 = int(ker["tok0"][0])
        t1 = int(ker["tok0"][-1] + ker["n_tok"][-1])
        o0 = int(ker["topo0"][0])
        o1 = int(ker["topo0"][-1] + ker["n_blk"][-1])
        blk = self.blk[b0:b1].copy()
        f0 = int(blk["fpred0"][0]) if len(blk) else 0
        f1 = int(blk["fpred0"][-1] + blk["n_fpred"][-1]) if len(blk) else 0
        p0, p1 = int(self.tok["pred0"][t0]), int(self.tok["pred0"][t1])
        tok = self.tok[t0:t1 + 1].copy()          # + the sentinel (its pred0 = p1)
        tok["pred0"] -= p0
        tok[-1] = np.zeros((), TOKEN_DT)
        tok["pred0"][-1] = p1 - p0
        blk["tok0"] -= t0
        blk["fpred0"] -= f0
        ker["blk0"] -= b0
        ker["topo0"] -= o0
        ker["tok0"] -= t0
        return Corpus(tok=tok, preds=self.preds[p0:p1].copy(), blk=blk,
                      fpreds=self.fpreds[f0:f1].copy(), topo=self.topo[o0:o1].copy(), ker=ker,
                      sigs=list(self.sigs), names=list(self.names[k0:k1]))

    def kernel_tokens(self, k: int) -> tuple[int, int]:
        return int(self.ker[k]["tok0"]), int(self.ker[k]["n_tok"])


class CorpusBuilder:
    """Accumulates kernels into one packed corpus with a shared signature table."""

    def __init__(self):
        self._sig: dict = {}
        self.sigs: list = []
        self._tok: list = []     # (res, cls, sig, lst_row, lst_len)
        self._pred_cnt: list = []
        self._preds: list = []
        self._blk: list = []
        self._fpreds: list = []
        self._topo: list = []
        self._ker: list = []
        self.names: list = []

    def _sig_id(self, klass: str, root: str, kind) -> int:
        key = (klass, root if klass not in ("GlobalMemory", "SharedMemory") else "",
               kind if klass not in ("GlobalMemory", "SharedMemory") else None)
        sid = self._sig.get(key)
        if sid is None:
            sid = self._sig[key] = len(self.sigs)
            self.sigs.append(key)
        return sid

    def add(self, graph) -> int:
        order = graph.topo_order()          # raises ScheduleError on a cyclic CFG
        mult = graph.loop_multipliers()     # raises ScheduleError on a missing trip count
        nb = len(graph.blocks)
        preds_of: list[list[int]] = [[] for _ in range(nb)]
        has_succ = [False] * nb
        for u, v in graph.edges:
            preds_of[v].append(u)
            has_succ[u] = True
        k = len(self._ker)
        blk0, tok0, topo0 = len(self._blk), len(self._tok), len(self._topo)
        max_n = 0
        for b, blk in enumerate(graph.blocks):
            ins = blk.instructions
            n = len(ins)
            max_n = max(max_n, n)
            dfg = [[] for _ in range(n)]
            for u, v in blk.dfg_edges:
                dfg[v].append(u)
            if n > 65535:
                raise ScheduleError("basic block longer than 65535 instructions")
            res_cnt = [0] * NRES
            for inst in ins:
                res_cnt[_code(inst.resource, RESOURCE_CODE)] += 1
            res_row = [sum(res_cnt[:r]) for r in range(NRES)]
            seen = [0] * NRES
            n_glob = 0
            t0 = len(self._tok)
            for i, inst in enumerate(ins):
                kl = getattr(inst.klass, "value", inst.klass)
                rc = _code(inst.resource, RESOURCE_CODE)
                cc = CLASS_CODE[kl]
                flags = cc
                if inst.is_branch:
                    flags |= _FLAG_BRANCH
                if kl == "GlobalMemory":
                    n_glob += 1
                    if inst.root in ("ld", "ldu"):
                        flags |= _FLAG_GLOAD
                    elif inst.root == "st":
                        flags |= _FLAG_GSTORE
                self._tok.append((rc, flags, self._sig_id(kl, inst.root, latency_kind(inst.suffixes)),
                                  res_row[rc], seen[rc]))
                seen[rc] += 1
                ps = sorted(set(dfg[i]))
                if any(p >= i or p < 0 for p in ps):
                    raise ScheduleError("DFG edge does not point forward inside its block")
                self._pred_cnt.append(len(ps))
                self._preds.extend(ps)
            fp0 = len(self._fpreds)
            self._fpreds.extend(preds_of[b])
            m = int(mult[b])
            if not -(1 << 63) <= m < (1 << 63):
                raise ScheduleError("loop multiplier exceeds int64")
            self._blk.append((m, t0, n, fp0, len(preds_of[b]), n_glob, res_cnt, int(not has_succ[b])))
        self._topo.extend(order)
        self._ker.append((blk0, nb, topo0, max_n, tok0, len(self._tok) - tok0))
        self.names.append(graph.name)
        return k

    def build(self) -> Corpus:
        n_tok = len(self._tok)
        tok = np.zeros(n_tok + 1, TOKEN_DT)
        if n_tok:
            arr = np.asarray(self._tok, dtype=np.int64)
            tok["res"][:n_tok] = arr[:, 0]
            tok["cls"][:n_tok] = arr[:, 1]
            tok["sig"][:n_tok] = arr[:, 2]
            tok["lst_row"][:n_tok] = arr[:, 3]
            tok["lst_len"][:n_tok] = arr[:, 4]
        cnt = np.asarray(self._pred_cnt, dtype=np.int64)
        tok["pred0"][1:] = np.cumsum(cnt)
        blk = np.zeros(len(self._blk), BLOCK_DT)
        for i, (m, t0, n, fp0, nfp, ng, rc, ex) in enumerate(self._blk):
            blk[i] = (m, t0, n, fp0, nfp, ng, rc, ex)
        ker = np.zeros(len(self._ker), KERNEL_DT)
        for i, row in enumerate(self._ker):
            ker[i] = row
        return Corpus(tok=tok, preds=np.asarray(self._preds, dtype=np.uint16),
                      blk=blk, fpreds=np.asarray(self._fpreds, dtype=np.uint32),
                      topo=np.asarray(self._topo, dtype=np.uint32), ker=ker,
                      sigs=list(self.sigs), names=list(self.names))


def pack_corpus(graphs) -> Corpus:
    b = CorpusBuilder()
    for g in graphs:
        b.add(g)
    return b.build()


def arch_record(p: ArchProfile) -> np.ndarray:
    """ArchProfile -> one ARCH_DT record (fields of reference ``profiles.py:104-135``)."""
    bp = p.gm_latency_model.breakpoints
    if len(bp) > GK_MAX_BP:
        raise ProfileError(f"piecewise model has {len(bp)} breakpoints; the device "
                           f"record holds at most {GK_MAX_BP}")
    r = np.zeros((), ARCH_DT)
    order = ("SP", "SFU", "DPU", "LSU", "WS")
    res = {getattr(k, "value", k): v for k, v in p.resources.items()}
    gaps = {getattr(k, "value", k): v for k, v in p.latency.issue_gap.items()}
    r["units"] = [res[n] for n in order]
    r["gap"] = [float(gaps.get(n, 0.0)) for n in order]
    r["pipeline"] = p.latency.pipeline
    for f in ("nSM", "L2_sz", "nTh_sm_max", "reg_b_max", "shm_b_max", "nB_max", "wSM_max",
              "Sz_w", "access_sz", "access_gm_sz", "access_shm_sz", "nWS", "nDU", "nu_gpu"):
        r[f] = getattr(p, f)
    r["tpg_a"], r["tpg_b"], r["tpg_c"] = p.tp_global.a, p.tp_global.b, p.tp_global.c
    r["tps_a"], r["tps_b"], r["tps_c"] = p.tp_shared.a, p.tp_shared.b, p.tp_shared.c
    r["tp_floor"] = p.tp_floor
    r["ov_slope"], r["ov_icpt"] = p.overhead.slope, p.overhead.intercept
    r["n_bp"] = len(bp)
    r["bp"][: len(bp)] = bp
    segs = p.gm_latency_model.segments
    r["seg_slope"][: len(segs)] = [s for s, _ in segs]
    r["seg_icpt"][: len(segs)] = [b for _, b in segs]
    return r


def arch_records(profiles) -> np.ndarray:
    return np.stack([arch_record(p) for p in profiles]).astype(ARCH_DT)


def latency_table(profiles, sigs) -> np.ndarray:
    """[n_arch][n_sig] f64; GLOBAL signatures are NaN (point-dependent gm_lat)."""
    out = np.full((len(profiles), max(len(sigs), 1)), np.nan)
    for a, p in enumerate(profiles):
        for s, (klass, root, kind) in enumerate(sigs):
            v = resolve_signature(p, klass, root, kind)
            if v is not None:
                out[a, s] = v
    return out


def config_array(configs) -> np.ndarray:
    """LaunchConfig-likes or (nB, tpb, regs, shmem) tuples -> CONFIG_DT."""
    out = np.zeros(len(configs), CONFIG_DT)
    for i, c in enumerate(configs):
        if hasattr(c, "n_blocks"):
            c = (c.n_blocks, c.threads_per_block, c.reg_per_thread, c.shmem_per_block)
        nb, tpb, regs, shm = c
        if nb < 1 or tpb < 1 or regs < 0 or shm < 0 or max(c) >= 2 ** 31:
            raise ScheduleError(f"launch config {tuple(c)} out of range")
        out[i] = (nb, tpb, regs, shm)
    return out


# The 15-feature selection shipped models use (reference features.py:56-75)
FEATURE_ORDER = (
    "avg_comp_lat", "avg_glob_lat", "avg_misc_lat", "avg_shar_lat", "branch",
    "comp_inst_kernel", "comp_inst_sm", "comp_lat_sm", "glob_inst_kernel", "glob_inst_sm",
    "glob_lat_sm", "glob_load_sm", "glob_store_sm", "misc_inst_kernel", "misc_inst_sm",
    "misc_lat_sm", "shar_inst_kernel", "shar_inst_sm", "shar_lat_sm", "sm_active", "n_warps",
    "waves", "total_threads", "inst_issue_cycles", "cache_penalty", "glb_penalty",
    "sh_penalty", "occupancy", "reg_thread", "shmem_block", "block_size", "grid_size",
)
_SEL = {"avg_comp_lat", "avg_glob_lat", "avg_shar_lat", "branch", "comp_inst_kernel",
        "glob_inst_kernel", "glob_load_sm", "glob_store_sm", "misc_inst_kernel",
        "inst_issue_cycles", "cache_penalty", "occupancy", "reg_thread", "shmem_block",
        "block_size"}
SELECTED_FEATURES = tuple(f for f in FEATURE_ORDER if f in _SEL)
assert len(FEATURE_ORDER) == 32 and len(SELECTED_FEATURES) == 15


def manifest_indices(manifest) -> np.ndarray:
    idx = []
    for name in manifest:
        if name not in FEATURE_ORDER:
            raise ValueError(f"manifest feature '{name}' is not a static feature")
        idx.append(FEATURE_ORDER.index(name))
    return np.asarray(idx, dtype=np.int32)


__all__ = ["Corpus", "CorpusBuilder", "pack_corpus", "arch_record", "arch_records",
           "latency_table", "config_array", "FEATURE_ORDER", "SELECTED_FEATURES",
           "manifest_indices", "InstClass"]
