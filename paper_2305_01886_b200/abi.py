"""ctypes mirror of the descriptor structs in ``include/gk.h``.

Pointer fields are plain integers (device addresses for libgk, host addresses
for the CPU oracle), so the same descriptors serve both.
"""

from __future__ import annotations

import ctypes as C

P = C.c_void_p


class GkCorpus(C.Structure):
    _fields_ = [("tok", P), ("preds", P), ("blk", P), ("fpreds", P), ("topo", P), ("ker", P),
                ("n_tok", C.c_uint32), ("n_blk", C.c_uint32), ("n_ker", C.c_uint32),
                ("n_sig", C.c_uint32), ("max_n", C.c_uint32), ("max_blk", C.c_uint32)]


class GkGrid(C.Structure):
    _fields_ = [("kernel_ids", P), ("cfg", P), ("arch", P), ("lat", P),
                ("n_tw_override", P), ("gm_override", P), ("order", P), ("tp_clamps", P),
                ("n_k", C.c_uint32), ("n_cfg", C.c_uint32), ("n_arch", C.c_uint32),
                ("pad_", C.c_uint32)]


class GkTrace(C.Structure):
    _fields_ = [("start", P), ("duration", P), ("latency", P), ("n_batches", P),
                ("blk_delay", P), ("blk_finish", P)]


class GkEnsemble(C.Structure):
    _fields_ = [("nodes", P), ("tree_off", P), ("tree_depth", P), ("scale_lo", P), ("scale_hi", P),
                ("base_score", C.c_double), ("n_trees", C.c_uint32), ("n_feat", C.c_uint32),
                ("max_depth", C.c_uint32), ("nodes8", P), ("blocks", P), ("thr64", P), ("leaf_val", P),
                ("root", P), ("blocks3", P)]


NSI, NSF, NFEAT = 6, 9, 32
SI_NAMES = ("threads_scheduled", "threads_per_sm", "blocks_per_sm", "waves", "n_global",
            "n_shared")
SF_NAMES = ("gm_latency", "d_kernel", "overhead_cycles", "gm_penalty", "sm_penalty",
            "cm_penalty", "d_total", "time_us", "cfg_delay")
STATUS_OK, STATUS_INFEASIBLE_LAUNCH, STATUS_INFEASIBLE_OCCUPANCY = 0, 1, 2

assert C.sizeof(GkCorpus) == 72 and C.sizeof(GkGrid) == 80 and C.sizeof(GkEnsemble) == 112
