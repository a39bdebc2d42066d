"""Synthetic workloads of BASELINE.json's configs, built in parallel on the host.

Corpus generation + parsing is the host front-end: it runs
once, outside any timed region, sharded over worker processes; each worker
generates its shard's PTX text, parses + packs it with the native tokenizer
(libgkhost, byte-identical to parse_ptx + pack_corpus), and the shards are
merged into one corpus with a single signature table.
"""

from __future__ import annotations

import multiprocessing as mp
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np

from . import corpus as CG
from . import pack, ptx_native


def _shard(args):
    n, seed, prefix = args
    return ptx_native.pack_ptx(CG.synth_corpus(n, seed, prefix), threads=1)


def merge_corpora(parts: list) -> pack.Corpus:
    """Concatenate packed corpora, remapping signatures and offsets."""
    sigs: list = []
    sig_id: dict = {}
    toks, preds, blks, fpreds, topos, kers, names = [], [], [], [], [], [], []
    n_tok = n_pred = n_blk = n_fp = n_topo = 0
    for c in parts:
        remap = np.zeros(max(len(c.sigs), 1), dtype=np.uint16)
        for i, s in enumerate(c.sigs):
            s = tuple(s)
            if s not in sig_id:
                sig_id[s] = len(sigs)
                sigs.append(s)
            remap[i] = sig_id[s]
        t = c.tok[:-1].copy()
        t["sig"] = remap[t["sig"]]
        t["pred0"] += n_pred
        toks.append(t)
        preds.append(c.preds)
        b = c.blk.copy()
        b["tok0"] += n_tok
        b["fpred0"] += n_fp
        blks.append(b)
        fpreds.append(c.fpreds)
        topos.append(c.topo)
        k = c.ker.copy()
        k["blk0"] += n_blk
        k["topo0"] += n_topo
        k["tok0"] += n_tok
        kers.append(k)
        names += c.names
        n_tok += len(t)
        n_pred += len(c.preds)
        n_blk += len(c.blk)
        n_fp += len(c.fpreds)
        n_topo += len(c.topo)
    tok = np.zeros(n_tok + 1, pack.TOKEN_DT)
    if n_tok:
        tok[:-1] = np.concatenate(toks)
    tok[-1]["pred0"] = n_pred
    return pack.Corpus(tok=tok, preds=np.concatenate(preds).astype(np.uint16),
                       blk=np.concatenate(blks).astype(pack.BLOCK_DT), fpreds=np.concatenate(fpreds).astype(np.uint32),
                       topo=np.concatenate(topos).astype(np.uint32),
                       ker=np.concatenate(kers).astype(pack.KERNEL_DT),
                       sigs=sigs, names=names)


def synth_packed(n_kernels: int, seed: int, prefix: str = "k", procs: int | None = None,
                 chunk: int = 500) -> pack.Corpus:
    """Packed corpus of `n_kernels` synthetic kernels (parallel generate+parse)."""
    procs = procs or min(os.cpu_count() or 1, 32)
    if n_kernels <= chunk or procs <= 1:
        return _shard((n_kernels, seed, prefix))
    # one generator stream per seed is sequential; shard by sub-seed instead so
    # workers are independent: kernel i of shard s comes from seed (seed, s)
    jobs = []
    for s, lo in enumerate(range(0, n_kernels, chunk)):
        hi = min(lo + chunk, n_kernels)
        jobs.append((hi - lo, seed * 100003 + s, f"{prefix}{seed}s{s}_"))
    # forkserver: callers (bench, tests) already run CUDA / torch threads, where fork is unsafe
    with ProcessPoolExecutor(max_workers=procs, mp_context=mp.get_context("forkserver")) as ex:
        parts = list(ex.map(_shard, jobs))
    return merge_corpora(parts)
