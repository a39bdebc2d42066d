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


CHUNK = 500  # kernels per generator chunk


def n_chunks(n_kernels: int, chunk: int = CHUNK) -> int:
    return -(-n_kernels // chunk)


def _chunk_job(n_kernels: int, seed: int, s: int, prefix: str, chunk: int):
    lo = s * chunk
    return (min(chunk, n_kernels - lo), seed * 100003 + s, f"{prefix}{seed}s{s}_")


def synth_chunks(n_kernels: int, seed: int, chunk_ids, prefix: str = "k",
                 procs: int | None = None, chunk: int = CHUNK) -> pack.Corpus:
    """The kernels of generator chunks `chunk_ids` (kernels [s * chunk, (s + 1) *
    chunk) of the `n_kernels`-kernel corpus synth_packed(n_kernels, seed)
    builds), packed in chunk order -- what one rank of a kernel-sharded sweep
    builds (dist.chunk_shard), without generating the other ranks' kernels."""
    jobs = [_chunk_job(n_kernels, seed, s, prefix, chunk) for s in chunk_ids]
    procs = procs or min(os.cpu_count() or 1, 32)
    if len(jobs) <= 1 or procs <= 1:
        parts = [_shard(j) for j in jobs]
    else:
        # forkserver: callers (bench, tests) already run CUDA / torch threads, where fork is unsafe
        with ProcessPoolExecutor(max_workers=procs, mp_context=mp.get_context("forkserver")) as ex:
            parts = list(ex.map(_shard, jobs))
    return parts[0] if len(parts) == 1 else merge_corpora(parts)


def synth_packed(n_kernels: int, seed: int, prefix: str = "k", procs: int | None = None,
                 chunk: int = CHUNK) -> pack.Corpus:
    """Packed corpus of `n_kernels` synthetic kernels (parallel generate+parse).
    One generator stream per seed is sequential; the corpus is built in chunks
    of `chunk` kernels from sub-seeds instead so workers are independent:
    kernel i of chunk s comes from seed (seed, s)."""
    procs = procs or min(os.cpu_count() or 1, 32)
    if n_kernels <= chunk or procs <= 1:
        return _shard((n_kernels, seed, prefix))
    return synth_chunks(n_kernels, seed, range(n_chunks(n_kernels, chunk)), prefix, procs, chunk)


def config3_table(rows: int, seed: int = 3) -> tuple[np.ndarray, np.ndarray]:
    """BASELINE config #3's static-feature table: 64 U[0,1)
    columns from ``default_rng(seed)`` (the last 8 rounded to integer counts in
    [0, 20)), y = 30 + 40 x0 + 20 x1^2 + 12 [x2 > 0.5] + 0.003*20000 x3 + N(0, 1).
    Raw (unscaled) values: ``trainer.train`` min-max scales per fold as the
    reference does (training.py:121-124)."""
    rng = np.random.default_rng(seed)
    X = rng.random((rows, 64))
    X[:, 56:] = np.floor(X[:, 56:] * 20)
    y = (30 + 40 * X[:, 0] + 20 * X[:, 1] ** 2 + 12 * (X[:, 2] > 0.5) + 0.003 * 20000 * X[:, 3]
         + rng.normal(0, 1, rows))
    return X, y
