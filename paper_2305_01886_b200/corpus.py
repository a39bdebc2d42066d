"""Synthetic PTX corpora and launch-config grids for the BASELINE.json configs.

SURVEY §8(d): kernels of U[40, 200] instructions drawn from an add / mul / fma /
mad / setp / cvt / sqrt / div / mov / ld-st global / ld-st shared / bar.sync /
f64 mix, 0-2 loops with trip counts U[2, 16], forward guards.  Each kernel is
emitted as PTX *text* plus its loop-count map, so the same input drives the
reference parser (golden generation) and this package's parser (device path).
"""

from __future__ import annotations

import itertools
import random

# (weight, template).  {d} dest, {a} {b} {c} sources, by register family.
_OPS = [
    (10, "add.s32", "r", "rr"), (4, "sub.s32", "r", "rr"), (6, "mul.lo.s32", "r", "rr"),
    (5, "mad.lo.s32", "r", "rrr"), (3, "shl.b32", "r", "ri"), (3, "and.b32", "r", "rr"),
    (8, "add.f32", "f", "ff"), (4, "sub.f32", "f", "ff"), (8, "mul.f32", "f", "ff"),
    (8, "fma.rn.f32", "f", "fff"), (2, "sqrt.rn.f32", "f", "f"), (2, "div.rn.f32", "f", "ff"),
    (1, "rcp.rn.f32", "f", "f"), (1, "ex2.approx.f32", "f", "f"), (3, "cvt.rn.f32.s32", "f", "r"),
    (2, "cvt.rzi.s32.f32", "r", "f"), (4, "mov.u32", "r", "r"), (2, "mov.f32", "f", "f"),
    (3, "setp.lt.s32", "p", "rr"), (2, "setp.gt.f32", "p", "ff"), (2, "selp.f32", "f", "ffp"),
    (3, "mul.wide.s32", "d", "ri"), (3, "add.s64", "d", "dd"), (2, "cvta.to.global.u64", "d", "d"),
    (2, "add.f64", "D", "DD"), (2, "mul.f64", "D", "DD"), (1, "fma.rn.f64", "D", "DDD"),
    (1, "cvt.f64.f32", "D", "f"), (1, "div.rn.f64", "D", "DD"),
    (7, "ld.global.f32", "f", "A"), (3, "st.global.f32", "", "Af"),
    (2, "ld.global.nc.f32", "f", "A"), (1, "ldu.global.f32", "f", "A"),
    (3, "ld.shared.f32", "f", "A"), (2, "st.shared.f32", "", "Af"), (1, "atom.global.add.u32", "r", "Ar"),
    (1, "bar.sync", "", "0"), (1, "ld.param.u64", "d", "P"), (1, "mov.u32", "r", "S"),
]
_W = [w for w, *_ in _OPS]
_FAM = {"r": "%r", "f": "%f", "d": "%rd", "D": "%fd", "p": "%p"}
_SPECIAL = ["%tid.x", "%ntid.x", "%ctaid.x", "%nctaid.x"]


class _Emitter:
    def __init__(self, rng: random.Random):
        self.rng = rng
        self.lines: list[str] = []
        self.n_instr = 0
        self.live = {k: [f"{_FAM[k]}{i}" for i in range(1, 4)] for k in _FAM}
        self.next = {k: 4 for k in _FAM}
        self.labels = 0
        self.loops: dict[str, int] = {}

    def reg(self, fam: str) -> str:
        pool = self.live[fam]
        # bias towards recent definitions so chains form
        return pool[-1 - min(int(self.rng.expovariate(0.6)), len(pool) - 1)]

    def fresh(self, fam: str) -> str:
        r = f"{_FAM[fam]}{self.next[fam]}"
        self.next[fam] += 1
        self.live[fam].append(r)
        if len(self.live[fam]) > 24:
            self.live[fam].pop(0)
        return r

    def emit(self, text: str) -> None:
        self.lines.append("\t" + text + ";")
        self.n_instr += 1

    def op(self) -> None:
        _, name, dst, srcs = self.rng.choices(_OPS, weights=_W)[0]
        ops = []
        for s in srcs:
            if s == "i":
                ops.append(str(self.rng.choice([1, 2, 4, 8, 12])))
            elif s == "A":
                off = self.rng.choice(["", "+4", "+8", "+16"])
                ops.append(f"[{self.reg('d')}{off}]")
            elif s == "P":
                ops.append(f"[param_{self.rng.randint(0, 3)}]")
            elif s == "S":
                ops.append(self.rng.choice(_SPECIAL))
            elif s == "0":
                ops.append("0")
            else:
                ops.append(self.reg(s))
        if name.startswith("st.") or name == "bar.sync":
            self.emit(f"{name} {', '.join(ops)}")
            return
        d = self.fresh(dst)
        self.emit(f"{name} {d}, {', '.join(ops)}")

    def label(self) -> str:
        self.labels += 1
        return f"$L__BB{self.labels}"

    def straight(self, n: int) -> None:
        for _ in range(n):
            self.op()


def synth_kernel(rng: random.Random, name: str) -> tuple[str, dict[str, int]]:
    """One synthetic kernel: (PTX text, loop trip counts by head label)."""
    e = _Emitter(rng)
    target = rng.randint(40, 200)
    n_loops = rng.choice([0, 0, 1, 1, 2])
    n_guards = rng.choice([0, 1, 1, 2])
    regions = ["loop"] * n_loops + ["guard"] * n_guards
    rng.shuffle(regions)
    budget = target - 2 * n_loops - 2 * n_guards - 1
    cuts = sorted(rng.randint(0, max(budget, 0)) for _ in range(2 * len(regions)))
    pieces = [b - a for a, b in zip([0] + cuts, cuts + [max(budget, 0)])]
    e.straight(pieces[0])
    for i, kind in enumerate(regions):
        body, tail = pieces[2 * i + 1], pieces[2 * i + 2]
        if kind == "loop":
            head = e.label()
            e.lines.append(f"{head}:")
            inner = rng.random() < 0.25 and body > 8
            if inner:
                part = body // 2
                e.straight(part // 2)
                ih = e.label()
                e.lines.append(f"{ih}:")
                e.straight(max(part - part // 2, 1))
                p = e.fresh("p")
                e.emit(f"setp.lt.s32 {p}, {e.reg('r')}, {e.reg('r')}")
                e.emit(f"@{p} bra {ih}")
                e.loops[ih] = rng.randint(2, 16)
                e.straight(max(body - part, 1))
            else:
                e.straight(max(body, 1))
            p = e.fresh("p")
            e.emit(f"setp.lt.s32 {p}, {e.reg('r')}, {e.reg('r')}")
            e.emit(f"@{p} bra {head}")
            e.loops[head] = rng.randint(2, 16)
        else:
            skip = e.label()
            p = e.fresh("p")
            e.emit(f"setp.ge.s32 {p}, {e.reg('r')}, {e.reg('r')}")
            e.emit(f"@{p} bra {skip}")
            e.straight(max(body, 1))
            e.lines.append(f"{skip}:")
        e.straight(tail)
    e.emit("ret")
    text = (
        ".version 7.0\n.target sm_70\n.address_size 64\n\n"
        f".visible .entry {name}(\n\t.param .u64 param_0\n)\n{{\n"
        "\t.reg .pred %p<64>;\n\t.reg .f32 %f<256>;\n\t.reg .b32 %r<256>;\n"
        "\t.reg .b64 %rd<128>;\n\t.reg .f64 %fd<64>;\n\n"
        + "\n".join(e.lines) + "\n}\n"
    )
    return text, dict(e.loops)


def synth_corpus(n_kernels: int, seed: int, prefix: str = "k") -> list[tuple[str, str, dict]]:
    """[(name, ptx_text, loop_counts)] for n_kernels deterministic kernels."""
    rng = random.Random(seed)
    out = []
    for i in range(n_kernels):
        name = f"{prefix}{seed}_{i}"
        text, loops = synth_kernel(rng, name)
        out.append((name, text, loops))
    return out


# ---------------------------------------------------------------- config grids

CONFIG1 = [(64, 256, 32, 0), (256, 128, 24, 4096), (1024, 1024, 16, 0), (13, 64, 40, 8192)]

_NB2 = (1, 13, 64, 256, 1024, 4096, 16384, 65535)
_TPB2 = (32, 64, 128, 256, 512, 1024)
_RS2 = ((0, 0), (32, 0), (64, 16384))


def config2_grid() -> list[tuple[int, int, int, int]]:
    """Config #2's 64 launch configs: (regs, shm) outer, then nB x tpb; the first
    64 of the 144 (all feasible on every shipped arch).  Includes the
    65535 x {512, 1024} pairs whose global latency is negative."""
    grid = [(nb, t, r, s) for (r, s) in _RS2 for nb in _NB2 for t in _TPB2]
    return grid[:64]


def config5_grid() -> list[tuple[int, int, int, int]]:
    """Config #5's 256 configs: 16 log-spaced grid sizes x tpb 64..1024, regs 32."""
    import numpy as np

    nbs = [int(v) for v in np.round(np.logspace(0, np.log10(65535), 16))]
    return [(nb, t, 32, 0) for nb in nbs for t in range(64, 1025, 64)]


def random_configs(rng: random.Random, n: int) -> list[tuple[int, int, int, int]]:
    """Mixed feasible / infeasible configs for parity tests."""
    out = []
    for _ in range(n):
        out.append((rng.choice([1, 2, 5, 13, 64, 100, 777, 4096, 65535, 200000]),
                    rng.choice([1, 31, 32, 33, 64, 96, 128, 192, 256, 384, 512, 1024, 2048]),
                    rng.choice([0, 0, 16, 32, 63, 64, 128, 255]),
                    rng.choice([0, 0, 1024, 4096, 16384, 24576, 49152, 65536])))
    return out


__all__ = ["synth_kernel", "synth_corpus", "CONFIG1", "config2_grid", "config5_grid",
           "random_configs"]
_ = itertools
