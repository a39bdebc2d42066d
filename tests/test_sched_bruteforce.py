"""Device schedule_block vs a brute-force scheduler on 500 random blocks --
the reference's own equivalence gate (pkg/tests/test_scheduler.py:153-160 with
pkg/tests/oracle_scheduler.py:16-49), restated here: integer latencies,
per-resource busy-cycle sets probed one cycle at a time.  Random profiles
(units, pipeline depth, issue gaps, latencies), random DAGs of <= 12
instructions, random thread counts; the device runs the whole block through
K3 (lane-per-point first fit, probes, insertion steps) and its per-
instruction starts and block delay must equal the brute force exactly.
Also the reference's schedule invariants (test_scheduler.py:163-182)."""

import random
from collections import defaultdict

import numpy as np
import pytest

from paper_2305_01886_b200 import pack
from paper_2305_01886_b200.ir import BasicBlock, InstClass, KernelGraph, PtxInstruction, Resource
from paper_2305_01886_b200.profiles import profile_from_dict

pytestmark = pytest.mark.gpu
RES = list(Resource)


def _inst(i, res):
    return PtxInstruction(root=f"op{i}", suffixes=(), klass=InstClass.COMPUTE, resource=res,
                          defs=frozenset({f"%r{i}"}), uses=frozenset(), operands=(f"%r{i}",),
                          line=i + 1)


def _case(rng):
    n = rng.randint(1, 12)
    insts = [_inst(i, rng.choice(RES)) for i in range(n)]
    edges = [(u, v) for v in range(n) for u in range(v) if rng.random() < 0.3]
    block = BasicBlock(label="bb0", instructions=insts, dfg_edges=edges)
    doc = {
        "schema_version": 1, "name": "random",
        "resources": {r.value: rng.choice([1, 2, 4, 32, 192]) for r in Resource},
        "attributes": {"nSM": 4, "nu_gpu_mhz": 1000, "nu_mem_mhz": 2000, "L2_sz": 1 << 20,
                       "nTh_sm_max": 2048, "reg_b_max": 65536, "shm_b_max": 49152,
                       "nB_max": 16, "wSM_max": 64, "Sz_w": 32, "access_sz": 4, "nWS": 4,
                       "nDU": 8},
        "latencies": {
            "pipeline": rng.randint(1, 2),
            "issue_gap": {r.value: rng.randint(0, 2) for r in Resource if rng.random() < 0.5},
            "instructions": {**{f"op{i}": rng.randint(1, 15) for i in range(n)}, "shared": 40},
            "class_defaults": {"Compute": 9, "Miscellaneous": 2}},
        "throughput_models": {"global": {"a": 1000.0, "b": 1.04, "c": 0.001},
                              "shared": {"a": 1000.0, "b": 1.0, "c": 0.001}},
        "penalty_models": {"launch_overhead": {"slope_us": 1e-5, "intercept_us": 1.0},
                           "global_latency_piecewise": {
                               "breakpoints": [1000],
                               "segments": [{"slope": 0.01, "intercept": 200},
                                            {"slope": 0.001, "intercept": 210}]}},
    }
    return profile_from_dict(doc), block, rng.choice([1, 32, 64, 128, 256, 512]), doc


def _bruteforce(doc, block, n_tw):
    """pkg/tests/oracle_scheduler.py:16-49, restated."""
    lat = doc["latencies"]
    preds = defaultdict(list)
    for u, v in block.dfg_edges:
        preds[v].append(u)
    busy = defaultdict(set)
    starts, fin, delay = [], [], 0
    for v, inst in enumerate(block.instructions):
        r = inst.resource.value
        units = doc["resources"][r]
        d = lat["instructions"][inst.root] + lat["pipeline"] * (-(-n_tw // units) - 1)
        span = d + lat["issue_gap"].get(r, 0)
        ready = max((fin[u] for u in preds[v]), default=0)
        t = ready
        while any((t + k) in busy[r] for k in range(span)):
            t += 1
        busy[r].update(range(t, t + span))
        starts.append(t)
        fin.append(t + d)
        delay = max(delay, t + d)
    return starts, delay


def test_device_schedule_equals_bruteforce_500_cases():
    from paper_2305_01886_b200 import runtime as rt

    rng = random.Random(20240817)
    bad = []
    for case in range(500):
        prof, block, n_tw, doc = _case(rng)
        g = KernelGraph(name=f"c{case}", blocks=[block])
        dc = rt.DeviceCorpus.upload(pack.pack_corpus([g]))
        dg = rt.DeviceGrid.build(dc, [prof], [(1, 32, 0, 0)], n_tw=[n_tw], gm=[0.0])
        out = rt.schedule_features(dc, dg, trace=True)
        got = out["tr_start"].cpu().numpy()[0]
        delay = float(out["tr_blk_delay"].cpu().numpy()[0, 0])
        want, want_delay = _bruteforce(doc, block, n_tw)
        if not (np.array_equal(got, np.asarray(want, np.float64)) and delay == want_delay):
            bad.append((case, got.tolist(), want, delay, want_delay))
        # invariants (test_scheduler.py:163-182)
        dur = out["tr_duration"].cpu().numpy()[0]
        for u, v in block.dfg_edges:
            assert got[v] >= got[u] + dur[u]
        spans = defaultdict(list)
        for i, inst in enumerate(block.instructions):
            gap = doc["latencies"]["issue_gap"].get(inst.resource.value, 0)
            spans[inst.resource].append((got[i], got[i] + dur[i] + gap))
        for sp in spans.values():
            sp.sort()
            for (s1, e1), (s2, e2) in zip(sp, sp[1:]):
                assert e1 <= s2
    assert not bad, bad[:2]
