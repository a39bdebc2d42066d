"""Golden outcomes of the REFERENCE feature-CSV functions
(gpukalc.features.features_to_csv / features_from_csv, features.py:250-272)
-- pins this package's native writer/parser (libgkhost, include/gk_featio.h)
and its Python mirror.

Run in the build container only (imports /root/reference):

    python tests/golden/make_featio_golden.py

Writes tests/golden/featio_cases.json:
  "write": per case the kernel names, the 32 feature values (float.hex, so NaN
           signs / -0.0 / subnormals survive JSON), `selected`, and the
           reference's CSV text;
  "read":  per case a CSV text and the reference outcome -- the rows (floats as
           float.hex, kernel strings as is) or the exception type + message.
"""

from __future__ import annotations

import json
import math
import random
import struct
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path[:0] = [str(REF / "src"), str(ROOT)]

from gpukalc.features import (  # noqa: E402
    FEATURE_ORDER,
    FeatureVector,
    features_from_csv,
    features_to_csv,
)

SPECIAL = [0.0, -0.0, 1.0, 57.0, 0.1, 1 / 3, 1e16, 1e17, 9007199254740993.0, 123456789.125,
           5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, -2.5e-7, 1e-5, 1e-4,
           float("inf"), float("-inf"), float("nan"),
           struct.unpack("<d", struct.pack("<Q", 0xFFF8000000000001))[0]]   # negative NaN
NAMES = ["vecadd[13x128]", "a,b", 'q"uote', "line\nbreak", "cr\rx", " spaced ", "", "unicodé",
         "tab\tx", '"', ",", "x\r\ny", "semi;colon", "'single'"]


def hx(v: float) -> str:
    if math.isnan(v):
        return "nan" if math.copysign(1.0, v) > 0 else "-nan"
    return v.hex()


def _rand_value(rng):
    r = rng.random()
    if r < 0.15:
        return rng.choice(SPECIAL)
    if r < 0.4:
        return float(rng.randint(-10 ** 6, 10 ** 12))
    if r < 0.7:
        return rng.uniform(-1e3, 1e3)
    return struct.unpack("<d", struct.pack("<Q", rng.getrandbits(64)))[0]


def write_cases():
    rng = random.Random(20261017)
    cases = []
    for c in range(24):
        n = rng.randint(0, 6) if c else 0
        rows = []
        for i in range(n):
            name = rng.choice(NAMES) if rng.random() < 0.6 else f"k{c}_{i}[{rng.randint(1, 65535)}x64]"
            vals = [_rand_value(rng) for _ in FEATURE_ORDER]
            rows.append((name, vals))
        for selected in (False, True):
            text = features_to_csv([(k, FeatureVector(*v)) for k, v in rows], selected=selected)
            cases.append({"kernels": [k for k, _ in rows],
                          "feat": [[hx(x) for x in v] for _, v in rows],
                          "selected": selected, "csv": text})
    return cases


def _outcome(text):
    try:
        rows = features_from_csv(text)
    except Exception as exc:   # noqa: BLE001 -- the reference's own exception
        return {"error": type(exc).__name__, "message": str(exc)}
    return {"rows": [{k: (v if isinstance(v, str) else hx(v)) for k, v in r.items()}
                     for r in rows]}


def read_cases(writes):
    texts = [w["csv"] for w in writes[:12]]
    texts += [
        "", "kernel\n", "kernel,a\n", "kernel,a\nk,1\n", "kernel,a\r\nk,1\r\n", "kernel,a\nk,1",
        "kernel,a\n\nk,1\n\n", "kernel,a\nk, 1.5\n", "kernel,a\nk,1_000\n", "kernel,a\nk,Infinity\n",
        "kernel,a\nk,-iNF\n", "kernel,a\nk,NaN\n", "kernel,a\nk,+1e5\n", "kernel,a\nk,.5\n",
        "kernel,a\nk,5.\n", "kernel,a\nk,0x10\n", "kernel,a\nk,\n", "kernel,a\nk\n",
        "kernel,a\nk,1,2\n", 'kernel,a\n"k,1",2\n', 'kernel,a\n"k""q",2\n', 'kernel,a\n"k\nz",3\n',
        'kernel,a\nk"x,4\n', 'kernel,a\n"k"x,5\n', "a,kernel\n1,k\n", "a,b\n1,2\n",
        "kernel,a,a\nk,1,2\n", "kernel,a\nk,1e400\n", "kernel,a\nk,1e-400\n",
        "kernel,a\nk,4.9406564584124654e-324\n", "kernel,a\nk,2.4703282292062328e-324\n",
        "kernel,a\nk,0.1000000000000000055511151231257827021181583404541015625\n",
        "kernel,a\nk,179769313486231580793728971405303415079934132710037826936173778980444968"
        "29257049521875\n",
        "kernel,a\rk,1\r", "kernel,a\nk,1\x00\n", "kernel,a\nk,١\n", "kernel,a\nk,abc\n",
        "﻿kernel,a\nk,1\n", "kernel,a\nk,-0\n", "kernel,a\nk,  \n", "kernel,a\nk,1 \n",
    ]
    return [{"csv": t, **_outcome(t)} for t in texts]


def main():
    writes = write_cases()
    out = {"write": writes, "read": read_cases(writes)}
    (HERE / "featio_cases.json").write_text(json.dumps(out, indent=1, ensure_ascii=False) + "\n")
    print(f"{len(out['write'])} write cases, {len(out['read'])} read cases")


if __name__ == "__main__":
    main()
