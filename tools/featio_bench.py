"""Feature-CSV I/O timing: native writer/parser (featio) vs the reference's
Python features_to_csv / features_from_csv algorithm, on config #2's shape
(640k points x 32 features).  Host-only; the Python side runs on a bounded
sample and is scaled linearly.

    python tools/featio_bench.py [--rows 640000] [--sample 20000]
"""

import argparse
import csv
import io
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_01886_b200 import featio  # noqa: E402
from paper_2305_01886_b200.pack import FEATURE_ORDER  # noqa: E402


def py_write(kernels, feat):
    out = io.StringIO()
    w = csv.writer(out, lineterminator="\n")
    w.writerow(("kernel",) + FEATURE_ORDER)
    for k, row in zip(kernels, feat.tolist()):
        w.writerow([k] + [format(v, ".17g") for v in row])
    return out.getvalue()


def py_read(text):
    return [{k: (v if k == "kernel" else float(v)) for k, v in r.items()}
            for r in csv.DictReader(io.StringIO(text))]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=640_000)
    ap.add_argument("--sample", type=int, default=20_000)
    a = ap.parse_args()
    rng = np.random.default_rng(2)
    feat = rng.random((a.rows, 32)) * 10.0 ** rng.integers(-3, 9, (a.rows, 32))
    kernels = [f"k{i // 64}[{1 + i % 977}x{64 * (1 + i % 16)}]" for i in range(a.rows)]
    t = time.perf_counter(); text = featio.features_csv(kernels, feat); tw = time.perf_counter() - t
    t = time.perf_counter(); rows = featio.features_from_csv(text); tr = time.perf_counter() - t
    t = time.perf_counter(); featio.features_from_csv_arrays(text); ta = time.perf_counter() - t
    s = a.sample
    t = time.perf_counter(); ptext = py_write(kernels[:s], feat[:s]); pw = (time.perf_counter() - t) * a.rows / s
    t = time.perf_counter(); py_read(ptext); pr = (time.perf_counter() - t) * a.rows / s
    assert ptext == featio.features_csv(kernels[:s], feat[:s])
    assert len(rows) == a.rows
    print(f"{a.rows} rows, {len(text) / 1e6:.0f} MB: write {tw:.2f} s (python {pw:.1f} s), "
          f"read dicts {tr:.2f} s / arrays {ta:.2f} s (python {pr:.1f} s)")


if __name__ == "__main__":
    main()
