"""Per-CUDA-source-line aggregates (stall samples, warp instructions) from an
.ncu-rep captured with -lineinfo + --import-source: the hot lines of a kernel."""
import csv
import io
import subprocess
import sys


def lines(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    out, path, head = [], None, None
    for r in csv.reader(io.StringIO(raw)):
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            head = r
            continue
        if head is None or not r[0]:
            continue
        d = dict(zip(head[2:], r[2:]))  # columns after (Line No, Source)
        try:
            s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            e = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            continue
        out.append((s, e, f"{path}:{r[0]}", r[1].strip()[:70]))
    return out


if __name__ == "__main__":
    data = lines(sys.argv[1])
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    ts = sum(d[0] for d in data) or 1
    te = sum(d[1] for d in data) or 1
    print(f"total samples {ts}, warp instructions {te}")
    print("--- by stall samples")
    for s, e, loc, src in sorted(data, reverse=True)[:n]:
        print(f"{100 * s / ts:5.1f}% smp {100 * e / te:5.1f}% ins  {loc:22s} {src}")
    print("--- by instructions")
    for s, e, loc, src in sorted(data, key=lambda d: -d[1])[:n // 2]:
        print(f"{100 * s / ts:5.1f}% smp {100 * e / te:5.1f}% ins  {loc:22s} {src}")
