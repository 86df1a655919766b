"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by
kernel (launches, total ms, share of the captured GPU time), optionally split at
a launch index so the SPAI builds + warm-up batch and the later steps read
separately. Usage: launch_summary.py LIST.csv[.gz] [--skip N]"""
import argparse
import collections
import csv
import gzip
import io
import re


def rows(path):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt", errors="replace") as f:
        text = f.read()
    start = text.find('"ID"')
    for r in csv.DictReader(io.StringIO(text[start:])):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            yield int(r["ID"]), r["Kernel Name"], float(r["Metric Value"].replace(",", "")), r["Metric Unit"]


def short(name):
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"\(.*$", "", name)  # argument list
    name = name.replace("mpg::<unnamed>::", "")
    return name[:45]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--skip", type=int, default=0, help="summarise launches with ID >= skip")
    ap.add_argument("--drop", default=None, help="regex of kernel names left out (e.g. the SPAI builds)")
    a = ap.parse_args()
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    n = 0
    for i, k, v, u in rows(a.csv):
        if i < a.skip or (a.drop and re.search(a.drop, k)):
            continue
        n += 1
        e = agg[short(k)]
        e[0] += 1
        e[1] += v * scale[u]
    tot = sum(e[1] for e in agg.values())
    drop = f", without /{a.drop}/" if a.drop else ""
    print(f"# {n} launches from ID {a.skip}{drop}, {tot:.1f} ms of serialised cold-cache GPU time")
    print(f"{'kernel':46s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}")
    for k, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:46s} {c:8d} {ms:10.2f} {ms / tot * 100:6.1f}%")


if __name__ == "__main__":
    main()
