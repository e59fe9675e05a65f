#!/usr/bin/env python
"""Re-pick a TuneDB from the tuner's full candidate table (tools/tune_sweep.py
--all-out): per signature, among the candidates within ``--slack`` x the
fastest time, the one minimising  time * (min(CTAs, SMs) / SMs) ** alpha.

alpha = 0 is the latency-optimal DB (what tune_sweep writes); alpha = 1 minimises
the SM-time an op occupies, which is what a concurrent schedule of the sweep's
independent ops packs onto the GPU (bench.py --streams).  Every candidate in
the table already passed the tuner's on-device check against conv_simple.

    python tools/pick_db.py --cands cands_fp32.csv --out db.tsv --alpha 0.5 --slack 2
"""

from __future__ import annotations

import argparse
import csv
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1611_06945_b200 import tuner  # noqa: E402
from paper_1611_06945_b200.backend import CostReport  # noqa: E402
from paper_1611_06945_b200.variants import TuneParams  # noqa: E402


def pick(cands, alpha: float, slack: float, sms: int = 148):
    best_t = min(c[0] for c in cands)
    pool = [c for c in cands if c[0] <= slack * best_t]
    return min(pool, key=lambda c: (c[0] * (min(c[1], sms) / sms) ** alpha, c[0]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cands", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--alpha", type=float, default=0.0)
    ap.add_argument("--slack", type=float, default=1.0)
    a = ap.parse_args()
    by = defaultdict(list)
    import gzip

    with (gzip.open(a.cands, "rt") if a.cands.endswith(".gz") else open(a.cands)) as fh:
        for r in csv.DictReader(fh):
            by[r["signature"]].append((float(r["ns"]), int(r["ctas"]), r["variant"], r["params"]))
    db = tuner.TuneDB()
    for sig, cands in sorted(by.items()):
        ns, ctas, vname, ps = pick(cands, a.alpha, a.slack)
        db.add(tuner.TuneRecord(sig, vname, TuneParams.from_string(ps), ns, CostReport(wall_ns=int(ns)),
                                objective=tuner.WALL))
    tuner.save_db(db, a.out)
    print(f"{len(db.records)} records (alpha={a.alpha}, slack={a.slack}) -> {a.out}")


if __name__ == "__main__":
    main()
