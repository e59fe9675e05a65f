#!/usr/bin/env python
"""Merge tuner candidate CSVs (tools/tune_sweep.py --all-out): rows of the newer
file replace every row of the same op signature in the older one.

    python tools/merge_cands.py OLD.csv[.gz] NEW.csv[.gz] OUT.csv
"""
import csv
import gzip
import sys


def _open(path):
    return gzip.open(path, "rt") if path.endswith(".gz") else open(path)


def main():
    old, new, out = sys.argv[1:4]
    with _open(new) as fh:
        new_rows = list(csv.reader(fh))
    header, new_rows = new_rows[0], new_rows[1:]
    sigs = {r[0] for r in new_rows}
    with _open(old) as fh:
        old_rows = [r for r in list(csv.reader(fh))[1:] if r[0] not in sigs]
    with open(out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(header)
        w.writerows(old_rows + new_rows)
    print(f"{len(old_rows)} kept + {len(new_rows)} new rows ({len(sigs)} signatures replaced) -> {out}")


if __name__ == "__main__":
    main()
