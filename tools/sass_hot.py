#!/usr/bin/env python3
"""Per-instruction shared-memory wavefronts from an ncu SASS source page.

    ncu -i REP --page source --csv --print-source sass | gzip > X.csv.gz
    python tools/sass_hot.py X.csv.gz [--top 25]

Lists the shared-memory instructions by wavefronts (with the excess over the
ideal, i.e. bank conflicts) and the top stall-sampled instructions.
"""
from __future__ import annotations

import csv
import gzip
import io
import sys


def main(path, top=25):
    txt = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
    rows = list(csv.reader(io.StringIO(txt)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
    h = rows[hi]
    col = {k: h.index(k) for k in ("Address", "Source", "Instructions Executed", "L1 Wavefronts Shared",
                                    "L1 Wavefronts Shared Ideal", "L1 Wavefronts Shared Excessive",
                                    "Warp Stall Sampling (All Samples)")}
    recs = []
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        f = lambda k: float(r[col[k]].replace(",", "") or 0)  # noqa: E731
        recs.append((r[col["Source"]].strip(), f("Instructions Executed"), f("L1 Wavefronts Shared"),
                     f("L1 Wavefronts Shared Ideal"), f("L1 Wavefronts Shared Excessive"),
                     f("Warp Stall Sampling (All Samples)"), r[col["Address"]]))
    tw = sum(x[2] for x in recs)
    te = sum(x[4] for x in recs)
    ts = sum(x[5] for x in recs)
    print(f"shared wavefronts {tw:.3e}, excessive {te:.3e} ({100 * te / max(tw, 1):.1f} %), stall samples {ts:.0f}")
    print("\n## shared-memory instructions by excessive wavefronts")
    for s, ie, w, wi, we, st, a in sorted(recs, key=lambda x: -x[4])[:top]:
        if w <= 0:
            continue
        print(f"{a[-5:]} {s[:60]:60s} exec {ie:.2e} wf {w:.2e} ideal {wi:.2e} excess {we:.2e} ({w / max(ie, 1):.1f}/inst)")
    print("\n## top stall-sampled instructions")
    for s, ie, w, wi, we, st, a in sorted(recs, key=lambda x: -x[5])[:top]:
        print(f"{a[-5:]} {s[:60]:60s} samples {st:.0f} ({100 * st / max(ts, 1):.1f} %)")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
