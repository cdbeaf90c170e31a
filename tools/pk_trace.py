"""Summarise a REBK_PK_TRACE dump of the persistent multi-RHS kernel
(globaltimer stamps [iteration][CTA][8]; see pk_stamp in rebk_mrhs_tc.cu).
usage: python tools/pk_trace.py pk_trace.bin G"""
import sys

import numpy as np


def main(fn, G):
    t = np.fromfile(fn, dtype=np.uint64).astype(np.float64).reshape(-1, G, 16)
    n = t.shape[0]
    rows = []
    sub = []
    for k in range(n - 1):
        a, b = t[k], t[k + 1]
        if not (a[:, :6].all() and b[:, 7].all()):
            continue
        rows.append([
            np.median(a[:, 0] - a[:, 7]),        # phase A work (producer start -> epilogue done)
            np.max(a[:, 0] - a[:, 7]),
            np.median(a[:, 1]) - a[:, 0].max(),  # barrier A (last arrival -> median release)
            np.median(a[:, 2] - a[:, 1]),        # U reduction (+check)
            np.median(a[:, 6]) - a[:, 2].max(),  # barrier B
            np.median(a[:, 3] - a[:, 6]),        # phase C work
            np.max(a[:, 3] - a[:, 6]),
            np.median(a[:, 4]) - a[:, 3].max(),  # barrier C
            np.median(a[:, 5] - a[:, 4]),        # R reduction
            np.median(b[:, 7]) - a[:, 5].max(),  # barrier D
            np.median(b[:, 7] - a[:, 7]),        # iteration period
        ])
        sub.append([np.median(a[:, 8] - a[:, 0]), np.median(a[:, 9] - a[:, 1]), np.median(a[:, 9] - a[:, 8]),
                    np.median(a[:, 10] - a[:, 3]), np.median(a[:, 11] - a[:, 4]), np.median(a[:, 11] - a[:, 10])])
    r = np.median(np.array(rows), axis=0) / 1e3
    rs = np.median(np.array(sub), axis=0) / 1e3
    names = ["A work med", "A work max", "bar A", "B reduce", "bar B", "C work med", "C work max", "bar C",
             "D reduce", "bar D", "period"]
    print(f"{len(rows)} iterations, G={G} (microseconds, medians over iterations)")
    for nm, v in zip(names, r):
        print(f"  {nm:12s} {v:8.2f}")
    for nm, v in zip(["A: arrive cost (fence+red)", "B: poll -> all 320 at barrier", "B: own arrival -> barrier",
                      "C: arrive cost", "D: poll -> barrier", "D: own arrival -> barrier"], rs):
        print(f"    {nm:32s} {v:8.2f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
