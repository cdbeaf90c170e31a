"""Summarise a REBK_TRACE dump of the split kernel's exchanges.

Stamps per (iteration, CTA): 0 exchange entry (products done), 1 cluster
scatter received, 2 LL slice polls done, 3 exchange exit, 4 first tile half
arrived, 5 first-half product done, 6 second half arrived, 7 second product
pass done (globaltimer ns).  Order within an iteration: 4 5 6 0 1 2 3 7.
Usage: python tools/trace_split.py rebk_trace.bin
"""
import sys

import numpy as np


def main(fn):
    with open(fn, "rb") as f:
        n, G, gsplit, CS = np.frombuffer(f.read(16), dtype=np.int32)
        t = np.frombuffer(f.read(), dtype=np.uint64).reshape(n, G, 8).astype(np.int64)
    ok = (t > 0).all(axis=(1, 2))
    t = t[ok]
    print(f"{t.shape[0]} iterations traced, G={G}, column CTAs={gsplit}, CS={CS}")
    for name, sl in (("column", slice(0, gsplit)), ("row", slice(gsplit, G))):
        g = t[:, sl, :]
        t0 = g[:, :, 0]
        first_in, last_in = t0.min(1), t0.max(1)
        out = g[:, :, 3]
        nc = g.shape[1] // CS
        cl = g.reshape(g.shape[0], nc, CS, 8)
        # per cluster: last entry -> scatter complete
        scat = (cl[:, :, :, 1].max(2) - cl[:, :, :, 0].max(2))
        # LL stage: last cluster's scatter done -> polls done (max over CTAs)
        ll = g[:, :, 2].max(1) - cl[:, :, :, 1].max(2).max(1)
        bc = g[:, :, 3].max(1) - g[:, :, 2].max(1)
        per_iter = np.diff(t0.min(1))
        pct = lambda a: f"p50 {np.median(a) / 1e3:6.3f}  mean {a.mean() / 1e3:6.3f}  p90 {np.percentile(a, 90) / 1e3:6.3f} us"
        print(f"[{name} group, {g.shape[1]} CTAs]")
        print("  iteration period       ", pct(per_iter))
        print("  entry spread (max-min) ", pct(last_in - first_in))
        print("  last entry -> first exit", pct(out.min(1) - last_in))
        print("  last entry -> last exit ", pct(out.max(1) - last_in))
        print("  scatter stage (per cl.) ", pct(scat.ravel()))
        print("  LL stage               ", pct(ll))
        print("  broadcast stage        ", pct(bc))
        # segments between stamps; for the last CTA to enter the exchange,
        # how much longer than the median CTA was each segment
        segs = {"prev exit->pass2 done": (3, 7, -1), "pass2 done->half A": (7, 4, 1), "half A->pass1a": (4, 5, 0),
                "pass1a->half B": (5, 6, 0), "half B->entry": (6, 0, 0)}
        last = t0[1:].argmax(1)
        rows = np.arange(last.size)
        for nm, (a, b, shift) in segs.items():
            if shift == -1:   # both stamps in the previous iteration
                d = g[:-1, :, b] - g[:-1, :, a]
            elif shift == 1:  # from the previous iteration's a to this iteration's b
                d = g[1:, :, b] - g[:-1, :, a]
            else:
                d = g[1:, :, b] - g[1:, :, a]
            med = np.median(d, axis=1)
            print(f"  seg {nm:24s} median {np.median(d) / 1e3:6.3f} us; last-arriver excess {np.mean(d[rows, last] - med) / 1e3:6.3f} us; spread p50 {np.median(d.max(1) - d.min(1)) / 1e3:6.3f}")
        # which CTA arrives last most often
        late = np.bincount(t0.argmax(1), minlength=g.shape[1])
        top = np.argsort(late)[::-1][:6]
        print("  most often last to arrive:", ", ".join(f"cta {sl.start + q} x{late[q]}" for q in top))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "rebk_trace.bin")
