"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) per kernel (dev aid)."""
import collections, csv, sys
def agg(path, top=14):
    rows = list(csv.reader(open(path)))
    hdr, out = None, collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        v = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1e-3) * v
        k = d["Kernel Name"][:70]
        out[k][0] += 1
        out[k][1] += v
    tot = sum(v[1] for v in out.values())
    print(f"{path}: total {tot/1e3:.2f} ms")
    for k, (c, t) in sorted(out.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{t/1e3:9.2f} ms {c:6d} x {t/c:9.1f} us  {k}")
if __name__ == "__main__":
    for p in sys.argv[1:]:
        agg(p)
