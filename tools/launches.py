"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys


def summarize(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                name = d["Kernel Name"].split("(")[0]
                agg[name].append(float(d["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append((k, len(v), sum(v) / len(v), sum(v) / tot))
    return out, tot


if __name__ == "__main__":
    res, tot = summarize(sys.argv[1])
    print(f"total {tot/1e3:.1f} us over {sum(r[1] for r in res)} launches")
    for k, cnt, avg, share in res:
        print(f"{share*100:5.1f}%  n={cnt:4d}  avg={avg/1e3:9.2f} us  {k}")
