#!/usr/bin/env python3
"""Per-instruction warp-stall samples from an ncu report's source page (SASS).

usage: tools/ncu_stalls.py REPORT.ncu-rep KERNEL_REGEX [TOP]
Prints the stall-reason totals and the top stalled instructions.
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          f"regex:{kre}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    num = lambda v: int(v) if v.strip().lstrip("-").isdigit() else 0
    i_s, i_src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    reasons = [h for h in hdr if h.startswith("stall_") and "(Not Issued)" not in h]
    tot = sum(num(r[i_s]) for r in data)
    print(f"{rows[0][1][:100]}\ntotal samples {tot}")
    agg = {h: sum(num(r[hdr.index(h)]) for r in data) for h in reasons}
    for h, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]:
        print(f"  {h:24s} {v:8d} {100.0 * v / max(tot, 1):5.1f}%")
    for r in sorted(data, key=lambda r: -num(r[i_s]))[:top]:
        why = sorted(((num(r[hdr.index(h)]), h) for h in reasons), reverse=True)[:2]
        print(f"  {r[0][-5:]} {r[i_src].strip()[:48]:48s} {num(r[i_s]):6d}  " + " ".join(f"{h[6:]}={v}" for v, h in why if v))


if __name__ == "__main__":
    main()
