#!/usr/bin/env python3
"""Static schedule of a kernel's loops from its SASS control bits.

ptxas encodes, per instruction, the cycles to stall before the next one
(fixed-latency pipes: DADD / DMUL / IMAD ... use stall counts, not
scoreboards) plus the scoreboard waits of variable-latency results (LDS,
LDG, ...).  Summing the stall counts over a loop body gives the cycles the
warp spends issuing one iteration when no scoreboard wait blocks it -- the
lower bound ptxas itself planned.  Used to iterate on the exact-mode chain
and A.D kernels on the CPU before measuring them.

usage: tools/sass_sched.py LIB.so FUNCTION_SUBSTRING [--dump]
"""
import re
import subprocess
import sys


def parse(so, fn_sub):
    txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", txt)
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        if fn_sub not in name:
            continue
        lines = f.splitlines()
        ins = []
        for i, l in enumerate(lines):
            m = re.match(r"\s*/\*([0-9a-f]{4,5})\*/\s+(.*?);\s*/\* (0x[0-9a-f]+) \*/", l)
            if m and i + 1 < len(lines):
                m2 = re.match(r"\s*/\* (0x[0-9a-f]+) \*/", lines[i + 1])
                if m2:
                    hi = int(m2.group(1), 16)
                    ctrl = hi >> 41
                    ins.append({"addr": int(m.group(1), 16), "op": m.group(2).strip(), "stall": ctrl & 0xF,
                                "yield": (ctrl >> 4) & 1, "wb": (ctrl >> 5) & 7, "rb": (ctrl >> 8) & 7,
                                "wait": (ctrl >> 11) & 0x3F})
        yield name, ins


def loops(ins):
    """(start, end) index pairs of backward branches (innermost first by size)."""
    by_addr = {x["addr"]: i for i, x in enumerate(ins)}
    out = []
    for i, x in enumerate(ins):
        m = re.search(r"BRA\S*\s+(?:!?U?P\d+,\s*)?(0x[0-9a-f]+)", x["op"])
        if m:
            tgt = int(m.group(1), 16)
            if tgt < x["addr"] and tgt in by_addr:
                out.append((by_addr[tgt], i))
    return sorted(out, key=lambda p: p[1] - p[0])


def straight_runs(body):
    """Split a loop body at branches / barrier waits: the straight-line runs."""
    runs, cur = [], []
    for x in body:
        cur.append(x)
        if "BRA" in x["op"] or "SYNCS" in x["op"]:
            runs.append(cur)
            cur = []
    runs.append(cur)
    return runs


def summary(run):
    cyc = sum(max(1, x["stall"]) for x in run)
    cnt = lambda k: sum(1 for x in run if re.sub(r"^@!?U?P\d+\s+", "", x["op"]).startswith(k))
    return cyc, cnt("DADD"), cnt("DMUL"), cnt("DFMA"), cnt("LDS"), sum(1 for x in run if x["wait"])


def main():
    so, fn = sys.argv[1], sys.argv[2]
    dump = "--dump" in sys.argv
    for name, ins in parse(so, fn):
        print(name)
        seen = set()
        for (a, b) in loops(ins):
            body = ins[a:b + 1]
            best = max(straight_runs(body), key=lambda r: summary(r)[1] + summary(r)[3])
            key = (best[0]["addr"], best[-1]["addr"])
            cyc, nd, nm, nf, nl, nw = summary(best)
            if nd + nf == 0 or key in seen:
                continue
            seen.add(key)
            print(f"  run {best[0]['addr']:#06x}-{best[-1]['addr']:#06x} (loop {ins[a]['addr']:#x}-{ins[b]['addr']:#x}): "
                  f"{len(best)} instr, {cyc} stall-cycles, DADD {nd} DMUL {nm} DFMA {nf} LDS {nl}, "
                  f"scoreboard waits {nw}, {cyc / max(nd + nf, 1):.2f} cycles per DADD/DFMA")
            if dump:
                for x in best:
                    print(f"    {x['addr']:05x} {x['op'][:60]:60s} s={x['stall']:2d} wb={x['wb']} rb={x['rb']} "
                          f"w={x['wait']:06b}")


if __name__ == "__main__":
    main()


def load_use(run):
    """For every LDS / LDG in a straight run: static cycles until the first
    instruction that waits on its write barrier (the load-to-use distance
    ptxas planned; shared loads take ~30 cycles, so shorter distances stall)."""
    out = []
    for i, x in enumerate(run):
        op = re.sub(r"^@!?U?P\d+\s+", "", x["op"])
        if not (op.startswith("LDS") or op.startswith("LDG")) or x["wb"] == 7:
            continue
        cyc = 0
        for y in run[i + 1:]:
            cyc += max(1, run[run.index(y) - 1]["stall"]) if False else 0
        # cycles = sum of stalls from this instruction up to the waiter
        c = 0
        for j in range(i, len(run) - 1):
            c += max(1, run[j]["stall"])
            if run[j + 1]["wait"] & (1 << x["wb"]):
                out.append((x["addr"], op[:30], c))
                break
    return out
