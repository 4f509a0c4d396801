#!/usr/bin/env python
"""Attribute ncu source-page (SASS) warp-stall samples to source lines.

  python scripts/ncu_regions.py <src.csv> <nvdisasm -g listing> [bucket]
The listing comes from `nvdisasm -g -c -fun <section index> <cubin>` of the same build.
"""
import collections
import csv
import re
import sys


def line_map(path):
    cur, m = None, {}
    inl = None
    for ln in open(path):
        if "//##" in ln:
            # outermost fused.cuh frame of the inline chain (the kernel-level source line)
            frames = re.findall(r'"([^"]+)", line (\d+)', ln)
            fr = [(f.split("/")[-1], int(n)) for f, n in frames]
            kern = [x for x in fr if x[0] == "fused.cuh"]
            if fr:
                cur = kern[-1] if kern else fr[-1]
            continue
        mm = re.search(r"/\*([0-9a-f]{4,6})\*/\s+[@A-Z]", ln)
        if mm:
            m[int(mm.group(1), 16)] = cur
    return m


def main():
    src, lst = sys.argv[1], sys.argv[2]
    bucket = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    lm = line_map(lst)
    rows = list(csv.reader(open(src)))
    hdr = rows[1]
    ia = hdr.index("Address")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    isamp = hdr.index("Warp Stall Sampling (All Samples)")
    base = None
    agg = collections.defaultdict(lambda: collections.Counter())
    tot = 0
    for r in rows[2:]:
        if len(r) <= ia or not r[ia].startswith("0x"):
            continue
        a = int(r[ia], 16)
        if base is None:
            base = a
        off = a - base
        key = lm.get(off, ("?", 0))
        if key[0] == "fused.cuh":
            key = (key[0], key[1] // bucket * bucket)
        else:
            key = (key[0], 0)
        s = int(r[isamp] or 0)
        tot += s
        agg[key]["samples"] += s
        for i in stall_cols:
            v = int(r[i] or 0)
            if v:
                agg[key][hdr[i][6:]] += v
    print("total samples", tot)
    for k, c in sorted(agg.items(), key=lambda x: -x[1]["samples"])[:45]:
        top = ", ".join(f"{n}={v}" for n, v in c.most_common(6) if n != "samples")
        print(f"{k[0]}:{k[1]:<5} {c['samples']:6d} {100.0 * c['samples'] / max(tot, 1):5.1f}%  {top}")


if __name__ == "__main__":
    main()
