#!/usr/bin/env python
"""SASS instruction census of selected libpi kernels (cuobjdump -sass of the build objects): the
mnemonics that show which hardware paths a kernel uses (TMA bulk copies and prefetches, mbarriers,
tensor-core MMAs, TMEM loads, global atomics)."""
import collections
import re
import subprocess
import sys

OPS = ("UBLKCP", "UBLKPF", "SYNCS", "UTCHMMA", "UTCBAR", "LDTM", "HMMA", "LDGSTS", "ATOMG", "ATOMS", "RED.", "REDUX", "LDS.128",
       "FFMA", "BAR.SYNC", "SHFL")
UNITS = {
    "fused bf16 B=1 ReLU (k_layer: default / GRP / SPEC / Q4)": "fused_inst_bf16_b1_relu.cu.o",
    "fused bf16 B=2 ReGLU (shared-memory x)": "fused_inst_bf16_b2_reglu.cu.o",
    "per-step + batched tensor-core (bf16)": "steps_inst_bf16.cu.o",
}
PICK = re.compile(sys.argv[1]) if len(sys.argv) > 1 else None


def census(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    fn, rows = None, collections.OrderedDict()
    for ln in out.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            fn = m.group(1)
            rows[fn] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", ln)
        if fn and m:
            op = m.group(1)
            rows[fn]["_total"] += 1
            for k in OPS:
                if op.startswith(k):
                    rows[fn][k] += 1
    return rows


print(__doc__.strip().replace("\n", " "))
for title, obj in UNITS.items():
    path = "paper_2312_12456_b200/build/" + obj
    print(f"\n== {title}: {path}")
    for fn, c in census(path).items():
        if "k_layer" in fn and not re.search(r"Li(4|3)ELi1E", fn):   # the c3/c4 shapes only
            continue
        print(f"  {fn}  ({c['_total']} instructions)")
        print("    " + ", ".join(f"{k} x{c[k]}" for k in OPS if c[k]))
