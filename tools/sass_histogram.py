"""SASS opcode histogram of one kernel of libslm_b200.so (cuobjdump -sass): the
evidence that the product kernels use TMA bulk copies (UBLKCP / UBLKPF), mbarrier
waits (SYNCS), packed FP32 (FFMA2 / FMUL2 / FADD2) and vector reductions.

    python tools/sass_histogram.py <mangled-or-substring> [out.md]
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2504_12905_b200", "libslm_b200.so")


def main():
    want = sys.argv[1]
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", out)
    hits = [f for f in funcs[1:] if want in f.splitlines()[0]]
    if not hits:
        raise SystemExit(f"no function matching {want}")
    name = hits[0].splitlines()[0].strip()
    ops = collections.Counter()
    for line in hits[0].splitlines():
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if m:
            ops[m.group(1).split(".")[0]] += 1
    total = sum(ops.values())
    lines = [f"# SASS opcode histogram: `{name}`\n", f"{total} instructions (static count, cuobjdump -sass of "
             f"libslm_b200.so, sm_100a)\n", "| opcode | count |", "|---|---|"]
    for op, n in ops.most_common():
        lines.append(f"| {op} | {n} |")
    text = "\n".join(lines) + "\n"
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(text)
    print(text[:1500])


if __name__ == "__main__":
    main()
