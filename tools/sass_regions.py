"""Per-region totals of an ncu source-page CSV (--page source --csv --print-source sass):
instructions executed, shared-memory wavefronts and stall samples for every loop body
(backward-branch target .. branch) and the code between loops."""
import csv
import re
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    recs = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        recs.append(r)
    base = int(recs[0][col["Address"]], 16)
    insts = []
    for r in recs:
        off = int(r[col["Address"]], 16) - base
        src = r[col["Source"]].strip()
        ie = float(r[col["Instructions Executed"]] or 0)
        wf = float(r[col["L1 Wavefronts Shared"]] or 0)
        st = float(r[col["Warp Stall Sampling (All Samples)"]] or 0)
        insts.append((off, src, ie, wf, st))
    # loops: backward branches
    loops = []
    for off, src, *_ in insts:
        m = re.search(r"BRA(?:\.\w+)* (0x[0-9a-f]+)", src)
        if m:
            tgt = int(m.group(1), 16)
            tgt = tgt - base if tgt >= base else tgt
            if tgt < off:
                loops.append((tgt, off))
    tot_i = sum(x[2] for x in insts)
    tot_w = sum(x[3] for x in insts)
    tot_s = sum(x[4] for x in insts)
    print(f"total: inst {tot_i:.4g}  shared wavefronts {tot_w:.4g}  stall samples {tot_s:.4g}")
    for lo, hi in sorted(set(loops)):
        sel = [x for x in insts if lo <= x[0] <= hi]
        i = sum(x[2] for x in sel)
        w = sum(x[3] for x in sel)
        s = sum(x[4] for x in sel)
        if i / tot_i < 0.01:
            continue
        n = len(sel)
        iters = max(x[2] for x in sel)
        print(f"loop {lo:#06x}-{hi:#06x} ({n:3d} instr, ~{iters:.3g} iters): inst {100 * i / tot_i:5.1f}%  "
              f"wavefronts {100 * w / tot_w:5.1f}%  stalls {100 * s / tot_s:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
