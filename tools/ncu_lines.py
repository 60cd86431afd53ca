"""Per-source-line instruction / stall breakdown of an ncu report (runs anywhere ncu is).

    python tools/ncu_lines.py gpurun_out/raster.ncu-rep [--top 40] [--ranges a-b:name,...]
"""
import argparse
import csv
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--file", default="raster.cu")
    ap.add_argument("--ranges", default="")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    f = None
    data = []
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No") or r[0] == "":
            continue
        try:
            data.append((int(r[7]), int(r[4]), f, int(r[0]), int(r[8]), r[1][:90]))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1
    ts = sum(d[1] for d in data) or 1
    print(f"total warp inst {tot/1e6:.1f}M, stall samples {ts}")
    if a.ranges:
        secs = {}
        for item in a.ranges.split(","):
            rng, name = item.split(":")
            lo, hi = rng.split("-")
            secs[name] = (int(lo), int(hi))
        agg = {}
        for d in data:
            key = d[2]
            if d[2] == a.file:
                key = "other"
                for k, (lo, hi) in secs.items():
                    if lo <= d[3] <= hi:
                        key = k
            x = agg.setdefault(key, [0, 0, 0])
            x[0] += d[0]
            x[1] += d[4]
            x[2] += d[1]
        for k, v in sorted(agg.items(), key=lambda x: -x[1][0]):
            print(f"{k:22s} {v[0]/tot*100:5.1f}% inst {v[2]/ts*100:5.1f}% stall  thr/inst {v[1]/max(v[0],1):5.1f}  {v[0]/1e6:.0f}M")
    for d in sorted(data, key=lambda x: -x[0])[: a.top]:
        print(f"{d[0]/tot*100:5.1f}% {d[1]/ts*100:5.1f}%st thr {d[4]/max(d[0],1):4.1f} {d[2]}:{d[3]}: {d[5]}")


if __name__ == "__main__":
    main()
