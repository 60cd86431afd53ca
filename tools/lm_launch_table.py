"""Per-launch table of the last LM step in an ncu launch-list CSV (gpu__time_duration.sum, launch__grid_size)."""
import csv
import sys


def main(path, n=60, start_kernel="k_prepare"):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    launch = {}
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        d = launch.setdefault(r[ii], {"name": r[ki]})
        d[r[mi]] = r[vi]
    L = [launch[k] for k in sorted(launch, key=int)]
    idx = [i for i, l in enumerate(L) if start_kernel in l["name"]]
    s = idx[-2]
    for l in L[s:s + n]:
        nm = l["name"].split("(")[0].replace("void ", "")
        t = float(l["gpu__time_duration.sum"].replace(",", "")) / 1e3
        print(f"{nm[:45]:45s} grid {l.get('launch__grid_size'):>8s} {t:9.1f} us")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 60)
