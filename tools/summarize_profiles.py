"""Summarise gpurun_out/ profiling artefacts into profiles/ (tracked).

    python tools/summarize_profiles.py <tag> --launches gpurun_out/launches_bench.csv \
        --ncu gpurun_out/raster_full.ncu-rep --bench gpurun_out/bench_r1.json

Writes profiles/<tag>_launches.md (per-kernel share of the bench command's
launch list — ncu's per-launch times are cold-cache and serialised, so the
SHARES are what matter), profiles/<tag>_ncu_<kernel>.md (key metrics of the
full capture, incl. dram__bytes_read/write = the roofline `traffic`), and
copies the bench JSON line.
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles")

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum",
        "launch__registers_per_thread", "launch__shared_mem_per_block_static", "launch__grid_size",
        "launch__block_size", "lts__t_sector_hit_rate.pct", "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct"]


def launches(path, tag):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v = v / 1e6 if r[ui] == "ns" else v / 1e3 if r[ui] == "us" else v
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(ms for _, ms in agg.values())
    lines = [f"# {tag}: launch list of the bench command (ncu --metrics gpu__time_duration.sum "
             f"--clock-control none)\n", "ncu serialises and cold-starts every launch: compare shares, not absolutes.\n",
             "| kernel | launches | total ms | avg ms | share |", "|---|---|---|---|---|"]
    for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {n} | {ms:.3f} | {ms / n:.4f} | {100 * ms / tot:.1f}% |")
    lines.append(f"| **total** | {sum(n for n, _ in agg.values())} | {tot:.3f} | | |")
    with open(os.path.join(OUT, f"{tag}_launches.md"), "w") as f:
        f.write("\n".join(lines) + "\n")


def ncu_full(path, tag):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        stalls = []
        for i, c in enumerate(h):
            if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued"):
                try:
                    stalls.append((float(r[i].replace(",", "")), c.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        lines = [f"# {tag}: ncu --set full, `{name}`\n", "| metric | value | unit |", "|---|---|---|"]
        try:
            dur = float(r[h.index("gpu__time_duration.sum")].replace(",", ""))
            dscale = {"ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}.get(
                u[h.index("gpu__time_duration.sum")], 1e-3)
            bytes_ = sum(float(r[h.index(k)].replace(",", "")) * SCALE[u[h.index(k)]]
                         for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            lines.append(f"| achieved DRAM GB/s (read+write / duration) | {bytes_ / (dur * dscale) / 1e9:.1f} | GB/s |")
        except (ValueError, KeyError):
            pass
        for k in KEYS:
            if k in h:
                lines.append(f"| {k} | {r[h.index(k)]} | {u[h.index(k)]} |")
        lines.append("\nTop stall reasons (pc sampling): " +
                     ", ".join(f"{c} {100 * v / tot:.0f}%" for v, c in sorted(stalls, reverse=True)[:8]))
        rd = float(r[h.index("dram__bytes_read.sum")].replace(",", "")) * SCALE[u[h.index("dram__bytes_read.sum")]]
        wr = float(r[h.index("dram__bytes_write.sum")].replace(",", "")) * SCALE[u[h.index("dram__bytes_write.sum")]]
        tj = os.path.join(OUT, "traffic.json")
        traffic = json.load(open(tj)) if os.path.exists(tj) else {}
        traffic[name] = {"bytes_per_launch": rd + wr, "read": rd, "write": wr, "source": f"{tag} ncu --set full"}
        with open(tj, "w") as f:
            json.dump(traffic, f, indent=1)
        safe = name.replace("slm::", "").replace("<", "_").replace(">", "").replace(" ", "")
        with open(os.path.join(OUT, f"{tag}_ncu_{safe}.md"), "w") as f:
            f.write("\n".join(lines) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--launches")
    ap.add_argument("--ncu", nargs="*", default=[])
    ap.add_argument("--bench")
    a = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    if a.launches:
        launches(a.launches, a.tag)
    for p in a.ncu:
        ncu_full(p, a.tag)
    if a.bench:
        line = [ln for ln in open(a.bench).read().splitlines() if ln.startswith("{")][-1]
        with open(os.path.join(OUT, f"{a.tag}_bench.json"), "w") as f:
            f.write(json.dumps(json.loads(line), indent=1) + "\n")


if __name__ == "__main__":
    main()
