"""Summarise an ncu report (and optional launch-list CSV) into profiles/.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [--launches gpurun_out/launches.csv] --out profiles/r1_x
Writes <out>.md (human summary) and <out>.json (metrics per kernel)."""
import argparse
import collections
import csv
import io
import json
import subprocess

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio",
    "smsp__inst_executed.sum",
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--launches", default=None)
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for row in rows[2:]:
        k = {"kernel": row[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                k[m] = {"value": row[i], "unit": units[i]}
        kernels.append(k)
    launches = None
    if a.launches:
        agg = collections.OrderedDict()
        with open(a.launches) as f:
            lines = [l for l in f if l.startswith('"')]
        for r in csv.DictReader(io.StringIO("".join(lines))):
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = r["Kernel Name"].split("(")[0].replace("void ", "")
            v = float(r["Metric Value"])
            scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(r["Metric Unit"], 1.0)
            e = agg.setdefault(name, [0, 0.0])
            e[0] += 1
            e[1] += v * scale
        tot = sum(v[1] for v in agg.values())
        launches = [{"kernel": k, "launches": n, "total_ms": t, "share": t / tot if tot else 0.0}
                    for k, (n, t) in agg.items()]
    with open(a.out + ".json", "w") as f:
        json.dump({"report": a.report, "note": a.note, "kernels": kernels, "launch_list": launches}, f, indent=1)
    with open(a.out + ".md", "w") as f:
        f.write(f"# ncu summary: {a.report}\n\n{a.note}\n\n")
        for k in kernels:
            f.write(f"## {k['kernel'][:100]}\n\n| metric | value |\n|---|---|\n")
            for m in METRICS:
                if m in k:
                    f.write(f"| {m} | {k[m]['value']} {k[m]['unit']} |\n")
            f.write("\n")
        if launches:
            f.write("## launch list (cold-cache, serialised: compare shares)\n\n| kernel | launches | total ms | share |\n|---|---|---|---|\n")
            for l in sorted(launches, key=lambda x: -x["total_ms"]):
                f.write(f"| {l['kernel']} | {l['launches']} | {l['total_ms']:.3f} | {l['share']*100:.1f}% |\n")
    print(open(a.out + ".md").read())


if __name__ == "__main__":
    main()
