#!/usr/bin/env python
"""Turn an .ncu-rep (ncu --set full --import-source on) into the text summary kept under profiles/.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/ncu_<name>.md [--top 12]

Runs here (no GPU): `ncu -i ... --page raw --csv` for the per-launch metrics and `--page source --csv`
for the per-instruction stall samples of every profiled launch.
"""
import csv
import io
import subprocess
import sys

RAW = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("lts__t_sectors.sum", "L2 sectors"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1/TEX throughput"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy"),
    ("sm__inst_executed.avg.per_cycle_elapsed", "IPC (per SM)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe busy"),
]


def ncu(args):
    out = subprocess.run(["ncu", *args], capture_output=True, text=True).stdout
    return [ln for ln in out.splitlines() if not ln.startswith("==")]


def main():
    rep, dst = sys.argv[1], sys.argv[2]
    top_n = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 12
    rows = list(csv.reader(io.StringIO("\n".join(ncu(["-i", rep, "--page", "raw", "--csv"])))))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu summary of `{rep.split('/')[-1]}`", "",
             "Source: `ncu --set full --clock-control none --import-source on` on one B200 (cold-cache, serialised "
             "replays: compare shares, not absolutes). Extracted here with `scripts/ncu_summary.py`.", ""]
    lines.append("## Per-launch metrics")
    lines.append("")
    lines.append("| # | kernel | " + " | ".join(lbl for key, lbl in RAW if key in col) + " |")
    lines.append("|---|---|" + "---|" * sum(1 for key, _ in RAW if key in col))
    for i, d in enumerate(data):
        cells = []
        for key, _ in RAW:
            if key not in col:
                continue
            v, u = d[col[key]], units[col[key]]
            try:
                f = float(v.replace(",", ""))
                v = f"{f:.3f}".rstrip("0").rstrip(".") if abs(f) < 1e6 else f"{f:.4g}"
            except ValueError:
                pass
            cells.append(f"{v} {u}".strip())
        name = d[col["Kernel Name"]].replace("|", "/")
        lines.append(f"| {i} | `{name[:70]}` | " + " | ".join(cells) + " |")
    lines.append("")
    # source pages, one per launch
    lines.append("## Warp-stall samples per SASS instruction (top lines per launch)")
    for i, d in enumerate(data):
        src = ncu(["-i", rep, "--page", "source", "--csv", "--launch-skip", str(i), "--launch-count", "1"])
        srows = list(csv.reader(io.StringIO("\n".join(src))))
        shdr, recs = None, []
        for r in srows:
            if r and r[0] == "Address":
                if shdr is not None:
                    break  # the page repeats per view; the first is enough
                shdr = r
                continue
            if shdr and len(r) == len(shdr):
                recs.append(dict(zip(shdr, r)))
        if not recs:
            continue
        stalls = [k for k in shdr if k.startswith("stall_") and "Not Issued" not in k]
        tot = sum(int(x["# Samples"] or 0) for x in recs)
        agg = sorted(((k, sum(int(x[k] or 0) for x in recs)) for k in stalls), key=lambda kv: -kv[1])
        lines.append("")
        lines.append(f"### launch {i}: `{d[col['Kernel Name']][:70]}` -- {tot} samples, {len(recs)} SASS instructions")
        lines.append("")
        lines.append("stall mix: " + ", ".join(f"{k[6:]} {100.0 * v / max(1, tot):.1f}%" for k, v in agg[:6]))
        lines.append("")
        lines.append("| samples | share | SASS | executed (warp) | dominant stall |")
        lines.append("|---|---|---|---|---|")
        for x in sorted(recs, key=lambda x: -int(x["# Samples"] or 0))[:top_n]:
            s = int(x["# Samples"] or 0)
            dom = max(stalls, key=lambda k: int(x[k] or 0))
            lines.append(f"| {s} | {100.0 * s / max(1, tot):.1f}% | `{x['Source'].strip()[:80]}` | "
                         f"{x['Instructions Executed']} | {dom[6:]} |")
    with open(dst, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("wrote", dst)


if __name__ == "__main__":
    main()
