"""Summarise a round's GPU evidence into profiles/ (run here, no GPU needed).

    python scripts/summarize_profiles.py r01

Reads gpurun_out/bench_<tag>.json, gpurun_out/launches_<tag>.csv and
gpurun_out/prof_<tag>.ncu-rep (via `ncu -i ... --page raw --csv`), writes
profiles/<tag>_summary.md, profiles/<tag>_launches.csv, profiles/<tag>_ncu_raw.csv,
profiles/<tag>_bench.json and profiles/traffic.json (per-launch DRAM bytes of
each kernel, read by bench.py's roofline["traffic"]).
"""

import collections
import csv
import io
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"
NAMES = {"k448_rows_fwd": "rows_fwd", "k448_cols": "cols", "k448_rows_inv": "rows_inv", "k448_colsinv": "cols",
         "k_select": "select", "k_rank": "rank", "k_splice16": "splice", "k_splice_ip": "splice", "k_splice_ip_bulk": "splice",
         "k_splice_plan": "splice_plan"}


def short(name):
    n = name.replace("void ", "").split("(")[0].split("<")[0]
    return NAMES.get(n, n)


def main(tag):
    PROF.mkdir(exist_ok=True)
    bench = json.loads((OUT / f"bench_{tag}.json").read_text())
    shutil.copy(OUT / f"bench_{tag}.json", PROF / f"{tag}_bench.json")
    # launch list
    rows = list(csv.reader(open(OUT / f"launches_{tag}.csv")))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    per = collections.defaultdict(list)
    with open(PROF / f"{tag}_launches.csv", "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["kernel", "duration_ns"])
        for r in data:
            if len(r) <= iv:
                continue
            v = float(r[iv].replace(",", ""))
            v *= {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(r[iu], 1)
            per[short(r[ik])].append(v)
            w.writerow([short(r[ik]), int(v)])
    tot = sum(sum(v) for v in per.values())
    # full capture
    raw = subprocess.run(["ncu", "-i", str(OUT / f"prof_{tag}.ncu-rep"), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    (PROF / f"{tag}_ncu_raw.csv").write_text(raw)
    rr = list(csv.reader(io.StringIO(raw)))
    rh, rd = rr[0], rr[2:]
    stalls = [h for h in rh if h.startswith("smsp__average_warps_issue_stalled")]

    def g(d, k):
        # "" for absent metrics; ncu writes "no data" / "n/a" for some counters
        v = d[rh.index(k)] if k in rh else ""
        if k == "Kernel Name":
            return v
        try:
            float(v)
        except ValueError:
            return ""
        return v

    traffic = {}
    lines = [f"# Round evidence `{tag}` (B200, sm_100a)", "",
             f"Bench (`python bench.py`, defaults): **{bench['value']:.0f} {bench['unit']}** "
             f"({bench['tokens_per_s'] / 1e6:.1f} M tokens/s), {bench['ms_per_step']:.3f} ms per step of "
             f"{bench['config']['streams_per_gpu']} streams; step roofline "
             f"{100 * bench['roofline_step']['frac']:.1f} % of {bench['roofline_step']['peak']} GB/s "
             f"(select {bench['roofline_step']['select_bytes']} B + splice {bench['roofline_step']['splice_bytes']} B per frame); "
             f"clocks {bench['clocks']}.",
             f"e2e (pinned host frames, H2D {bench['e2e']['h2d_bytes_per_step'] / 1e9:.2f} GB/step): "
             f"{bench['e2e']['value']:.0f} frames/s"
             + (f" (frames as P6 uint8 payloads: {bench['e2e_u8']['value']:.0f} frames/s)" if "e2e_u8" in bench else "")
             + f".  CPU baseline ({bench['cpu_baseline']['kind']}, "
             f"{bench['cpu_baseline']['cores']} cores): {bench['cpu_baseline']['value']:.0f} frames/s.", "",
             "## Launch list (ncu `gpu__time_duration.sum`, serialised, cold cache)", "",
             "| kernel | launches | mean us | share |", "|---|---|---|---|"]
    for k, v in sorted(per.items(), key=lambda x: -sum(x[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f} % |")
    lines += ["", "## Full capture (`--set full`), one launch per kernel at the bench configuration", "",
              "| kernel | us | DRAM read MB | DRAM write MB | warp-inst (M) | issue active % | warps active % | FMA pipe % | FP64 pipe % | tensor pipe % | top stalls |",
              "|---|---|---|---|---|---|---|---|---|---|---|"]
    for d in rd:
        k = short(g(d, "Kernel Name"))
        rdb = float(g(d, "dram__bytes_read.sum") or 0)
        wrb = float(g(d, "dram__bytes_write.sum") or 0)
        units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rdb *= units.get(rr[1][rh.index("dram__bytes_read.sum")], 1)
        wrb *= units.get(rr[1][rh.index("dram__bytes_write.sum")], 1)
        scale = 1
        traffic.setdefault(k, []).append(rdb + wrb)
        st = sorted(((h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                      float(g(d, h) or 0)) for h in stalls), key=lambda x: -x[1])[:3]
        tu = rr[1][rh.index("gpu__time_duration.sum")]
        tscale = {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(tu, 1)
        lines.append(f"| {k} | {float(g(d, 'gpu__time_duration.sum')) * tscale:.1f} | {rdb * scale / 1e6:.1f} | "
                     f"{wrb * scale / 1e6:.1f} | {float(g(d, 'smsp__inst_executed.sum')) / 1e6:.2f} | "
                     f"{float(g(d, 'smsp__issue_active.avg.pct_of_peak_sustained_active')):.1f} | "
                     f"{float(g(d, 'sm__warps_active.avg.pct_of_peak_sustained_active')):.1f} | "
                     f"{float(g(d, 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active') or 0):.1f} | "
                     f"{float(g(d, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active') or 0):.1f} | "
                     f"{float(g(d, 'TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed') or 0):.1f} | "
                     + ", ".join(f"{h} {v:.2f}" for h, v in st) + " |")
    lines += ["", "## Per-kernel timing inside bench.py (CUDA events, serialised pass)", "",
              "| kernel | ms | share | interface bytes | GB/s |", "|---|---|---|---|---|"]
    for k, v in bench["kernels"].items():
        lines.append(f"| {k} | {v['ms']:.3f} | {100 * v['share']:.1f} % | {v['bytes'] / 1e6:.0f} MB | {v['gbs']:.0f} |")
    (PROF / f"{tag}_summary.md").write_text("\n".join(lines) + "\n")
    # per-launch DRAM bytes (mean over the captured launches); the bench's
    # "splice" timing covers the plan kernel and the copy kernel together
    traffic = {k: sum(v) / len(v) for k, v in traffic.items()}
    if "splice_plan" in traffic and "splice" in traffic:
        traffic["splice"] += traffic.pop("splice_plan")
    (PROF / "traffic.json").write_text(json.dumps(
        {"capture": f"{tag} (profiles/{tag}_ncu_raw.csv): dram__bytes_read.sum + dram__bytes_write.sum per launch",
         "kernels": traffic}, indent=1))
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
