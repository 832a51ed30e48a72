"""Summarise ncu captures into profiles/ (tracked).

    python scripts/ncu_summarize.py --tag r1 --launches gpurun_out/launches.csv \
        edge_bwd=gpurun_out/prof_bwd.ncu-rep edge_fwd=gpurun_out/prof_fwd.ncu-rep

Writes profiles/ncu_summary.json (per kernel class: duration, DRAM bytes per
launch, SOL fractions, tensor-pipe activity, stall mix) and
profiles/<tag>_ncu.md (human-readable), plus profiles/<tag>_launches.md (share
of each kernel in the launch list of the bench command).
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
RAW = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_bytes": ("dram__bytes_read.sum", 1.0),
    "dram_write_bytes": ("dram__bytes_write.sum", 1.0),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "mem_throughput_pct": ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", 1.0),
    "issue_active_pct": ("sm__inst_issued.avg.pct_of_peak_sustained_active", 1.0),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "grid": ("launch__grid_size", 1.0),
    "block": ("launch__block_size", 1.0),
    "smem_dynamic_bytes": ("launch__shared_mem_per_block_dynamic", 1.0),
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1, "ns": 1, "usecond": 1e3,
        "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9, "s": 1e9}


def raw_metrics(rep: str) -> dict:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {"kernel": vals[hdr.index("Kernel Name")]}
    for key, (name, scale) in RAW.items():
        for i, h in enumerate(hdr):
            if h.endswith(name):
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                v *= UNIT.get(units[i], 1.0) if units[i] in UNIT else 1.0
                res[key] = v * scale if key == "duration_ms" else v
                break
    return res


def stall_mix(rep: str) -> dict:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO("\n".join(out.splitlines()[1:]))))
    hdr, data = rows[0], rows[1:]
    ix = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = collections.Counter()
    for r in data:
        for s in stalls:
            try:
                agg[s] += int(r[ix[s]] or 0)
            except ValueError:
                pass
    tot = sum(agg.values()) or 1
    return {k[6:]: round(v / tot, 3) for k, v in agg.most_common() if v / tot >= 0.01}


def launches(path: str) -> list:
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    hdr = rows[0]
    kn, mv, mu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    per = collections.OrderedDict()
    for r in rows[1:]:
        name = r[kn].split("(")[0].replace("void ", "").replace("hgnn_b200::", "")
        ns = float(r[mv].replace(",", "")) * UNIT.get(r[mu], 1.0)
        n, t = per.get(name, (0, 0.0))
        per[name] = (n + 1, t + ns)
    tot = sum(t for _, t in per.values()) or 1.0
    return [{"kernel": k, "launches": n, "total_ms": t / 1e6, "share": t / tot} for k, (n, t) in
            sorted(per.items(), key=lambda kv: -kv[1][1])]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--command", default="python bench.py --steps 2 --warmup 3 --profile")
    ap.add_argument("reps", nargs="*")
    a = ap.parse_args()
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    summ_path = prof / "ncu_summary.json"
    summ = json.load(open(summ_path)) if summ_path.exists() else {"kernels": {}}
    md = [f"# ncu captures, {a.tag}", "", f"Command: `{a.command}` under `ncu --set full --clock-control none "
          "--import-source on -k <kernel> -s <skip> -c 1` (one launch, cold-cache replay).", ""]
    for spec in a.reps:
        cls, rep = spec.split("=", 1)
        m = raw_metrics(rep)
        m["dram_bytes_per_launch"] = m.get("dram_read_bytes", 0) + m.get("dram_write_bytes", 0)
        m["stalls"] = stall_mix(rep)
        m["report"] = Path(rep).name
        m["tag"] = a.tag
        summ["kernels"][cls] = m
        md += [f"## {cls}: `{m['kernel']}`", ""]
        md += [f"- {k}: {v:.4g}" if isinstance(v, float) else f"- {k}: {v}" for k, v in m.items()
               if k not in ("kernel", "stalls")]
        md += [f"- stall mix (share of warp samples): {m['stalls']}", ""]
    summ["command"] = a.command
    json.dump(summ, open(summ_path, "w"), indent=1)
    (prof / f"{a.tag}_ncu.md").write_text("\n".join(md) + "\n")
    if a.launches:
        rows = launches(a.launches)
        lm = [f"# Launch list, {a.tag}", "", f"`ncu --metrics gpu__time_duration.sum --clock-control none` over "
              f"`{a.command}` (serialised, cold-cache per launch).", "",
              "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        lm += [f"| {r['kernel']} | {r['launches']} | {r['total_ms']:.3f} | {r['share']:.3f} |" for r in rows]
        (prof / f"{a.tag}_launches.md").write_text("\n".join(lm) + "\n")
        import shutil
        shutil.copy(a.launches, prof / f"{a.tag}_launches.csv")


if __name__ == "__main__":
    main()
