"""Summarise gpurun_out/ ncu artefacts into profiles/<round>/ (committed).

  python tools/ncu_summarize.py round1
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_sector_hit_rate.pct"]


def raw(rep: str) -> list[dict]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        d["_units"] = dict(zip(hdr, units))
        out.append(d)
    return out


def num(v: str):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return v


def main(tag: str) -> None:
    dst = os.path.join(ROOT, "profiles", tag)
    os.makedirs(dst, exist_ok=True)
    summary = {}
    md = [f"# ncu summaries ({tag})\n",
          "Captured with `tools/profile_round.sh` under gpurun on one B200 "
          "(`ncu --set full --clock-control none`); numbers per launch.\n"]
    for name in ("ncu_gemm_ring", "ncu_k7_decode", "ncu_k7_decode_q1", "ncu_k6_prefill",
                 "ncu_k10_cluster", "ncu_k11_pair", "ncu_cublas_gu4096"):
        rep = os.path.join(OUT, name + ".ncu-rep")
        if not os.path.exists(rep):
            continue
        rows = raw(rep)
        md.append(f"\n## {name}\n")
        md.append("| kernel | " + " | ".join(k.split(".")[0].replace("__", ".") + "." +
                                             ".".join(k.split(".")[1:]) for k in KEYS) + " |")
        md.append("|" + "---|" * (len(KEYS) + 1))
        keep = []
        for r in rows:
            kname = r.get("Kernel Name", r.get("Function Name", "?"))[:60]
            vals = {k: f"{r.get(k, '')} {r['_units'].get(k, '')}".strip() for k in KEYS}
            keep.append({"kernel": kname, **vals})
            md.append(f"| {kname} | " + " | ".join(str(vals[k]) for k in KEYS) + " |")
        summary[name] = keep
        with open(os.path.join(dst, name + "_raw.csv"), "w") as fh:
            txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                 capture_output=True, text=True).stdout
            fh.write(txt)
    # launch lists -> per-kernel share of GPU time in the bench step
    for lname, title in (("launches.csv", "bench.py --steps 1 (C2), steady state"),
                         ("launches_c5.csv", "bench.py --workload c5 --steps 1 (256 sessions, "
                                             "batched plans)")):
        lpath = os.path.join(OUT, lname)
        if not os.path.exists(lpath):
            continue
        lines = open(lpath).read().splitlines()
        start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
        rd = csv.DictReader(lines[start:])
        tot = defaultdict(float)
        cnt = defaultdict(int)
        for r in rd:
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            k = r["Kernel Name"].split("(")[0][:70]
            v = num(r["Metric Value"])
            unit = r.get("Metric Unit", "")
            scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
                     "ms": 1e3}
            v = v * scale.get(unit, 1e-3)  # -> us
            tot[k] += v
            cnt[k] += 1
        T = sum(tot.values())
        md.append(f"\n## launch list share ({title}; cold-cache serialised)\n")
        md.append("| kernel | launches | total us | share |")
        md.append("|---|---|---|---|")
        share = {}
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            md.append(f"| {k} | {cnt[k]} | {v:.1f} | {v / T * 100:.1f}% |")
            share[k] = v / T
        summary["launch_share" if lname == "launches.csv" else "launch_share_c5"] = share
        with open(os.path.join(dst, lname), "w") as fh:
            fh.write(open(lpath).read())
    g = summary.get("ncu_gemm_ring")
    if g:
        summary["gemm_ring_dram"] = [[r["dram__bytes_read.sum"], r["dram__bytes_write.sum"]]
                                     for r in g]
    for f in ("timeline_verify_m1000.txt", "timeline_prefill_m1000.txt", "fwd_time.txt",
              "forward_critical_path.txt", "bench_gemm_pair.txt", "bench_gemm_pair_epi.txt"):
        src = os.path.join(OUT, f)
        if os.path.exists(src):
            with open(src) as fi, open(os.path.join(dst, f), "w") as fo:
                fo.write(fi.read())
    with open(os.path.join(dst, "summary.md"), "w") as fh:
        fh.write("\n".join(md) + "\n")
    with open(os.path.join(dst, "summary.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "round1")
