"""Summarise ncu output for profiles/: a launch list (--metrics
gpu__time_duration.sum --csv) and/or one --set full report of the top kernel.

  python tools/ncu_summary.py --launches gpurun_out/launches_c1.csv \
      --rep gpurun_out/prof_c1.ncu-rep --title "..." --out profiles/r01_c1.md \
      [--traffic-key C1]   # also records dram read+write bytes in profiles/traffic.json

Runs here (no GPU): `ncu -i` reads the report.
"""
import argparse
import collections
import csv
import io
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr, agg = None, collections.OrderedDict()
    for r in rows:
        if r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v = v / 1e3 if d["Metric Unit"] == "ns" else (v * 1e3 if d["Metric Unit"] == "ms" else v)
        agg.setdefault(d["Kernel Name"].split("(")[0], []).append(v)
    total = sum(sum(v) for v in agg.values())
    out = ["| launches | mean us | share of listed device time | kernel |", "|---:|---:|---:|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| {len(v)} | {sum(v) / len(v):.2f} | {100 * sum(v) / total:.1f}% | `{k[:110]}` |")
    return out


def full(rep):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = r[0], r[1], r[2]
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    got = {k: (v, u) for k, u, v in zip(hdr, units, vals) if k in KEYS}
    out = [f"kernel: `{name[:160]}`", "", "| metric | value | unit |", "|---|---:|---|"]
    for k in KEYS:
        if k in got:
            out.append(f"| {k} | {got[k][0]} | {got[k][1]} |")

    def nbytes(k):
        v, u = got.get(k, ("0", "byte"))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        return float(v.replace(",", "")) * scale
    return out, nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--title", required=True)
    ap.add_argument("--cmd", default="")
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic-key")
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    if a.cmd:
        lines += [f"command: `{a.cmd}`", ""]
    if a.launches:
        lines += ["## launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold, serialised)", ""]
        lines += launches(a.launches) + [""]
    if a.rep:
        lines += ["## top kernel, ncu --set full --clock-control none (one launch)", ""]
        body, traffic = full(a.rep)
        lines += body + ["", f"traffic (dram read + write) per launch: {traffic:.0f} bytes", ""]
        if a.traffic_key:
            tf = ROOT / "profiles" / "traffic.json"
            d = json.loads(tf.read_text()) if tf.exists() else {}
            d[a.traffic_key] = traffic
            tf.write_text(json.dumps(d, indent=1) + "\n")
    Path(a.out).write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
