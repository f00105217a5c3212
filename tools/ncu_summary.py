"""Summarise ncu output for profiles/: a launch-list CSV (--metrics
gpu__time_duration.sum) into per-kernel shares, and .ncu-rep captures into
the metrics the roofline and DESIGN.md cite.

  python tools/ncu_summary.py launches <launches.csv>
  python tools/ncu_summary.py rep <file.ncu-rep> [...]
  python tools/ncu_summary.py json <out.json> <file.ncu-rep> [...]   (profiles/ncu_metrics.json)
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
        "smsp__inst_executed.sum"]


def launches(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        v *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(unit, 1.0)
        k = r["Kernel Name"].split("(")[0]
        tot[k] += v
        cnt[k] += 1
    s = sum(tot.values())
    print(f"# {path}: {sum(cnt.values())} launches, {s:.3f} ms total (cold-cache, serialised)")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k:40s} {cnt[k]:7d} launches {tot[k]:10.3f} ms {100 * tot[k] / s:6.2f} %")


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for v in rows[2:]:
        print(f"# {path}: {v[h.index('Kernel Name')][:60]}")
        for w in WANT:
            if w in h:
                print(f"  {w:70s} {v[h.index(w)]:>16s} {units[h.index(w)]}")


def _num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return None


def to_json(out_path, paths):
    """Per-kernel counters (one --set full capture each) for bench.py's roofline fields."""
    import json
    import os

    res = {}
    for path in paths:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        h, units = rows[0], rows[1]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                 "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9}
        for v in rows[2:]:
            def g(m):
                if m not in h:
                    return None
                x = _num(v[h.index(m)])
                return None if x is None else x * scale.get(units[h.index(m)], 1)
            name = v[h.index("Kernel Name")].split("(")[0].split("<")[0].strip()
            if name.startswith("void "):
                name = name[5:]
            dram = (g("dram__bytes_read.sum") or 0) + (g("dram__bytes_write.sum") or 0)
            conf = sum(g(m) or 0 for m in WANT if "bank_conflicts" in m)
            res[name] = {
                "source": f"profiles/{os.path.basename(out_path)} <- ncu --set full --clock-control none, {os.path.basename(path)}",
                "gpu_time_ms": (g("gpu__time_duration.sum") or 0) / 1e6,
                "issue_active": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "warps_active": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
                "pipe_alu": g("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
                "pipe_fma": g("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
                "pipe_fp64": g("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
                "pipe_lsu": g("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
                "dram_bytes_per_launch": dram,
                "dram_throughput_pct": g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                "shared_bank_conflicts": conf,
                "registers": g("launch__registers_per_thread"),
                "grid": g("launch__grid_size"), "block": g("launch__block_size"),
            }
    json.dump(res, open(out_path, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "json":
        to_json(sys.argv[2], sys.argv[3:])
        sys.exit(0)
    f = {"launches": launches, "rep": rep}[sys.argv[1]]
    for p in sys.argv[2:]:
        f(p)
