"""Summarise an ncu report: key metrics, stall ratios, and the source lines with
the most stall samples.  usage: python tools/ncu_stalls.py REPORT.ncu-rep [nlines]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 12
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, v = r[0], r[2]
keep = ("gpu__time_duration.sum", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_requests_srcunit_tex_op_write.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active")
for k, x in zip(h, v):
    if k in keep or ("stall" in k and "ratio" in k and "not_issued" not in k):
        try:
            if float(x.replace(",", "")) > 0.1:
                print(f"  {k:70s} {x}")
        except ValueError:
            pass
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = next(x for x in rows if x and x[0] == "Line No")
idx = {n: i for i, n in enumerate(hdr)}
names = [n for n in hdr if n.startswith("stall_") and "Not Issued" not in n]
f, agg, det, text, tot = None, collections.Counter(), collections.defaultdict(collections.Counter), {}, 0
for x in rows:
    if not x:
        continue
    if x[0] == "File Path":
        f = x[1].split("/")[-1]
        continue
    if len(x) > 6 and x[0].isdigit():
        key = (f, int(x[0]))
        text[key] = x[1].strip()[:90]
        try:
            s = int(float(x[4]))
        except ValueError:
            s = 0
        agg[key] += s
        tot += s
        for n in names:
            try:
                det[key][n[6:]] += int(float(x[idx[n]]))
            except (ValueError, KeyError):
                pass
print(f"  stall samples: {tot}")
for k, s in agg.most_common(nl):
    print(f"  {s:6d} {100 * s / max(1, tot):5.1f}% {k[0]}:{k[1]} {text[k]}  {dict(det[k].most_common(3))}")
