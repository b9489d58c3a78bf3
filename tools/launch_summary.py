"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per
kernel: launches, summed serialized time and share of this library's
kernels. cuBLAS (FP64 peak probe) and PyTorch kernels are listed apart.
Usage: python tools/launch_summary.py gpurun_out/launches_raw.csv > profiles/launches_c2_rNN.csv"""
import csv
import sys
from collections import defaultdict

SCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}
FOREIGN = ("xmma", "cutlass", "cublas", "at::", "void at", "elementwise_kernel", "gemmk", "gemv")

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
head = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[head]
ki, mi, ui, vi = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
agg = defaultdict(lambda: [0, 0.0])
for r in rows[head + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    a = agg[r[ki]]
    a[0] += 1
    a[1] += float(r[vi].replace(",", "")) * SCALE[r[ui]]
own = {k: v for k, v in agg.items() if not any(f in k for f in FOREIGN)}
other = {k: v for k, v in agg.items() if k not in own}
tot = sum(v[1] for v in own.values())
w = csv.writer(sys.stdout)
w.writerow(["kernel", "launches", "total_ms", "share_pct"])
for k, (n, ms) in sorted(own.items(), key=lambda x: -x[1][1]):
    w.writerow([k, n, f"{ms:.2f}", f"{100 * ms / tot:.1f}"])
for k, (n, ms) in sorted(other.items(), key=lambda x: -x[1][1]):
    w.writerow(["(not this library) " + k, n, f"{ms:.2f}", ""])
