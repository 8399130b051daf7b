"""Summaries of an ncu --page source/details CSV pair: top stall SASS lines and key metrics."""
import csv, sys
tag = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rows = list(csv.reader(open(f"gpurun_out/{tag}_source.csv")))
hdr = rows[1]; data = rows[2:]
si = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[si]) for r in data if r[si].isdigit())
print("total samples", tot)
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
for r in sorted(data, key=lambda r: -int(r[si]) if r[si].isdigit() else 0)[:n]:
    top = sorted(((int(r[i]) if r[i].isdigit() else 0, hdr[i]) for i in stall_cols), reverse=True)[:2]
    print(r[si], r[0][-5:], r[1].strip()[:70], top)
rows = list(csv.reader(open(f"gpurun_out/{tag}_details.csv")))
hdr = rows[0]; idx = {h: i for i, h in enumerate(hdr)}
for r in rows[1:]:
    if r[idx["Metric Name"]] in ("Duration", "Achieved Occupancy", "DRAM Throughput", "L2 Hit Rate",
                                  "Issue Slots Busy", "Registers Per Thread", "Memory Throughput"):
        print(r[idx["Kernel Name"]][:30], r[idx["Metric Name"]], r[idx["Metric Value"]], r[idx["Metric Unit"]])
