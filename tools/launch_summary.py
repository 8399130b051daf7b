"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per-kernel totals."""
import collections, csv, gzip, sys
path = sys.argv[1]
op = gzip.open if path.endswith(".gz") else open
rows = list(csv.reader(op(path, "rt")))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[h + 1:]:
    name = r[ki].split("(")[0][:60]
    tot[name] += float(r[vi].replace(",", "")) / 1e6
    cnt[name] += 1
print(f"total {sum(tot.values()):.3f} ms over {sum(cnt.values())} launches")
for n, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:8.3f} ms {cnt[n]:4d}  {n}")
