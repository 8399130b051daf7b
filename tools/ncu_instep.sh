# In-step DRAM traffic of the finest-level refinement kernels: no cache
# control (L2 keeps what the previous kernels left), one metric pass.
O=gpurun_out; mkdir -p $O; T=${1:-instep}
HS_NCU_LEVEL0=1 timeout 900 ncu --cache-control none --clock-control none --profile-from-start off \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --csv --log-file $O/instep_$T.csv python tools/ncu_kway.py > $O/instep_$T.log 2>&1
echo "rc=$?"
python - "$O/instep_$T.csv" <<'PY'
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]; ki = hdr.index("Kernel Name"); mi = hdr.index("Metric Name"); vi = hdr.index("Metric Value"); ii = hdr.index("ID")
per = collections.defaultdict(dict)
names = {}
for r in rows[h + 1:]:
    per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
    names[r[ii]] = r[ki].split("(")[0][:40]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0])
for i, m in per.items():
    a = agg[names[i]]
    a[0] += 1; a[1] += m.get("gpu__time_duration.sum", 0) / 1e6
    a[2] += m.get("dram__bytes_read.sum", 0) / 1e6; a[3] += m.get("dram__bytes_write.sum", 0) / 1e6
    a[4] += m.get("lts__t_sector_hit_rate.pct", 0)
for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:40s} x{a[0]:3d} {a[1]:7.3f} ms  DRAM rd {a[2]/a[0]:8.1f} MB wr {a[3]/a[0]:8.1f} MB /launch  L2 hit {a[4]/a[0]:5.1f}%")
PY
