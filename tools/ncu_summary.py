"""Summarise ncu captures into profiles/ncu_summary.json (+ launch-list shares).

usage: python tools/ncu_summary.py OUT.json name=report.ncu-rep[:kernel_regex] ... [--launches launches.csv]
Each named entry records, for the first matching kernel launch, duration, DRAM
bytes (read+write = the bench's `traffic` field), throughput fractions,
occupancy and registers.
"""
import csv
import io
import json
import re
import subprocess
import sys


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def summarise(rep, pattern):
    h, units, rows = raw_rows(rep)
    picked = []
    for r in rows:
        d = dict(zip(h, r))
        if pattern and not re.search(pattern, d.get("Kernel Name", "")):
            continue
        picked.append(d)
    if not picked:
        return None
    keys = {
        "duration": "gpu__time_duration.sum",
        "dram_read": "dram__bytes_read.sum", "dram_write": "dram__bytes_write.sum",
        "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1_pct": "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "issue_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "registers": "launch__registers_per_thread",
        "l2_hit_pct": "lts__t_sector_hit_rate.pct",
        "tensor_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "dmma_inst": "sm__sass_inst_executed_op_dmma.sum",
    }
    ui = {k: units[h.index(v)] if v in h else "" for k, v in keys.items()}
    out = []
    for d in picked:
        e = {"kernel": d["Kernel Name"][:120]}
        for k, v in keys.items():
            x = num(d.get(v))
            if x is None:
                continue
            u = ui[k]
            if k.startswith("dram_") and k != "dram_pct":
                x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            if k == "duration":
                x *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3,
                      "ms": 1.0}.get(u, 1)
                k = "duration_ms"
            e[k] = x
        if "dram_read" in e and "dram_write" in e:
            e["dram_bytes_per_launch"] = e["dram_read"] + e["dram_write"]
        out.append(e)
    return out


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = {}, {}
    for r in rows[hi + 1:]:
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("<unnamed>::", "")
        v = num(r[vi]) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "nsecond": 1e-6, "usecond": 1e-3,
                          "msecond": 1.0}[r[ui]]
        tot[name] = tot.get(name, 0.0) + v
        cnt[name] = cnt.get(name, 0) + 1
    T = sum(tot.values())
    return {k: {"launches": cnt[k], "ms": round(v, 4), "share": round(v / T, 4)}
            for k, v in sorted(tot.items(), key=lambda kv: -kv[1])}


def main():
    out_path = sys.argv[1]
    res = {"kernels": {}, "note": "ncu --set full captures; per-launch dram bytes feed bench.py's "
                                   "roofline.traffic. Durations are under ncu (locked clocks, "
                                   "cold caches): compare shares, not absolutes."}
    args = sys.argv[2:]
    if "--launches" in args:
        i = args.index("--launches")
        res["launch_list"] = launch_shares(args[i + 1])
        args = args[:i] + args[i + 2:]
    for spec in args:
        name, rest = spec.split("=", 1)
        rep, _, pat = rest.partition(":")
        s = summarise(rep, pat)
        if s:
            res["kernels"][name] = s[0] | {"captures": len(s)}
    json.dump(res, open(out_path, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main()
