"""Multilevel policy sweep (temporary knobs) on layered and tiled-Cholesky DAGs."""
import os, subprocess, sys
code = r'''
import sys, time, torch
sys.path.insert(0, "."); sys.path.insert(0, "tools")
from paper_1502_07451_b200 import kway
spec = sys.argv[1]
if spec.startswith("chol"):
    from sweep_small import chol_ug
    ug, _ = chol_ug(int(spec[4:]))
else:
    n, d = map(int, spec.split("x"))
    ug = kway.symmetrize(kway.layered_dag(n, d * n, seed=3))
k = int(sys.argv[2])
kway.partition_kway(ug, k, tol=0.03, seed=0); torch.cuda.synchronize()
t0 = time.perf_counter(); r = kway.partition_kway(ug, k, tol=0.03, seed=0); torch.cuda.synchronize()
print("RES", r.cut, r.levels, round((time.perf_counter() - t0) * 1e3, 2))
'''
cfgs = [("full", {}), ("cap0", {"HS_FM_CAP": "0", "HS_FM_NINIT": "148"}),
        ("cap0t15", {"HS_FM_CAP": "0", "HS_FM_NINIT": "148", "HS_KWAY_CTARGET": "15"}),
        ("nofm", {"HS_FM_CAP": "0", "HS_FM_INITCAP": "0"}),
        ("nofmt15", {"HS_FM_CAP": "0", "HS_FM_INITCAP": "0", "HS_KWAY_CTARGET": "15"}),
        ("band", {"HS_KWAY_NOCOARSEN": "1"})]
for spec, k in (("20000x3", 8), ("20000x10", 8), ("100000x3", 8), ("100000x5", 8), ("chol32", 8), ("chol64", 2), ("chol64", 8)):
    out = []
    for name, env in cfgs:
        e = dict(os.environ, **env)
        o = subprocess.run([sys.executable, "-c", code, spec, str(k)], env=e, capture_output=True, text=True)
        res = [l for l in o.stdout.splitlines() if l.startswith("RES")]
        out.append(f"{name}: " + (" ".join(res[-1].split()[1:4:2]) if res else "ERR"))
    print(f"{spec:9s} k={k}: " + " | ".join(out), flush=True)
