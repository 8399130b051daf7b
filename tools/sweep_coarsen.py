"""Config-4 partition time and cut: probe shortcut vs forced coarsening, matching rounds, passes."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SETTINGS = [dict(), dict(HS_KWAY_PASSES="8"), dict(HS_KWAY_COARSEN="1")] + [
    dict(HS_KWAY_COARSEN="1", HS_KWAY_ROUNDS=r) for r in ("1", "2")] + [
    dict(HS_KWAY_COARSEN="1", HS_KWAY_PASSES=p) for p in ("3", "4")] + [
    dict(HS_KWAY_COARSEN="1", HS_KWAY_ROUNDS="1", HS_KWAY_PASSES="4")]
for st in SETTINGS:
    env = dict(os.environ, **st)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools/launches_kway.py")], env=env,
                         capture_output=True, text=True).stdout.strip()
    print(st, out, flush=True)
