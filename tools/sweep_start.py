"""Config-4 partition time and cut under env knobs (one subprocess per setting)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SETTINGS = [dict(), dict(HS_KWAY_NOCOARSEN="1")] + [
    dict(HS_KWAY_NOCOARSEN="1", HS_KWAY_PASSES=str(p)) for p in (3, 5, 6)] + [
    dict(HS_KWAY_PASSES=str(p)) for p in (3, 5)] + [dict(HS_KWAY_ROUNDS="1"), dict(HS_KWAY_ROUNDS="2")]
for st in SETTINGS:
    env = dict(os.environ, **st)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools/launches_kway.py")], env=env,
                         capture_output=True, text=True).stdout.strip()
    print(st, out, flush=True)
