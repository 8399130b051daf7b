import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
print(json.dumps(bench.policy_sweep(int(sys.argv[1]) if len(sys.argv) > 1 else 4096), indent=1))
