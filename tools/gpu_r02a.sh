set -u
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi_r02a.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_r02a.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu_r02a.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_r02a.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke_r02a.log
timeout 900 python tools/probe_kway_quality.py > $O/kwayq_r02a.log 2>&1; echo "probe rc=$?"
timeout 900 python bench.py > $O/bench_r02a.json 2> $O/bench_r02a.err; echo "bench rc=$?"; tail -c 400 $O/bench_r02a.json
