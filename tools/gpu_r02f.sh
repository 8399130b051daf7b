set -u
O=gpurun_out; mkdir -p $O
T=${1:-r02f}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi_$T.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$T.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke_$T.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/smoke_launches_$T.csv python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1; echo "ncu smoke rc=$?"
python tools/launch_summary.py $O/smoke_launches_$T.csv 2>/dev/null | head -30
timeout 900 python bench.py > $O/bench_$T.json 2> $O/bench_$T.err; echo "bench rc=$?"; tail -c 400 $O/bench_$T.json
