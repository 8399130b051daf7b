#!/usr/bin/env bash
# usage (under gpurun): bash tools/gpu_small.sh TAG [pytest files...]
# partition A/B numbers (cut, part hash, ms), the partition step's launch list,
# then the named GPU tests
TAG=$1; shift
O=gpurun_out; mkdir -p $O
timeout 600 python tools/ab_defer.py 2>&1 | tail -2
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file $O/step_launches_$TAG.csv python tools/launches_kway.py > /dev/null 2>&1
echo "ncu rc=$?"
python tools/launch_summary.py $O/step_launches_$TAG.csv > $O/step_summary_$TAG.txt 2>&1
head -40 $O/step_summary_$TAG.txt
if [ $# -gt 0 ]; then
  timeout 1800 python -m pytest "$@" -m gpu -q -x > $O/pytest_$TAG.log 2>&1
  echo "pytest rc=$?"; tail -5 $O/pytest_$TAG.log
fi
