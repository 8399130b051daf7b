#!/usr/bin/env bash
# usage (under gpurun): bash tools/gpu_tests.sh TAG [pytest args...]
TAG=$1; shift
O=gpurun_out; mkdir -p $O
make -j8 >/dev/null 2>&1 || { echo "build failed"; make 2>&1 | tail -20; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q "$@" > $O/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error" $O/pytest_gpu_$TAG.log | tail -25
