# usage (under gpurun): bash tools/gpu_ab.sh TAG [case,case...]
set -u
T=$1; C=${2:-}
O=gpurun_out; mkdir -p $O
timeout 900 python tools/ab_fm.py ab_old $C > $O/ab_old_$T.txt 2>&1; echo "old rc=$?"
timeout 900 python tools/ab_fm.py . $C > $O/ab_new_$T.txt 2>&1; echo "new rc=$?"
paste <(awk '{print $1,$2,$4,$5,$6}' $O/ab_old_$T.txt) <(awk '{print $4,$5,$6}' $O/ab_new_$T.txt)
HS_KWAY_TRACE=1 python tools/trace_fm.py . 20000 8 2>&1 | grep -E "fm level|^cut" | tail -8
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/smoke_launches_$T.csv python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1; echo "ncu smoke rc=$?"
python tools/launch_summary.py $O/smoke_launches_$T.csv 2>/dev/null | head -8
