# Round-2 final evidence: tests, bench, launch list, ncu of the partition
# kernels, K9, K7 dataflow, topo/trace/rgen kernels (one GPU).
set -u
T=${1:-r02z}
O=gpurun_out; mkdir -p $O
bash tools/gpu_round.sh $T tests bench launches ncu chol
timeout 600 ncu --set full --clock-control none --import-source on -k regex:levels_flow -c 1 \
  -o $O/k7_$T -f python tools/time_levels.py > $O/ncu_k7_$T.log 2>&1; echo "ncu k7 rc=$?"
python tools/ncu_summary.py $O/ncu_k7_summary_$T.json levels_flow=$O/k7_$T.ncu-rep:levels_flow > /dev/null 2>&1
rm -f $O/k7_$T.ncu-rep
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/misc_launches_$T.csv python tools/sanitize_all.py > /dev/null 2>&1; echo "misc launches rc=$?"
python tools/launch_summary.py $O/misc_launches_$T.csv > $O/misc_launch_summary_$T.txt 2>&1
head -25 $O/misc_launch_summary_$T.txt
