# ncu --set full of the DOT ingestion kernels on the config-2 text (one GPU)
T=${1:-r02}
O=gpurun_out; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"count_lines|fill_lines|terms|line_spans|edge_values|name_heads" -c 7 \
  -o $O/dot_$T -f python tools/probe_dot.py > $O/ncu_dot_$T.log 2>&1
echo "ncu dot rc=$?"
python tools/ncu_summary.py $O/ncu_dot_summary_$T.json \
  count_lines=$O/dot_$T.ncu-rep:count_lines fill_lines=$O/dot_$T.ncu-rep:fill_lines \
  terms_count=$O/dot_$T.ncu-rep:"terms<0>|termsILb0" terms_write=$O/dot_$T.ncu-rep:"terms<1>|termsILb1" \
  line_spans=$O/dot_$T.ncu-rep:line_spans edge_values=$O/dot_$T.ncu-rep:edge_values \
  name_heads=$O/dot_$T.ncu-rep:name_heads > /dev/null 2>&1
echo "summary rc=$?"
rm -f $O/dot_$T.ncu-rep
